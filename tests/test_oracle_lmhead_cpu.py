"""Pin the LM-head oracle (oracle/lmhead_oracle.py) on CPU.

The reference has no LM head, so the oracle's equations cannot be checked
against reference output; instead they are checked against an independent
implementation of their *definition*: torch float64 `log_softmax` for the
forward, and torch autograd of  L = sum_t g_t logp_t + c_t ent_t  for the
backward (dZ = g (onehot - p) - c p (z - E_p z) is exactly dL/dz).  Both
oracle entry points the GPU tests use are covered: the numpy
`lmhead_forward` / `lmhead_backward` (small shapes) and the torch
`lmhead_fwd_bwd_f64` (full-shape checker)."""

import numpy as np
import pytest

from oracle import lmhead_oracle as LH

torch = pytest.importorskip("torch")


def _inputs(seed, T=37, H=64, V=301, scale=0.3):
    rng = np.random.default_rng(seed)
    h = LH.to_bf16_f32(rng.standard_normal((T, H)).astype(np.float32))
    W = LH.to_bf16_f32((rng.standard_normal((V, H)) * scale).astype(np.float32))
    y = rng.integers(0, V, T)
    g = rng.standard_normal(T)
    c = rng.standard_normal(T) * 0.1
    return h, W, y, g, c


def _autograd(h, W, y, g, c):
    ht = torch.tensor(h, dtype=torch.float64, requires_grad=True)
    Wt = torch.tensor(W, dtype=torch.float64, requires_grad=True)
    z = ht @ Wt.T
    lp_all = torch.log_softmax(z, dim=1)
    logp = lp_all[torch.arange(len(y)), torch.tensor(y)]
    ent = -(lp_all.exp() * lp_all).sum(1)
    lse = torch.logsumexp(z, dim=1)
    L = (torch.tensor(g) * logp).sum() + (torch.tensor(c) * ent).sum()
    L.backward()
    return (logp.detach().numpy(), ent.detach().numpy(), lse.detach().numpy(),
            ht.grad.numpy(), Wt.grad.numpy())


@pytest.mark.parametrize("seed,scale", [(0, 0.3), (1, 3.0)])
def test_numpy_oracle_matches_torch_definition(seed, scale):
    h, W, y, g, c = _inputs(seed, scale=scale)
    lp, en, lse = LH.lmhead_forward(h, W, y, chunk=16, exact=True)
    rlp, ren, rlse, rdh, rdw = _autograd(h, W, y, g, c)
    assert np.abs(lp - rlp).max() <= 1e-10
    assert np.abs(en - ren).max() <= 1e-10
    assert np.abs(lse - rlse).max() <= 1e-10
    # numpy backward forms dZ in fp64 and the GEMMs in fp32
    dH, dW = LH.lmhead_backward(h, W, y, g, c, chunk=16)
    assert np.linalg.norm(dH - rdh) <= 1e-5 * np.linalg.norm(rdh)
    assert np.linalg.norm(dW - rdw) <= 1e-5 * np.linalg.norm(rdw)


def test_torch_f64_checker_matches_torch_definition():
    h, W, y, g, c = _inputs(2, T=53, H=48, V=517, scale=2.0)
    hb = torch.tensor(h).bfloat16()
    Wb = torch.tensor(W).bfloat16()
    gt = torch.tensor(g)
    lp, en, lse, dH, dW = LH.lmhead_fwd_bwd_f64(hb, Wb, torch.tensor(y), lambda logp: gt,
                                                torch.tensor(c), chunk=20)
    rlp, ren, rlse, rdh, rdw = _autograd(h, W, y, g, c)
    assert np.abs(lp.numpy() - rlp).max() <= 1e-10
    assert np.abs(en.numpy() - ren).max() <= 1e-10
    assert np.abs(lse.numpy() - rlse).max() <= 1e-10
    assert np.abs(dH.numpy() - rdh).max() <= 1e-10 * max(1.0, np.abs(rdh).max())
    assert np.abs(dW.numpy() - rdw).max() <= 1e-10 * max(1.0, np.abs(rdw).max())
