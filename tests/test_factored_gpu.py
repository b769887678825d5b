"""Factored LM-head backward (store mode, entropy_coef == 0).

Without the entropy bonus dLoss/dz = g (onehot(y) - p) is, row by row, a
multiple of q = e^(z - m0) for an anchor m0 fixed before the forward, so the
forward stores bf16 q, the strip merge computes alpha_r = -g_r e^(m0 - lse)
and rewrites the target element, and dH = diag(alpha) (q W),
dW = q^T (diag(alpha) h_c) need no elementwise dS pass
(csrc/lmhead_epilogue.cuh, combine_row / EpiLseStatsT<true>).

Checked here:
  * forward outputs (logp, entropy, report) bitwise equal to the fp16-logit
    store (TL_LMHEAD_NO_FACTORED): the log-sum-exp is unchanged;
  * dH / dW against the float64 oracle (rel Frobenius 5e-3, as every other
    backward test);
  * the out-of-range fallback (rows whose lse - m0 leaves [-45, 80] are
    recomputed on CUDA cores with m0 = lse): forced on every row
    (TL_LMHEAD_DEBUG_FIXUP), and reached naturally with |z| ~ 100 logits and
    behaviour log-probs that are far from the current policy;
  * far-off-anchor rows without a gradient (|z| ~ 150): exact-zero dH rows,
    no NaN / inf.
"""

import numpy as np
import pytest

from oracle import grpo_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2509_01055_b200 import grpo, packing  # noqa: E402
from paper_2509_01055_b200.rl import loss as L  # noqa: E402
from test_gpu_parity import BWD_TOL, _bf16_np, _bwd_err, _oracle_report, _synthetic_batch, _traj  # noqa: E402


def _setup(H, V, seed=4, wstd=0.05):
    trajs, rewards, go, _, lold, lref = _synthetic_batch(seed, n_groups=6, G=4)
    for tr in trajs:
        for i, (o, toks) in enumerate(tr):
            tr[i] = (o, [t % V for t in toks])
    packed = packing.pack([_traj(s) for s in trajs])
    T = packed.n_tokens
    g = torch.Generator(device="cuda").manual_seed(17 + seed)
    h = torch.randn(T, H, device="cuda", generator=g).bfloat16()
    W = (torch.randn(V, H, device="cuda", generator=g) * wstd).bfloat16()
    return trajs, rewards, go, lold, lref, packed, h, W


def _oracle_grads(trajs, rewards, go, packed, h, W, lold, lref, beta):
    from oracle import lmhead_oracle as LH

    T = packed.n_tokens
    ids = packed.input_ids.cpu().numpy()
    act = packed.act_idx.cpu().numpy()
    hn, Wn = _bf16_np(h), _bf16_np(W)
    lp, en, lse = LH.lmhead_forward(hn[act], Wn, ids[act], exact=True)
    lnew = np.zeros(T)
    lnew[act] = lp
    lo32 = lold.astype(np.float32).astype(np.float64)
    lr32 = None if lref is None else lref.astype(np.float32).astype(np.float64)
    ref, groups = _oracle_report(trajs, rewards, go, lnew, lo32, lr32, beta=beta)
    n_groups = len(go) - 1
    gl = np.zeros(T)
    pos = 0
    for recs_g, rw in groups:
        for row in O.clipped_grad(recs_g, O.group_advantages(rw), 0.2, beta):
            for e in row:
                gl[pos] = -e / n_groups
                pos += 1
    dH, dW = LH.lmhead_backward(hn[act], Wn, ids[act], gl[act], np.zeros(len(act)))
    return lp, lse, ref, gl, dH, dW


def _f(a):
    return torch.from_numpy(np.asarray(a, dtype=np.float32)).cuda()


def _check_vs_oracle(name, res, packed, lp, ref, dH, dW, lp_tol=1e-4):
    act = packed.act_idx.cpu().numpy()
    got_lp = res.logp.cpu().numpy()
    assert np.abs(got_lp[act] - lp).max() <= lp_tol
    assert res.report["masked_tokens"] == ref["masked_tokens"]
    got_dh = res.dhidden.float().cpu().numpy()
    assert np.all(got_dh[packed.loss_mask.cpu().numpy() == 0] == 0)
    assert _bwd_err(f"{name}_dH", got_dh[act], dH) <= BWD_TOL
    assert _bwd_err(f"{name}_dW", res.dweight.cpu().numpy(), dW) <= BWD_TOL


def _same_forward(a, b):
    assert torch.equal(a.logp, b.logp)
    assert torch.equal(a.entropy, b.entropy)
    assert a.report == b.report


@pytest.mark.parametrize("H,V,chunk", [(256, 1000, None), (128, 2304, 256), (192, 517, 128),
                                       (128, 1000, 200), (64, 100, None), (64, 257, 64)])
def test_factored_vs_fp16_store_and_oracle(H, V, chunk):
    trajs, rewards, go, lold, lref, packed, h, W = _setup(H, V)
    cfg = L.LossConfig(kl_beta=0.1)  # entropy_coef 0: the factored store applies
    res = grpo.GRPOStep(H, V, cfg, chunk_rows=chunk)(packed, go, rewards, h, W, _f(lold), _f(lref))
    old = grpo.GRPOStep(H, V, cfg, chunk_rows=chunk, factored=False)(
        packed, go, rewards, h, W, _f(lold), _f(lref))
    torch.cuda.synchronize()
    _same_forward(res, old)
    lp, _, ref, _, dH, dW = _oracle_grads(trajs, rewards, go, packed, h, W, lold, lref, 0.1)
    _check_vs_oracle(f"factored_H{H}_V{V}_c{chunk}", res, packed, lp, ref, dH, dW)
    _check_vs_oracle(f"fp16store_H{H}_V{V}_c{chunk}", old, packed, lp, ref, dH, dW)


@pytest.mark.parametrize("H,V,chunk", [(256, 1000, None), (192, 517, 128)])
def test_factored_fixup_path_every_row(H, V, chunk):
    """Every row through the out-of-range fallback (q rewritten with m0 = lse
    from CUDA-core logits): same forward, same oracle bar."""
    trajs, rewards, go, lold, lref, packed, h, W = _setup(H, V, seed=5)
    cfg = L.LossConfig(kl_beta=0.1)
    res = grpo.GRPOStep(H, V, cfg, chunk_rows=chunk, debug_fixup=True)(
        packed, go, rewards, h, W, _f(lold), _f(lref))
    base = grpo.GRPOStep(H, V, cfg, chunk_rows=chunk)(packed, go, rewards, h, W, _f(lold), _f(lref))
    torch.cuda.synchronize()
    _same_forward(res, base)
    lp, _, ref, _, dH, dW = _oracle_grads(trajs, rewards, go, packed, h, W, lold, lref, 0.1)
    _check_vs_oracle(f"fixup_all_H{H}_V{V}_c{chunk}", res, packed, lp, ref, dH, dW)


def test_factored_out_of_range_rows_natural():
    """Logits with |z| ~ 100 and behaviour log-probs of 0 (anchor m0 = z_y):
    rows with logp_new < -80 leave the anchor's range; their gradient comes
    from the KL term (the ratio is clamped there), so the fallback must
    produce it."""
    H, V = 256, 1000
    trajs, rewards, go, _, _, packed, h, W = _setup(H, V, seed=6, wstd=25.0 / 16.0)
    from oracle import lmhead_oracle as LH

    T = packed.n_tokens
    act = packed.act_idx.cpu().numpy()
    ids = packed.input_ids.cpu().numpy()
    lp, _, _ = LH.lmhead_forward(_bf16_np(h)[act], _bf16_np(W), ids[act], exact=True)
    lold = np.zeros(T)
    rng = np.random.default_rng(3)
    lref = np.full(T, -1.0)
    lref[act] = lp + rng.normal(0, 0.5, len(act))
    beta = 0.2
    far = lp < -85.0
    assert far.sum() >= 10, "the case must reach the fallback"
    cfg = L.LossConfig(kl_beta=beta)
    res = grpo.GRPOStep(H, V, cfg)(packed, go, rewards, h, W, _f(lold), _f(lref))
    old = grpo.GRPOStep(H, V, cfg, factored=False)(packed, go, rewards, h, W, _f(lold), _f(lref))
    torch.cuda.synchronize()
    _same_forward(res, old)
    lp2, lse, ref, gl, dH, dW = _oracle_grads(trajs, rewards, go, packed, h, W, lold, lref, beta)
    assert np.any(gl[act][far] != 0)
    tol = 1e-4 + 1e-5 * float(np.abs(lse).max())
    _check_vs_oracle("factored_far_rows", res, packed, lp2, ref, dH, dW, lp_tol=tol)
    # the far rows alone (the fallback's output), per row
    got = res.dhidden.float().cpu().numpy()[act][far]
    assert _bwd_err("factored_far_rows_only_dH", got, dH[far]) <= BWD_TOL


def test_entropy_bonus_keeps_fp16_store():
    """entropy_coef != 0: dS has a p * z term, the factored store does not
    apply and the call runs the fp16-logit store + dS pass (bitwise equal to
    forcing it)."""
    H, V = 128, 1000
    trajs, rewards, go, lold, lref, packed, h, W = _setup(H, V, seed=7)
    cfg = L.LossConfig(kl_beta=0.1, entropy_coef=0.01)
    a = grpo.GRPOStep(H, V, cfg)(packed, go, rewards, h, W, _f(lold), _f(lref))
    b = grpo.GRPOStep(H, V, cfg, factored=False)(packed, go, rewards, h, W, _f(lold), _f(lref))
    torch.cuda.synchronize()
    _same_forward(a, b)
    assert torch.equal(a.dhidden, b.dhidden)
    assert torch.equal(a.dweight, b.dweight)


def test_factored_far_rows_without_gradient_stay_finite():
    """|z| ~ 150 logits, logp_old = 0 and no KL term: rows with logp_new
    < -88 sit e^88+ above their anchor and have a zero gradient (clamped
    ratio).  Their q saturates near the bf16 range and their dH accumulators
    may overflow fp32; the zero row scale must still give exact-zero dH rows
    and leave dW untouched (no NaN / inf anywhere)."""
    H, V = 256, 1000
    trajs, rewards, go, _, _, packed, h, W = _setup(H, V, seed=8, wstd=38.0 / 16.0)
    from oracle import lmhead_oracle as LH

    T = packed.n_tokens
    act = packed.act_idx.cpu().numpy()
    ids = packed.input_ids.cpu().numpy()
    lp, _, _ = LH.lmhead_forward(_bf16_np(h)[act], _bf16_np(W), ids[act], exact=True)
    assert (lp < -100).sum() >= 10, "the case must reach far-off-anchor rows"
    lold = np.zeros(T)
    cfg = L.LossConfig()
    res = grpo.GRPOStep(H, V, cfg)(packed, go, rewards, h, W, _f(lold))
    torch.cuda.synchronize()
    assert torch.isfinite(res.dweight).all() and torch.isfinite(res.dhidden.float()).all()
    far = act[lp < -30]  # ratio clamped (|logp_new - logp_old| > 20): zero gradient
    assert torch.all(res.dhidden[torch.from_numpy(far).cuda()] == 0)
    lp2, lse, ref, gl, dH, dW = _oracle_grads(trajs, rewards, go, packed, h, W, lold, None, 0.0)
    tol = 1e-4 + 1e-5 * float(np.abs(lse).max())
    _check_vs_oracle("factored_far_rows_no_grad", res, packed, lp2, ref, dH, dW, lp_tol=tol)
