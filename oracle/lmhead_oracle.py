"""numpy restatement of the fused LM-head log-prob / entropy and its gradient.

TEST INFRASTRUCTURE ONLY.  "Parity unpinned": the reference has no log-prob
computation; its contract is `PolicyAction.token_logprobs` — one
log-probability per generated token (rollout/policy.py:3-6, :25-28) — consumed
as `TokenRecord.logp_new` (rl/loss.py:30).  The build's definition:

  z[t, v]   = sum_k h[t, k] * W[v, k]            (bf16 inputs, fp32 products)
  lse[t]    = log sum_v exp(z[t, v])
  logp[t]   = z[t, y_t] - lse[t]
  ent[t]    = lse[t] - sum_v p[t, v] z[t, v],     p = exp(z - lse)
  dZ[t, v]  = g[t] (onehot(y_t)[v] - p[t, v]) - c[t] p[t, v] (z[t, v] - E_p[z_t])
  dH        = dZ @ W,   dW = dZ^T @ h

with g = dLoss/dlogp and c = dLoss/dent per token.  Inputs are bf16-rounded
(round-to-nearest-even) and held in fp32; reductions over V run in fp64.
"""

from __future__ import annotations

import numpy as np


def to_bf16_f32(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (RNE) and return the value as fp32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit patterns (uint16), RNE."""
    return (to_bf16_f32(x).view(np.uint32) >> 16).astype(np.uint16)


def bf16_from_bits(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


def lmhead_forward(h: np.ndarray, W: np.ndarray, y: np.ndarray, chunk: int = 512,
                   exact: bool = False):
    """h [T, H] fp32 (bf16 values), W [V, H] fp32 (bf16 values), y [T] int.
    Returns logp, ent, lse (fp64 [T]).  exact=True forms the logits in fp64
    (bf16 products are exact in fp64), so the only error left is the GPU's."""
    T = h.shape[0]
    logp = np.empty(T)
    ent = np.empty(T)
    lse = np.empty(T)
    Wt = np.ascontiguousarray(W.T, dtype=np.float64 if exact else W.dtype)
    for s in range(0, T, chunk):
        e = min(T, s + chunk)
        hs = h[s:e].astype(np.float64) if exact else h[s:e]
        z = (hs @ Wt).astype(np.float64)
        m = z.max(axis=1, keepdims=True)
        ex = np.exp(z - m)
        se = ex.sum(axis=1, keepdims=True)
        l = (m + np.log(se))[:, 0]
        p = ex / se
        lse[s:e] = l
        logp[s:e] = z[np.arange(e - s), y[s:e]] - l
        ent[s:e] = l - (p * z).sum(axis=1)
    return logp, ent, lse


def lmhead_fwd_bwd_f64(h, W, y, g_fn, c, chunk: int = 4096):
    """The same equations in torch float64 on whatever device h / W live on
    (large-shape checker for the GPU tests: C2 / C5 vocab at tens of
    thousands of rows is hours in numpy).  h [T, H], W [V, H] bf16 tensors,
    y [T] int.  The upstream gradients may depend on the forward: g_fn(logp)
    -> g [T] (float64 tensor), c scalar or [T] tensor = dLoss/dent.  Returns
    (logp, ent, lse, dH, dW) in float64; dS is kept in float64 (no rounding),
    so dH / dW are the exact-arithmetic gradients of the bf16 inputs."""
    import torch

    T = h.shape[0]
    dev = h.device
    W64 = W.to(torch.float64)
    y = y.to(device=dev, dtype=torch.long)
    logp = torch.empty(T, dtype=torch.float64, device=dev)
    ent = torch.empty_like(logp)
    lse = torch.empty_like(logp)
    ez = torch.empty_like(logp)
    for s in range(0, T, chunk):
        e = min(T, s + chunk)
        z = h[s:e].to(torch.float64) @ W64.T
        l = torch.logsumexp(z, dim=1)
        p = torch.exp(z - l[:, None])
        lse[s:e] = l
        logp[s:e] = z.gather(1, y[s:e, None])[:, 0] - l
        ez[s:e] = (p * z).sum(1)
        ent[s:e] = l - ez[s:e]
        del z, p
    g = g_fn(logp).to(device=dev, dtype=torch.float64)
    c = torch.as_tensor(c, dtype=torch.float64, device=dev).expand(T)
    dH = torch.empty((T, W.shape[1]), dtype=torch.float64, device=dev)
    dW = torch.zeros_like(W64)
    for s in range(0, T, chunk):
        e = min(T, s + chunk)
        hs = h[s:e].to(torch.float64)
        z = hs @ W64.T
        p = torch.exp(z - lse[s:e, None])
        dz = -g[s:e, None] * p - c[s:e, None] * p * (z - ez[s:e, None])
        dz[torch.arange(e - s, device=dev), y[s:e]] += g[s:e]
        dH[s:e] = dz @ W64
        dW += dz.T @ hs
        del z, p, dz
    return logp, ent, lse, dH, dW


def lmhead_backward(h, W, y, g, c=None, chunk: int = 512):
    """Returns dH [T, H] fp32 and dW [V, H] fp32 for per-token upstream grads
    g = dLoss/dlogp and c = dLoss/dent (None -> 0)."""
    T, H = h.shape
    V = W.shape[0]
    dH = np.zeros((T, H), dtype=np.float32)
    dW = np.zeros((V, H), dtype=np.float32)
    Wt = np.ascontiguousarray(W.T)
    for s in range(0, T, chunk):
        e = min(T, s + chunk)
        z = (h[s:e] @ Wt).astype(np.float64)
        m = z.max(axis=1, keepdims=True)
        ex = np.exp(z - m)
        p = ex / ex.sum(axis=1, keepdims=True)
        dz = -g[s:e, None] * p
        dz[np.arange(e - s), y[s:e]] += g[s:e]
        if c is not None:
            ez = (p * z).sum(axis=1, keepdims=True)
            dz -= c[s:e, None] * p * (z - ez)
        dz32 = dz.astype(np.float32)
        dH[s:e] = dz32 @ W
        dW += dz32.T @ h[s:e]
    return dH, dW
