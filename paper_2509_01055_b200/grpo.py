"""Batched GRPO trajectory-to-loss step on device-resident tensors.

    packed  = packing.pack_table(table)                        # K1
    step    = GRPOStep(hidden_dim, vocab, LossConfig(...))
    res     = step(packed, group_off, rewards, hidden, weight, logp_old, logp_ref)
              # K2 advantages -> K4 fused LM-head logp + surrogate -> K5 backward

Reference semantics: cli.loss (cli.py:272-345) drives token_records ->
group_advantages -> grpo_multi_turn_loss per task_id group and aggregates
objective = sum_g obj_g / n_groups.  Here one call does the whole batch with
the log-probs computed by the fused LM head instead of read from a sidecar,
and returns the trainer-facing loss gradients (loss = -objective).
Multi-rank: shard whole groups across ranks (parallel.shard_groups), pass the
global normalisers, and all-reduce the report (parallel.allreduce_report).
"""

from __future__ import annotations

from dataclasses import dataclass

import ctypes as C

import numpy as np

from . import _lib
from .packing import PackedBatch
from .rl.loss import AGG_TOKEN_MEAN, LossConfig

REPORT_KEYS = ("objective", "clip_fraction", "masked_tokens", "kl", "groups", "episodes",
               "total_tokens", "clamp_count", "clipped", "kl_sum", "entropy_sum",
               "objective_sum")

DEFAULT_CHUNK_ROWS = 148 * 128 * 2  # two 128-row M-tiles per SM per vocab strip wave
# The step picks the largest multiple (up to this) of DEFAULT_CHUNK_ROWS
# whose workspace fits in half of the free HBM: fewer, larger chunks amortise
# each GEMM's ramp / tail and the dW accumulation (C2: 2x -0.7 %, 4x -1.2 %,
# tools/experiments/gpu_r43.sh).  Pass chunk_rows for a fixed size.
MAX_CHUNK_MULT = 4


def report_dict(rep) -> dict:
    vals = rep.tolist() if hasattr(rep, "tolist") else list(rep)
    d = dict(zip(REPORT_KEYS, vals))
    for k in ("masked_tokens", "groups", "episodes", "total_tokens", "clamp_count", "clipped"):
        d[k] = int(d[k])
    return d


class _Workspace:
    def __init__(self):
        self.buf = None

    def get(self, nbytes: int, device):
        import torch

        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            self.buf = None
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
        return self.buf


def _group_sizes(group_off) -> np.ndarray:
    go = np.asarray(group_off, dtype=np.int64)
    return np.diff(go)


def _check_groups(go: np.ndarray, n_rewards: int | None, n_traj: int | None) -> None:
    """Host-side shape checks before any launch (the reference raises
    MaskMismatch for these length mismatches, loss.py:45-49, :85-90)."""
    from .errors import MaskMismatch

    if go.ndim != 1 or len(go) < 1 or go[0] != 0 or np.any(np.diff(go) < 0):
        raise ValueError("group_off must be a non-decreasing offset array starting at 0")
    if n_rewards is not None and n_rewards != int(go[-1]):
        raise MaskMismatch(f"{n_rewards} rewards for {int(go[-1])} trajectories in group_off")
    if n_traj is not None and n_traj != int(go[-1]):
        raise MaskMismatch(f"group_off covers {int(go[-1])} trajectories, the batch has {n_traj}")


def _check_tensor(name: str, t, dtype, n: int | None, device, *, rank: int = 1) -> None:
    """Every tensor handed to the C ABI: dtype, contiguity, device and length
    (a float64 log-prob tensor would otherwise be reinterpreted as float32)."""
    if t is None:
        return
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")
    if t.dim() != rank:
        raise ValueError(f"{name} must have {rank} dimension(s), got shape {tuple(t.shape)}")
    if n is not None and t.shape[0] != n:
        from .errors import MaskMismatch

        raise MaskMismatch(f"{name} has {t.shape[0]} entries, expected {n}")


def _on(stream):
    """Run the host side of an operator with `stream` as torch's current
    stream, so its temporaries are allocated (and freed) in that stream's
    order and the final report read (.cpu()) is ordered after the kernels."""
    import contextlib

    import torch

    return torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()


def _stream_scoped(fn):
    """Operators taking `stream=`: the whole host side runs under _on(stream)."""
    import functools

    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        with _on(kwargs.get("stream")):
            return fn(*args, **kwargs)

    return wrapped


def _n_rewards(rewards) -> int:
    return int(rewards.numel()) if hasattr(rewards, "numel") else len(rewards)


@_stream_scoped
def advantages(rewards, group_off, n_act_per_traj=None, *, std_floor: float = 1e-6,
               agg: int = 0, norm_groups: float | None = None, norm_tokens: float | None = None,
               act_off=None, device=None, stream=None):
    """K2 over a whole batch.  Returns (adv64, adv32, traj_w, traj_group) device
    tensors.  group_off (host int array) delimits contiguous groups."""
    import torch

    L = _lib.lib()
    go = np.asarray(group_off, dtype=np.int32)
    _check_groups(go, _n_rewards(rewards), None)
    sizes = _group_sizes(go)
    if np.any(sizes < 2):
        from .errors import GroupTooSmall

        g = int(np.argmax(sizes < 2))
        raise GroupTooSmall(f"group {g}: need at least 2 rewards, got {int(sizes[g])}")
    device = torch.device(device or "cuda")
    n_groups = len(go) - 1
    B = int(go[-1])
    r = rewards if torch.is_tensor(rewards) else torch.from_numpy(
        np.ascontiguousarray(np.asarray(rewards, dtype=np.float64)))
    r = r.to(device=device, dtype=torch.float64)
    d_go = torch.from_numpy(go).to(device)
    adv64 = torch.empty(B, dtype=torch.float64, device=device)
    adv32 = torch.empty(B, dtype=torch.float32, device=device)
    traj_w = torch.empty(B, dtype=torch.float32, device=device)
    tgroup = torch.empty(B, dtype=torch.int32, device=device)
    ng = float(norm_groups if norm_groups is not None else n_groups)
    nt = float(norm_tokens if norm_tokens is not None else 1.0)
    _lib.check(L.tl_group_advantages(r.data_ptr(), d_go.data_ptr(), n_groups, B, std_floor,
                                     _lib.ptr(act_off), agg, ng, nt, adv64.data_ptr(),
                                     adv32.data_ptr(), traj_w.data_ptr(), tgroup.data_ptr(),
                                     _lib.stream_handle(stream)))
    return adv64, adv32, traj_w, tgroup, d_go


@dataclass
class StepResult:
    report: dict
    report_tensor: "object"   # float64 [TL_REPORT_LEN] on device
    logp: "object"            # float32 [T] (0 at observation positions)
    entropy: "object"         # float32 [T]
    dhidden: "object"         # bf16 [T, H] or None
    dweight: "object"         # float32 [V, H] or None
    adv: "object"             # float64 [B]


class GRPOStep:
    """Fused GRPO step: advantages + LM-head log-prob/entropy + surrogate +
    backward, all on the device.  Reusable across steps (workspace cached)."""

    def __init__(self, hidden_dim: int, vocab: int, cfg: LossConfig | None = None,
                 chunk_rows: int | None = None, recompute: bool = False,
                 pipelined: bool = False, split_tail: bool = True, factored: bool = True,
                 debug_fixup: bool = False):
        """recompute=False keeps each chunk's logits for the backward
        (6*T*H*V FLOPs; bf16 q when factored, else fp16); True recomputes them in a second GEMM (8*T*H*V) so no
        logit ever leaves TMEM.  pipelined=True (store mode) double-buffers the
        chunk workspace and runs each chunk's dS pass beside the next chunk's
        forward GEMM (include/toolloop_b200.h, TL_LMHEAD_*); bitwise equal to
        the serial schedule but measured 3 % slower at C2 on a power-capped
        B200 (the GEMM slows by as much as the pass it hides), so off by
        default.  factored=True (store mode, entropy_coef == 0): the forward
        stores bf16 q = e^(z - m0) against a per-row anchor and dS = alpha_r q
        reaches the dH / dW GEMMs without an elementwise pass (False:
        TL_LMHEAD_NO_FACTORED); debug_fixup (tests) routes every row through
        the out-of-range fallback."""
        self.H = int(hidden_dim)
        self.V = int(vocab)
        self.cfg = cfg or LossConfig()
        self.chunk_rows = chunk_rows
        if recompute:
            self.mode = _lib.LMHEAD_RECOMPUTE
        elif pipelined:
            self.mode = _lib.LMHEAD_STORE_LOGITS_PIPELINED
        else:
            self.mode = _lib.LMHEAD_STORE_LOGITS
        # split_tail=False (tests): the dW GEMM's partial last wave runs unsplit
        self.flags = 0 if split_tail else _lib.LMHEAD_NO_SPLIT_TAIL
        if not factored:
            self.flags |= _lib.LMHEAD_NO_FACTORED
        if debug_fixup:
            self.flags |= _lib.LMHEAD_DEBUG_FIXUP
        self._ws = _Workspace()
        self.last_chunk = None  # chunk rows used by the latest call

    def workspace_bytes(self, n_act: int, n_tokens: int, n_traj: int, n_groups: int) -> int:
        L = _lib.lib()
        return int(L.tl_lmhead_step_workspace_bytes(self._chunk(n_act), self.H, self.V, n_tokens,
                                                    n_traj, n_groups, self.mode))

    def _chunk(self, n_act: int, n_tokens: int = 0, n_traj: int = 0, n_groups: int = 0,
               device=None) -> int:
        if self.chunk_rows:
            return int(self.chunk_rows)
        rows = max(128, (n_act + 127) // 128 * 128)
        if rows <= DEFAULT_CHUNK_ROWS:
            return int(rows)
        mult = min(MAX_CHUNK_MULT, -(-n_act // DEFAULT_CHUNK_ROWS))
        if device is not None and mult > 1:
            import torch

            L = _lib.lib()
            free, _ = torch.cuda.mem_get_info(device)
            free += torch.cuda.memory_reserved(device) - torch.cuda.memory_allocated(device)
            if self._ws.buf is not None and self._ws.buf.device == device:
                free += self._ws.buf.numel()
            while mult > 1 and L.tl_lmhead_step_workspace_bytes(
                    mult * DEFAULT_CHUNK_ROWS, self.H, self.V, n_tokens, n_traj, n_groups,
                    self.mode) > free // 2:
                mult -= 1
        return int(mult * DEFAULT_CHUNK_ROWS)

    def __call__(self, packed: PackedBatch, group_off, rewards, hidden, weight, logp_old,
                 logp_ref=None, *, backward: bool = True, norm_groups: float | None = None,
                 norm_tokens: float | None = None, stream=None, outputs=None,
                 adv_cache=None, sync_report: bool = True,
                 accumulate_dweight: bool = False, want_dhidden: bool = True,
                 want_dweight: bool = True, dw_ready=None, reserve_sms: int = 0) -> StepResult:
        """One step over `packed`.  Micro-batching an optimizer step: call once
        per micro-batch with the step's global norm_groups / norm_tokens and
        accumulate_dweight=True after the first (outputs["dweight"] reused),
        then combine the reports with parallel.combine_reports.
        want_dweight=False: frozen LM head (dS + dH only, no dW GEMM);
        want_dhidden=False: dW only.  `stream`: a torch.cuda.Stream to run on
        (temporaries are allocated in its order; the report read waits on it).
        dw_ready: a torch.cuda.Event recorded as soon as dweight is final,
        before the last chunk's dH GEMM, which then leaves reserve_sms SMs
        free — make another stream wait on it and issue the dW all-reduce
        there to overlap N2 with that GEMM (parallel.NcclComm.allreduce_grad;
        include/toolloop_b200.h, tl_grpo_lmhead_step_overlap)."""
        with _on(stream):
            plan = self._prepare(packed, group_off, rewards, hidden, weight, logp_old, logp_ref,
                                 backward=backward, norm_groups=norm_groups,
                                 norm_tokens=norm_tokens, outputs=outputs, adv_cache=adv_cache,
                                 accumulate_dweight=accumulate_dweight,
                                 want_dhidden=want_dhidden, want_dweight=want_dweight,
                                 dw_ready=dw_ready, reserve_sms=reserve_sms)
            if stream is not None:
                plan.ws.record_stream(stream)
            self._launch(plan, stream)
            return plan.result(sync_report)

    def capture(self, packed: PackedBatch, group_off, rewards, hidden, weight, logp_old,
                logp_ref=None, *, norm_groups: float | None = None,
                norm_tokens: float | None = None, outputs=None) -> "CapturedStep":
        """Record the whole device side of a step (advantages + fused LM-head
        step + reductions) as one CUDA graph.  Every argument becomes a
        static buffer: refill packed / hidden / logp / rewards tensors in place
        (same shapes) and call replay().  rewards must be a device tensor."""
        import torch

        plan = self._prepare(packed, group_off, rewards, hidden, weight, logp_old, logp_ref,
                             backward=True, norm_groups=norm_groups, norm_tokens=norm_tokens,
                             outputs=outputs, adv_cache=None, accumulate_dweight=False,
                             want_dhidden=True, want_dweight=True)
        if plan.rewards.data_ptr() != getattr(rewards, "data_ptr", lambda: -1)():
            raise ValueError("capture() needs rewards as a float64 device tensor (static input)")
        side = torch.cuda.Stream(device=hidden.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # warm-up (occupancy queries, lazy loads) off-capture
            self._launch(plan, None)
        torch.cuda.current_stream().wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            self._launch(plan, None)
        return CapturedStep(graph, plan)

    def _prepare(self, packed, group_off, rewards, hidden, weight, logp_old, logp_ref, *,
                 backward, norm_groups, norm_tokens, outputs, adv_cache, accumulate_dweight,
                 want_dhidden, want_dweight, dw_ready=None, reserve_sms=0):
        import torch

        L = _lib.lib()
        dev = hidden.device
        if hidden.dtype != torch.bfloat16 or weight.dtype != torch.bfloat16:
            raise TypeError("hidden and weight must be bfloat16")
        if hidden.shape != (packed.n_tokens, self.H) or weight.shape != (self.V, self.H):
            raise ValueError(f"hidden {tuple(hidden.shape)} / weight {tuple(weight.shape)} do not "
                             f"match T={packed.n_tokens}, H={self.H}, V={self.V}")
        _check_tensor("hidden", hidden, torch.bfloat16, packed.n_tokens, dev, rank=2)
        _check_tensor("weight", weight, torch.bfloat16, self.V, dev, rank=2)
        _check_tensor("logp_old", logp_old, torch.float32, packed.n_tokens, dev)
        _check_tensor("logp_ref", logp_ref, torch.float32, packed.n_tokens, dev)
        for k in ("input_ids", "loss_mask", "act_idx", "traj_of_token", "cu_seqlens", "act_off"):
            if getattr(packed, k).device != dev:
                raise ValueError(f"packed.{k} is on {getattr(packed, k).device}, expected {dev}")
        cfg = self.cfg
        agg = 1 if cfg.loss_agg == AGG_TOKEN_MEAN else 0
        go = np.asarray(group_off, dtype=np.int32)
        _check_groups(go, _n_rewards(rewards) if adv_cache is None else None, packed.n_traj)
        n_groups = len(go) - 1
        plan = _StepPlan()
        plan.L = L
        if adv_cache is None:
            sizes = _group_sizes(go)
            if np.any(sizes < 2):
                from .errors import GroupTooSmall

                g = int(np.argmax(sizes < 2))
                raise GroupTooSmall(f"group {g}: need at least 2 rewards, got {int(sizes[g])}")
            B = int(go[-1])
            r = rewards if torch.is_tensor(rewards) else torch.from_numpy(
                np.ascontiguousarray(np.asarray(rewards, dtype=np.float64)))
            plan.rewards = r.to(device=dev, dtype=torch.float64)
            plan.d_go = torch.from_numpy(go).to(dev)
            plan.adv64 = torch.empty(B, dtype=torch.float64, device=dev)
            plan.adv32 = torch.empty(B, dtype=torch.float32, device=dev)
            plan.traj_w = torch.empty(B, dtype=torch.float32, device=dev)
            plan.tgroup = torch.empty(B, dtype=torch.int32, device=dev)
            nt = norm_tokens if norm_tokens is not None else max(packed.n_act, 1)
            plan.adv_args = (plan.rewards.data_ptr(), plan.d_go.data_ptr(), n_groups, B,
                             cfg.std_floor, _lib.ptr(packed.act_off), agg,
                             float(norm_groups if norm_groups is not None else n_groups),
                             float(nt), plan.adv64.data_ptr(), plan.adv32.data_ptr(),
                             plan.traj_w.data_ptr(), plan.tgroup.data_ptr())
        else:
            plan.adv64, plan.adv32, plan.traj_w, plan.d_go = adv_cache
            plan.adv_args = None
        T = packed.n_tokens
        out = outputs or {}

        def buf(key, shape, dtype):
            t = out.get(key)
            return t if t is not None else torch.empty(shape, dtype=dtype, device=dev)

        plan.T = T
        plan.logp = buf("logp", max(T, 1), torch.float32)
        plan.ent = buf("entropy", max(T, 1), torch.float32)
        plan.dh = buf("dhidden", (T, self.H), torch.bfloat16) if backward and want_dhidden else None
        plan.dw = buf("dweight", (self.V, self.H), torch.float32) if backward and want_dweight else None
        _check_tensor("outputs['dhidden']", plan.dh, torch.bfloat16, T, dev, rank=2)
        _check_tensor("outputs['dweight']", plan.dw, torch.float32, self.V, dev, rank=2)
        plan.rep = buf("report", _lib.TL_REPORT_LEN, torch.float64)
        chunk = self._chunk(packed.n_act, T, packed.n_traj, n_groups, dev)
        self.last_chunk = chunk
        ws_bytes = int(L.tl_lmhead_step_workspace_bytes(chunk, self.H, self.V, T, packed.n_traj,
                                                        n_groups, self.mode))
        plan.ws = self._ws.get(ws_bytes, dev)
        plan.cfg_c = cfg.to_c(use_mask=1, has_ref=int(logp_ref is not None), objective=0,
                              entropy_norm=float(norm_tokens if norm_tokens is not None
                                                 else max(packed.n_act, 1)))
        plan.keep = (packed, hidden, weight, logp_old, logp_ref)  # pointers stay valid
        plan.overlap = None
        if dw_ready is not None:  # N2 overlap (tl_grpo_lmhead_step_overlap)
            ev = dw_ready.cuda_event
            if not ev:  # torch creates the CUDA event lazily, on its first record
                dw_ready.record()
                ev = dw_ready.cuda_event
            plan.overlap = _lib.StepOverlapC(C.c_void_p(ev), int(reserve_sms))
            plan.keep = plan.keep + (dw_ready,)
        plan.step_args = (
            hidden.data_ptr(), weight.data_ptr(), packed.input_ids.data_ptr(),
            packed.loss_mask.data_ptr(), packed.act_idx.data_ptr(), packed.n_act,
            packed.traj_of_token.data_ptr(), packed.cu_seqlens.data_ptr(), plan.d_go.data_ptr(),
            logp_old.data_ptr(), _lib.ptr(logp_ref), plan.adv32.data_ptr(),
            plan.traj_w.data_ptr(), T, self.H, self.V, packed.n_traj, n_groups, plan.cfg_c,
            plan.logp.data_ptr(), plan.ent.data_ptr(), _lib.ptr(plan.dh), _lib.ptr(plan.dw),
            plan.rep.data_ptr(), chunk,
            self.mode | self.flags | (_lib.LMHEAD_ACCUMULATE_DW if accumulate_dweight else 0),
            plan.ws.data_ptr(), ws_bytes)
        return plan

    @staticmethod
    def _launch(plan, stream):
        """Device work only (stream-ordered launches, no host sync): K2 then
        the fused LM-head step; capturable."""
        L = plan.L
        s = _lib.stream_handle(stream)
        if plan.adv_args is not None:
            _lib.check(L.tl_group_advantages(*plan.adv_args, s))
        if plan.overlap is not None:
            _lib.check(L.tl_grpo_lmhead_step_overlap(*plan.step_args, s, C.byref(plan.overlap)))
        else:
            _lib.check(L.tl_grpo_lmhead_step(*plan.step_args, s))


class _StepPlan:
    """Buffers and C-call arguments of one GRPOStep call (see _prepare)."""

    def result(self, sync_report: bool = True) -> StepResult:
        T = self.T
        return StepResult(report=report_dict(self.rep.cpu()) if sync_report else {},
                          report_tensor=self.rep, logp=self.logp[:T], entropy=self.ent[:T],
                          dhidden=self.dh, dweight=self.dw, adv=self.adv64)


class CapturedStep:
    """A GRPO step recorded as one CUDA graph (GRPOStep.capture): replay()
    re-runs advantages + fused LM-head forward / surrogate / backward +
    reductions on the current contents of the captured input buffers."""

    def __init__(self, graph, plan):
        self.graph = graph
        self.plan = plan

    def replay(self) -> None:
        self.graph.replay()

    def result(self, sync_report: bool = True) -> StepResult:
        return self.plan.result(sync_report)


@_stream_scoped
def grpo_loss(packed: PackedBatch, group_off, rewards, logp_new, logp_old, logp_ref=None,
              cfg: LossConfig | None = None, *, want_grad: bool = True, stream=None):
    """Standalone fp32 K3 over a packed batch with given logp_new (e.g. from a
    sidecar).  Returns (report dict, grad d objective / d logp_new [T])."""
    import torch

    L = _lib.lib()
    cfg = cfg or LossConfig()
    dev = logp_new.device
    for k, t in (("logp_new", logp_new), ("logp_old", logp_old), ("logp_ref", logp_ref)):
        _check_tensor(k, t, torch.float32, packed.n_tokens, dev)
    agg = 1 if cfg.loss_agg == AGG_TOKEN_MEAN else 0
    go = np.asarray(group_off, dtype=np.int32)
    _check_groups(go, _n_rewards(rewards), packed.n_traj)
    n_groups = len(go) - 1
    _, adv32, traj_w, _, d_go = advantages(rewards, go, std_floor=cfg.std_floor, agg=agg,
                                           norm_tokens=max(packed.n_act, 1),
                                           act_off=packed.act_off, device=dev, stream=stream)
    T = packed.n_tokens
    grad = torch.empty(max(T, 1), dtype=torch.float32, device=dev) if want_grad else None
    rep = torch.empty(_lib.TL_REPORT_LEN, dtype=torch.float64, device=dev)
    ws_bytes = int(L.tl_loss_f32_workspace_bytes(max(T, 1), packed.n_traj, n_groups))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    c = cfg.to_c(use_mask=1, has_ref=int(logp_ref is not None), objective=0)
    _lib.check(L.tl_loss_f32(logp_new.data_ptr(), logp_old.data_ptr(), _lib.ptr(logp_ref),
                             packed.loss_mask.data_ptr(), packed.traj_of_token.data_ptr(),
                             packed.cu_seqlens.data_ptr(), d_go.data_ptr(), adv32.data_ptr(),
                             traj_w.data_ptr(), packed.n_traj, n_groups, T, c, _lib.ptr(grad),
                             rep.data_ptr(), ws.data_ptr(), ws_bytes, _lib.stream_handle(stream)))
    return report_dict(rep.cpu()), (grad[:T] if want_grad else None)


@_stream_scoped
def report_f64(packed: PackedBatch, group_off, rewards, logp_new, logp_old, logp_ref=None,
               cfg: LossConfig | None = None, stream=None) -> dict:
    """cli.loss's report (cli.py:309-345) for a whole packed batch in the fp64
    parity kernels: K2 advantages per group, K3 per group in reference order,
    then the reference aggregation.  logp_* are float64 device tensors [T]
    (logp_ref may hold NaN where a token has no reference)."""
    import torch

    L = _lib.lib()
    cfg = cfg or LossConfig()
    dev = packed.cu_seqlens.device
    for k, t in (("logp_new", logp_new), ("logp_old", logp_old), ("logp_ref", logp_ref)):
        _check_tensor(k, t, torch.float64, packed.n_tokens, dev)
    go = np.asarray(group_off, dtype=np.int32)
    _check_groups(go, _n_rewards(rewards), packed.n_traj)
    n_groups = len(go) - 1
    adv64, _, _, _, d_go = advantages(rewards, go, std_floor=cfg.std_floor, device=dev,
                                      stream=stream)
    T = packed.n_tokens
    ws_bytes = int(L.tl_loss_f64_workspace_bytes(max(T, 1)))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    gout = torch.empty(max(n_groups, 1) * _lib.TL_GROUP_OUT_LEN, dtype=torch.float64, device=dev)
    rep = torch.empty(_lib.TL_REPORT_LEN, dtype=torch.float64, device=dev)
    c = cfg.to_c(use_mask=1, has_ref=int(logp_ref is not None), objective=0)
    s = _lib.stream_handle(stream)
    _lib.check(L.tl_loss_f64(logp_new.data_ptr(), logp_old.data_ptr(), _lib.ptr(logp_ref),
                             packed.loss_mask.data_ptr(), packed.cu_seqlens.data_ptr(),
                             d_go.data_ptr(), adv64.data_ptr(), packed.n_traj, n_groups, T, c,
                             None, gout.data_ptr(), ws.data_ptr(), ws_bytes, s))
    _lib.check(L.tl_report_f64(gout.data_ptr(), n_groups, packed.n_traj, rep.data_ptr(), s))
    return report_dict(rep.cpu())


@_stream_scoped
def lmhead_logprobs(hidden, weight, targets, rows=None, *, chunk_rows: int | None = None,
                    stream=None):
    """Forward-only fused LM head (F3: rollout-side logp_old / logp_ref).
    Returns (logp, entropy, lse) float32 for hidden rows `rows` (default all)."""
    import torch

    L = _lib.lib()
    H = hidden.shape[1]
    V = weight.shape[0]
    n = hidden.shape[0] if rows is None else rows.shape[0]
    dev = hidden.device
    _check_tensor("hidden", hidden, torch.bfloat16, None, dev, rank=2)
    _check_tensor("weight", weight, torch.bfloat16, None, dev, rank=2)
    if weight.shape[1] != H:
        raise ValueError(f"weight {tuple(weight.shape)} does not match hidden dim {H}")
    _check_tensor("targets", targets, torch.int32, None, dev)
    _check_tensor("rows", rows, torch.int32, None, dev)
    if rows is None and targets.shape[0] < n:
        from .errors import MaskMismatch

        raise MaskMismatch(f"{targets.shape[0]} targets for {n} hidden rows")
    # forward-only workspace is small (h_c + per-row stats, no dS buffer):
    # always the largest chunk
    chunk = int(chunk_rows or min(MAX_CHUNK_MULT * DEFAULT_CHUNK_ROWS, max(128, (n + 127) // 128 * 128)))
    ws_bytes = int(L.tl_lmhead_logprobs_workspace_bytes(chunk, H, V))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    logp = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
    ent = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
    lse = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
    _lib.check(L.tl_lmhead_logprobs(hidden.data_ptr(), weight.data_ptr(), targets.data_ptr(),
                                    _lib.ptr(rows), n, H, V, logp.data_ptr(), ent.data_ptr(),
                                    lse.data_ptr(), chunk, ws.data_ptr(), ws_bytes,
                                    _lib.stream_handle(stream)))
    return logp[:n], ent[:n], lse[:n]


def gemm(A, B, *, a_mn_major=False, b_mn_major=False, out=None, out_fp32=False,
         accumulate=False, stream=None):
    """tcgen05 GEMM building block: C = A_op @ B_op^T where A_op is A ([M,K])
    or A^T (A given [K,M] when a_mn_major) and likewise for B ([N,K] / [K,N])."""
    import torch

    L = _lib.lib()
    M, K = (A.shape[1], A.shape[0]) if a_mn_major else (A.shape[0], A.shape[1])
    N = B.shape[1] if b_mn_major else B.shape[0]
    KB = B.shape[0] if b_mn_major else B.shape[1]
    if KB != K:
        raise ValueError("K mismatch")
    if out is None:
        out = torch.empty((M, N), dtype=torch.float32 if out_fp32 else torch.bfloat16,
                          device=A.device)
    _lib.check(L.tl_gemm_bf16(A.data_ptr(), int(a_mn_major), A.stride(0), B.data_ptr(),
                              int(b_mn_major), B.stride(0), M, N, K, out.data_ptr(),
                              int(out.dtype == torch.float32), out.stride(0), int(accumulate),
                              _lib.stream_handle(stream)))
    return out
