"""Drop-in for toolloop/rl/loss.py — the same names, signatures, defaults,
return types and exceptions, computed by the CUDA kernels.

Reference anchors (toolloop/rl/loss.py): RATIO_CLAMP :22-24, TokenRecord
:27-33, GroupBatch :36-49, LossConfig :52-64, LossDiagnostics :67-73,
token_records :76-100, group_advantages :103-116, token_ratio :119-126,
grpo_multi_turn_loss :150-201, grpo_single_turn_loss :204-227,
unclipped_objective :230-270.

These per-group entry points run the fp64 parity kernels (tl_loss_f64,
tl_group_advantages): the reference's operation order in IEEE fp64, exact
(fsum) group sums, correctly rounded exp.  Host-side validation mirrors the
reference's eager checks so the same exception fires before any launch.
Batched / fp32 training paths live in paper_2509_01055_b200.grpo.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .. import _lib
from ..errors import GroupTooSmall, MaskMismatch
from ..trajectory import Trajectory

RATIO_CLAMP = 20.0

AGG_REFERENCE = "seq-mean-token-mean"
AGG_TOKEN_MEAN = "token-mean"


@dataclass(frozen=True)
class TokenRecord:
    token: int
    logp_new: float
    logp_old: float
    action_bit: int
    logp_ref: float | None = None


@dataclass
class GroupBatch:
    """G trajectories answering the same input, with one scalar reward each."""

    group_id: str
    trajectories: list[list[TokenRecord]]
    rewards: list[float]

    def __post_init__(self) -> None:
        if len(self.trajectories) != len(self.rewards):
            raise MaskMismatch(
                f"group {self.group_id!r}: {len(self.trajectories)} trajectories "
                f"vs {len(self.rewards)} rewards"
            )


@dataclass(frozen=True)
class LossConfig:
    """Reference fields first (positional-compatible); the rest are build
    extensions with reference-neutral defaults."""

    epsilon_clip: float = 0.2
    kl_beta: float = 0.0
    std_floor: float = 1e-6
    eps_high: float | None = None        # DAPO clip-higher; None = epsilon_clip
    loss_agg: str = AGG_REFERENCE        # or "token-mean" (DAPO)
    entropy_coef: float = 0.0            # LM-head path only

    def __post_init__(self) -> None:
        if not 0.0 < self.epsilon_clip < 1.0:
            raise ValueError("epsilon_clip must lie in (0, 1)")
        if self.kl_beta < 0.0:
            raise ValueError("kl_beta must be non-negative")
        if self.std_floor <= 0.0:
            raise ValueError("std_floor must be positive")
        if self.eps_high is not None and self.eps_high <= 0.0:
            raise ValueError("eps_high must be positive")
        if self.loss_agg not in (AGG_REFERENCE, AGG_TOKEN_MEAN):
            raise ValueError(f"loss_agg must be {AGG_REFERENCE!r} or {AGG_TOKEN_MEAN!r}")

    def to_c(self, *, use_mask: int = 1, has_ref: int = 0, objective: int = 0,
             entropy_norm: float = 0.0) -> _lib.LossConfigC:
        return _lib.LossConfigC(
            eps_low=self.epsilon_clip,
            eps_high=self.epsilon_clip if self.eps_high is None else self.eps_high,
            kl_beta=self.kl_beta, entropy_coef=self.entropy_coef, use_mask=use_mask,
            has_ref=has_ref, objective=objective,
            agg=1 if self.loss_agg == AGG_TOKEN_MEAN else 0, entropy_norm=float(entropy_norm))


@dataclass
class LossDiagnostics:
    masked_tokens: int
    total_tokens: int
    clip_fraction: float
    clamp_count: int
    kl: float


def token_records(
    traj: Trajectory,
    logp_new: Sequence[float],
    logp_old: Sequence[float],
    logp_ref: Sequence[float] | None = None,
) -> list[TokenRecord]:
    """Pair a trajectory's flattened tokens with per-token log-probabilities
    (ids and mask from the GPU packer)."""
    from ..packing import pack

    packed = pack([traj])
    tokens = packed.input_ids.cpu().tolist()
    mask = packed.loss_mask.cpu().tolist()
    if not (len(tokens) == len(logp_new) == len(logp_old)):
        raise MaskMismatch(
            f"{len(tokens)} tokens vs {len(logp_new)} new / {len(logp_old)} old logps"
        )
    if logp_ref is not None and len(logp_ref) != len(tokens):
        raise MaskMismatch(f"{len(tokens)} tokens vs {len(logp_ref)} ref logps")
    return [
        TokenRecord(t, float(logp_new[i]), float(logp_old[i]), mask[i],
                    float(logp_ref[i]) if logp_ref is not None else None)
        for i, t in enumerate(tokens)
    ]


# ------------------------------------------------------------- device glue --

def _cuda(a: np.ndarray):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")


def group_advantages(rewards: Sequence[float], std_floor: float = 1e-6) -> list[float]:
    """Centre by the group mean, divide by max(population std, floor) — K2."""
    if len(rewards) < 2:
        raise GroupTooSmall(f"need at least 2 rewards, got {len(rewards)}")
    import torch

    L = _lib.lib()
    r = _cuda(np.asarray(rewards, dtype=np.float64))
    off = _cuda(np.asarray([0, len(rewards)], dtype=np.int32))
    adv = torch.empty(len(rewards), dtype=torch.float64, device="cuda")
    _lib.check(L.tl_group_advantages(r.data_ptr(), off.data_ptr(), 1, len(rewards), std_floor,
                                     None, 0, 1.0, 1.0, adv.data_ptr(), None, None, None,
                                     _lib.stream_handle()))
    return adv.cpu().tolist()


def token_ratio(rec: TokenRecord) -> float:
    """exp(clamp(logp_new - logp_old, +-20)) on the device (fp64)."""
    import torch

    L = _lib.lib()
    a = torch.tensor([rec.logp_new], dtype=torch.float64, device="cuda")
    b = torch.tensor([rec.logp_old], dtype=torch.float64, device="cuda")
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    _lib.check(L.tl_token_ratio_f64(a.data_ptr(), b.data_ptr(), 1, out.data_ptr(),
                                    _lib.stream_handle()))
    return float(out.item())


def _check_alignment(batch: GroupBatch, advantages: Sequence[float]) -> None:
    if len(advantages) != len(batch.trajectories):
        raise MaskMismatch(
            f"group {batch.group_id!r}: {len(advantages)} advantages "
            f"vs {len(batch.trajectories)} trajectories"
        )
    if not batch.trajectories:
        raise GroupTooSmall("empty group")


def _group_f64(batch: GroupBatch, advantages: Sequence[float], cfg: LossConfig, *, use_mask: int,
               objective: int, want_grad: bool):
    """Run tl_loss_f64 on one group; returns (group_out row, per-token grads)."""
    import torch

    L = _lib.lib()
    recs = [r for t in batch.trajectories for r in t]
    n = len(recs)
    lens = [len(t) for t in batch.trajectories]
    cu = np.zeros(len(lens) + 1, dtype=np.int32)
    cu[1:] = np.cumsum(lens)
    has_ref = any(r.logp_ref is not None for r in recs)
    new = np.fromiter((r.logp_new for r in recs), dtype=np.float64, count=n)
    old = np.fromiter((r.logp_old for r in recs), dtype=np.float64, count=n)
    ref = (np.fromiter((math.nan if r.logp_ref is None else r.logp_ref for r in recs),
                       dtype=np.float64, count=n) if has_ref else None)
    mask = np.fromiter((1 if r.action_bit else 0 for r in recs), dtype=np.uint8, count=n)
    pad1 = lambda a: a if len(a) else np.zeros(1, a.dtype)  # noqa: E731
    d_new, d_old, d_mask = _cuda(pad1(new)), _cuda(pad1(old)), _cuda(pad1(mask))
    d_ref = _cuda(pad1(ref)) if has_ref else None
    d_cu = _cuda(cu)
    d_off = _cuda(np.asarray([0, len(lens)], dtype=np.int32))
    d_adv = _cuda(np.asarray(advantages, dtype=np.float64))
    grad = torch.empty(max(n, 1), dtype=torch.float64, device="cuda") if want_grad else None
    out = torch.empty(_lib.TL_GROUP_OUT_LEN, dtype=torch.float64, device="cuda")
    ws_bytes = L.tl_loss_f64_workspace_bytes(max(n, 1))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    c = cfg.to_c(use_mask=use_mask, has_ref=int(has_ref), objective=objective)
    _lib.check(L.tl_loss_f64(d_new.data_ptr(), d_old.data_ptr(), _lib.ptr(d_ref),
                             d_mask.data_ptr(), d_cu.data_ptr(), d_off.data_ptr(),
                             d_adv.data_ptr(), len(lens), 1, n, c, _lib.ptr(grad),
                             out.data_ptr(), ws.data_ptr(), ws_bytes, _lib.stream_handle()))
    row = out.cpu().tolist()
    grads = None
    if want_grad:
        flat = grad[:n].cpu().tolist()
        grads = [flat[cu[i]:cu[i + 1]] for i in range(len(lens))]
    return row, grads


def grpo_multi_turn_loss(
    batch: GroupBatch, advantages: Sequence[float], cfg: LossConfig
) -> tuple[float, LossDiagnostics]:
    """Clipped objective over action tokens only (observation tokens are
    skipped, so their log-probs cannot change the result — bitwise)."""
    _check_alignment(batch, advantages)
    row, _ = _group_f64(batch, advantages, cfg, use_mask=1, objective=0, want_grad=False)
    diag = LossDiagnostics(
        masked_tokens=int(row[1]), total_tokens=int(row[2]), clip_fraction=row[6],
        clamp_count=int(row[4]), kl=row[7])
    return row[0], diag


def grpo_single_turn_loss(
    batch: GroupBatch, advantages: Sequence[float], cfg: LossConfig
) -> float:
    """Clipped objective normalised over all tokens, ignoring the mask; the
    same kernel and op order as the multi-turn loss (bitwise equal on
    all-action trajectories)."""
    _check_alignment(batch, advantages)
    row, _ = _group_f64(batch, advantages, cfg, use_mask=0, objective=0, want_grad=False)
    return row[0]


def unclipped_objective(
    batch: GroupBatch, advantages: Sequence[float], cfg: LossConfig
) -> tuple[float, list[list[float]]]:
    """Unclipped arm and its gradient w.r.t. each logp_new (0 on observation
    tokens and where the ratio clamp is active)."""
    _check_alignment(batch, advantages)
    row, grads = _group_f64(batch, advantages, cfg, use_mask=1, objective=1, want_grad=True)
    return row[0], grads


def clipped_objective_grad(
    batch: GroupBatch, advantages: Sequence[float], cfg: LossConfig
) -> tuple[float, list[list[float]]]:
    """Build extension: the clipped objective and its gradient (the r*A arm
    where it is the active min, else 0; parity unpinned, oracle-checked)."""
    _check_alignment(batch, advantages)
    row, grads = _group_f64(batch, advantages, cfg, use_mask=1, objective=0, want_grad=True)
    return row[0], grads
