"""Seeded synthetic GRPO workloads of the BASELINE.json shapes.

Per trajectory: k tool turns -> 2k+1 alternating segments ending on an
action; length l ~ U[L/2, L] (C5: lognormal, ragged); observation share
f_obs split over the k observation segments and the rest over the k+1
action segments by Dirichlet(1) partitions (>= 1 action token each); ids
~ U[0, V).  logp_old = -Exp(1); logp_ref = logp_old + N(0, 0.05).  Segments
are laid into the token pool in arrival order (turn-major across the batch,
as an asynchronous rollout would deliver them), so the packer's scatter is
real.  Hidden states / LM-head weights are generated on the device by the
caller (bench.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .packing import SegmentTable

SEED0 = 250901055


@dataclass(frozen=True)
class WorkloadConfig:
    name: str
    prompts: int
    n: int               # rollouts per prompt (group size G)
    turns: tuple         # (min, max) tool turns
    seq: int             # L
    hidden: int
    vocab: int
    f_obs: float
    rewards: str         # "pm1", "math", "swe"
    loss_agg: str = "seq-mean-token-mean"
    ragged: bool = False
    desc: str = ""


CONFIGS = {
    "c1": WorkloadConfig("c1", 8, 4, (2, 2), 1024, 896, 32000, 0.25, "math",
                         desc="math TIR GRPO step: 8x4, 2 turns, seq 1k, H 896, V 32k"),
    "c2": WorkloadConfig("c2", 256, 8, (0, 4), 4096, 3584, 152064, 0.30, "pm1",
                         desc="Qwen2.5-7B-shape GRPO step: 256x8, <=4 turns, seq 4k, H 3584, V 152064, bf16"),
    "c3": WorkloadConfig("c3", 512, 8, (6, 6), 8192, 3584, 152064, 0.50, "pm1",
                         desc="search-R1/SQL: 512x8, 6 turns, ~50% obs, seq 8k"),
    "c4": WorkloadConfig("c4", 128, 8, (0, 3), 16384, 3584, 152064, 0.50, "pm1",
                         desc="Pixel-Reasoner VL shape: image/video obs masked, seq 16k, varlen"),
    "c5": WorkloadConfig("c5", 64, 8, (30, 40), 32768, 4096, 151936, 0.50, "swe",
                         loss_agg="token-mean", ragged=True,
                         desc="SWE long-horizon: 64x8, 30+ turns, seq 32k, ragged, DAPO token-mean"),
    # small shapes for tests / profiling
    "c2s": WorkloadConfig("c2s", 32, 8, (0, 4), 4096, 3584, 152064, 0.30, "pm1",
                          desc="1/8 of C2 (profiling)"),
    "tiny": WorkloadConfig("tiny", 4, 4, (0, 3), 256, 256, 1000, 0.30, "pm1", desc="smoke"),
}


def _partition(rng, total: int, parts: int, minimum: int) -> np.ndarray:
    if parts == 0:
        return np.zeros(0, dtype=np.int64)
    base = np.full(parts, minimum, dtype=np.int64)
    rest = total - minimum * parts
    if rest <= 0:
        return base
    return base + rng.multinomial(rest, rng.dirichlet(np.ones(parts)))


@dataclass
class Workload:
    cfg: WorkloadConfig
    table: SegmentTable
    group_off: np.ndarray     # int32 [n_groups+1]
    rewards: np.ndarray       # float64 [B]
    logp_old: np.ndarray      # float32 [T]
    logp_ref: np.ndarray      # float32 [T]
    group_ids: np.ndarray     # global group index of each local group

    @property
    def n_tokens(self) -> int:
        return self.table.n_tokens

    @property
    def n_act(self) -> int:
        return self.table.n_act


def group_act_tokens(cfg: WorkloadConfig, group_ids, seed: int | None = None) -> np.ndarray:
    """Action-token count per group without materialising ids (for LPT)."""
    return np.asarray([_group_shape(cfg, int(g), seed)[1] for g in group_ids])


def group_tokens(cfg: WorkloadConfig, group_ids, seed: int | None = None) -> np.ndarray:
    """Packed-token count per group (action + observation) without ids."""
    return np.asarray([sum(int(l.sum()) for l in _group_shape(cfg, int(g), seed)[0])
                       for g in group_ids])


def _group_shape(cfg: WorkloadConfig, g: int, seed: int | None):
    rng = np.random.default_rng([SEED0 if seed is None else seed, g])
    segs = []
    act = 0
    for _ in range(cfg.n):
        k = int(rng.integers(cfg.turns[0], cfg.turns[1] + 1))
        if cfg.ragged:
            length = int(np.clip(rng.lognormal(np.log(cfg.seq / 3), 0.6), 2 * k + 2, cfg.seq))
        else:
            length = int(rng.integers(cfg.seq // 2, cfg.seq + 1))
        n_obs = int(round(cfg.f_obs * length)) if k > 0 else 0
        n_act = max(length - n_obs, k + 1)
        a = _partition(rng, n_act, k + 1, 1)
        o = _partition(rng, n_obs, k, 0)
        lens = np.empty(2 * k + 1, dtype=np.int64)
        lens[0::2] = a
        lens[1::2] = o
        segs.append(lens)
        act += int(a.sum())
    rewards = _rewards(cfg, rng)
    return segs, act, rewards


def _rewards(cfg: WorkloadConfig, rng) -> np.ndarray:
    if cfg.rewards == "math":
        return rng.choice([1.0, -1.25], cfg.n)          # rewards.py reward_math
    if cfg.rewards == "swe":
        return (rng.random(cfg.n) < 0.2).astype(np.float64)  # reward_swe {0, 1}
    return rng.choice([1.0, -1.0], cfg.n)               # reward_match +-1


def make_workload(cfg: WorkloadConfig, group_ids=None, seed: int | None = None,
                  arrival_order: bool = True) -> Workload:
    """Generate the groups `group_ids` (default: all prompts) of `cfg`."""
    if group_ids is None:
        group_ids = np.arange(cfg.prompts)
    group_ids = np.asarray(group_ids, dtype=np.int64)
    seg_lens, traj_nseg, rewards = [], [], []
    for g in group_ids:
        segs, _, r = _group_shape(cfg, int(g), seed)
        for lens in segs:
            seg_lens.append(lens)
            traj_nseg.append(len(lens))
        rewards.append(r)
    seg_len = np.concatenate(seg_lens).astype(np.int32) if seg_lens else np.zeros(0, np.int32)
    S = len(seg_len)
    traj_seg_off = np.zeros(len(traj_nseg) + 1, dtype=np.int32)
    traj_seg_off[1:] = np.cumsum(traj_nseg)
    seg_pos = np.concatenate([np.arange(n) for n in traj_nseg]) if traj_nseg else np.zeros(0, int)
    is_act = (seg_pos % 2 == 0).astype(np.uint8)
    T = int(seg_len.sum(dtype=np.int64))
    rng = np.random.default_rng([SEED0 if seed is None else seed, 1 << 30, int(group_ids[0]) if len(group_ids) else 0])
    # pool in arrival order: turn-major (segment position), then trajectory
    order = np.lexsort((np.arange(S), seg_pos)) if arrival_order else np.arange(S)
    src = np.zeros(S, dtype=np.int64)
    src[order] = np.concatenate([[0], np.cumsum(seg_len[order])[:-1]]) if S else src
    pool = rng.integers(0, cfg.vocab, T, dtype=np.int32)
    table = SegmentTable(pool, src.astype(np.int32), seg_len, is_act, traj_seg_off)
    logp_old = (-rng.exponential(1.0, T)).astype(np.float32)
    logp_ref = (logp_old + rng.normal(0.0, 0.05, T)).astype(np.float32)
    G = cfg.n
    group_off = np.arange(0, len(group_ids) * G + 1, G, dtype=np.int32)
    return Workload(cfg, table, group_off, np.concatenate(rewards) if rewards else np.zeros(0),
                    logp_old, logp_ref, group_ids)
