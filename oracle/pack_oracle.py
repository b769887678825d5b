"""Restatement of the packed batch layouts (TEST INFRASTRUCTURE ONLY).

ids and mask follow flatten/action_mask (trajectory.py:154-167, pinned by the
reference's own tests).  The remaining arrays have no reference
implementation ("parity unpinned"); their definitions are the build's
contract, stated once here and in DESIGN.md:

  cu_seqlens[b]     exclusive prefix sum of trajectory lengths, cu[B] = T
  position_ids[t]   t - cu_seqlens[traj(t)]         (per-trajectory iota)
  traj_of_token[t]  index b of the trajectory holding packed token t
  act_off[b]        exclusive prefix sum of per-trajectory action counts
  act_idx[k]        packed position of the k-th action token (packed order)
  padded [B, Lmax]  row b = trajectory b left-aligned; pad slots get
                    pad_id / mask 0 / position 0
  drop[b]           (optional) trajectory b keeps its tokens but every mask
                    bit is 0 — error / timed-out episodes whose gradients the
                    paper masks; not in the reference code
"""

from __future__ import annotations

import numpy as np

from .grpo_oracle import action_mask, flatten


def pack_varlen(trajectories, drop=None):
    """trajectories: list of segment lists [(origin, tokens), ...]."""
    ids, mask, pos, tot, cu, act_off, act_idx = [], [], [], [], [0], [0], []
    for b, segs in enumerate(trajectories):
        f = flatten(segs)
        m = action_mask(segs)
        if drop is not None and drop[b]:
            m = [0] * len(m)
        base = cu[-1]
        for j, (tok, bit) in enumerate(zip(f, m)):
            ids.append(tok)
            mask.append(bit)
            pos.append(j)
            tot.append(b)
            if bit:
                act_idx.append(base + j)
        cu.append(base + len(f))
        act_off.append(act_off[-1] + sum(m))
    i32 = np.int32
    return {
        "input_ids": np.asarray(ids, dtype=i32),
        "loss_mask": np.asarray(mask, dtype=np.uint8),
        "position_ids": np.asarray(pos, dtype=i32),
        "cu_seqlens": np.asarray(cu, dtype=i32),
        "traj_of_token": np.asarray(tot, dtype=i32),
        "act_off": np.asarray(act_off, dtype=i32),
        "act_idx": np.asarray(act_idx, dtype=i32),
    }


def pack_padded(trajectories, pad_id: int = 0, lmax: int | None = None):
    lens = [len(flatten(s)) for s in trajectories]
    L = max(lens, default=0) if lmax is None else lmax
    B = len(trajectories)
    ids = np.full((B, L), pad_id, dtype=np.int32)
    mask = np.zeros((B, L), dtype=np.uint8)
    pos = np.zeros((B, L), dtype=np.int32)
    for b, segs in enumerate(trajectories):
        f = flatten(segs)
        m = action_mask(segs)
        n = len(f)
        ids[b, :n] = f
        mask[b, :n] = m
        pos[b, :n] = np.arange(n, dtype=np.int32)
    return {"input_ids": ids, "loss_mask": mask, "position_ids": pos}
