"""Batched trajectory packing (K1) — host segment table -> device varlen batch.

The host side only lays the ragged segments out as a flat segment table
(the natural shape of asynchronously collected turns: each segment's ids sit
anywhere in one token pool); the GPU packer does the scans and the scatter
(csrc/pack.cu).  Reference semantics: trajectory.flatten / action_mask
(trajectory.py:154-167) and the per-token zip of rl.loss.token_records
(loss.py:76-100).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from .trajectory import ACTION, OBSERVATION, Trajectory


@dataclass
class SegmentTable:
    """Host SoA description of a batch of trajectories."""

    token_pool: np.ndarray     # int32 [P]  ids of every segment, any order
    seg_src_off: np.ndarray    # int32 [S]  start of segment s in token_pool
    seg_len: np.ndarray        # int32 [S]
    seg_is_action: np.ndarray  # uint8 [S]
    traj_seg_off: np.ndarray   # int32 [B+1]

    @property
    def n_traj(self) -> int:
        return len(self.traj_seg_off) - 1

    @property
    def n_seg(self) -> int:
        return len(self.seg_len)

    @property
    def n_tokens(self) -> int:
        return int(self.seg_len.sum(dtype=np.int64))

    @property
    def n_act(self) -> int:
        return int(self.seg_len[self.seg_is_action.astype(bool)].sum(dtype=np.int64))

    def n_act_kept(self, drop=None) -> int:
        """Action tokens left after dropping trajectories (drop: [B] bool)."""
        if drop is None:
            return self.n_act
        keep = ~np.repeat(np.asarray(drop, dtype=bool), np.diff(self.traj_seg_off))
        return int(self.seg_len[self.seg_is_action.astype(bool) & keep].sum(dtype=np.int64))

    def traj_lengths(self) -> np.ndarray:
        c = np.concatenate([[0], np.cumsum(self.seg_len, dtype=np.int64)])
        return c[self.traj_seg_off[1:]] - c[self.traj_seg_off[:-1]]

    def validate(self, vocab: int | None = None) -> None:
        S = self.n_seg
        if not (len(self.seg_src_off) == len(self.seg_is_action) == S):
            raise ValueError("segment table columns disagree in length")
        if self.traj_seg_off[0] != 0 or self.traj_seg_off[-1] != S or np.any(np.diff(self.traj_seg_off) < 0):
            raise ValueError("traj_seg_off must be a monotone offset array ending at n_seg")
        if S and (np.any(self.seg_len < 0) or np.any(self.seg_src_off < 0)
                  or np.any(self.seg_src_off.astype(np.int64) + self.seg_len > len(self.token_pool))):
            raise ValueError("segment outside the token pool")
        if self.n_tokens >= 2 ** 31:
            raise ValueError("batch exceeds 2^31 tokens")
        if vocab is not None and len(self.token_pool) and (
                self.token_pool.min() < 0 or self.token_pool.max() >= vocab):
            raise ValueError("token id outside [0, vocab)")


def segment_table(trajectories: Sequence[Trajectory]) -> SegmentTable:
    """Lay out Trajectory objects as a segment table (pool in segment order)."""
    lens, acts, offs = [], [], [0]
    for tr in trajectories:
        for s in tr.segments:
            if s.origin not in (ACTION, OBSERVATION):
                raise ValueError(f"unknown origin {s.origin!r}")
            lens.append(len(s.tokens))
            acts.append(1 if s.origin == ACTION else 0)
        offs.append(len(lens))
    seg_len = np.asarray(lens, dtype=np.int32)
    total = int(seg_len.sum(dtype=np.int64))
    pool = np.empty(total, dtype=np.int32)
    pos = 0
    for tr in trajectories:
        for s in tr.segments:
            n = len(s.tokens)
            if n:
                pool[pos:pos + n] = s.tokens
            pos += n
    src = np.zeros(len(lens), dtype=np.int32)
    if len(lens) > 1:
        src[1:] = np.cumsum(seg_len[:-1], dtype=np.int64)
    return SegmentTable(pool, src, seg_len, np.asarray(acts, dtype=np.uint8),
                        np.asarray(offs, dtype=np.int32))


@dataclass
class PackedBatch:
    """Device varlen batch (all torch CUDA tensors)."""

    input_ids: "object"      # int32 [T]
    loss_mask: "object"      # uint8 [T]
    position_ids: "object"   # int32 [T]
    traj_of_token: "object"  # int32 [T]
    cu_seqlens: "object"     # int32 [B+1]
    act_off: "object"        # int32 [B+1]
    act_idx: "object"        # int32 [A]
    n_traj: int
    n_tokens: int
    n_act: int


def _dev(a: np.ndarray, device, non_blocking: bool = False):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(a))
    if non_blocking:
        t = t.pin_memory()
    return t.to(device, non_blocking=non_blocking)


def pack_table(table: SegmentTable, device=None, stream=None, validate: bool = True,
               vocab: int | None = None, device_inputs: dict | None = None,
               drop=None) -> PackedBatch:
    """Pack a segment table on the GPU.  `device_inputs` may supply the table
    columns already resident on the device (keys as SegmentTable fields).
    drop ([B] bool, optional): trajectories dropped from the update (error /
    timed-out episodes) — packed with loss_mask 0 and no action
    rows, so they add no LM-head work and no gradient but still count in their
    group (as an all-observation trajectory, loss.py:173-174)."""
    import torch

    L = _lib.lib()
    if validate:
        table.validate(vocab)
        if drop is not None and len(drop) != table.n_traj:
            raise ValueError(f"drop has {len(drop)} entries for {table.n_traj} trajectories")
    device = torch.device(device or "cuda")
    B, S, T = table.n_traj, table.n_seg, table.n_tokens
    A = table.n_act_kept(drop)
    d_drop = None
    if drop is not None:
        d_drop = _dev(np.asarray(drop, dtype=np.uint8), device)
    d = device_inputs or {}
    pool = d.get("token_pool")
    if pool is None:
        pool = _dev(table.token_pool if len(table.token_pool) else np.zeros(1, np.int32), device)
    src = d.get("seg_src_off")
    src = _dev(table.seg_src_off, device) if src is None else src
    ln = d.get("seg_len")
    ln = _dev(table.seg_len, device) if ln is None else ln
    isa = d.get("seg_is_action")
    isa = _dev(table.seg_is_action, device) if isa is None else isa
    tso = d.get("traj_seg_off")
    tso = _dev(table.traj_seg_off, device) if tso is None else tso
    i32 = dict(dtype=torch.int32, device=device)
    out = PackedBatch(
        input_ids=torch.empty(max(T, 1), **i32)[:T],
        loss_mask=torch.empty(max(T, 1), dtype=torch.uint8, device=device)[:T],
        position_ids=torch.empty(max(T, 1), **i32)[:T],
        traj_of_token=torch.empty(max(T, 1), **i32)[:T],
        cu_seqlens=torch.empty(B + 1, **i32),
        act_off=torch.empty(B + 1, **i32),
        act_idx=torch.empty(max(A, 1), **i32)[:A],
        n_traj=B, n_tokens=T, n_act=A,
    )
    ws_bytes = L.tl_pack_workspace_bytes(B, S)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=device)
    _lib.check(L.tl_pack_varlen(
        pool.data_ptr(), src.data_ptr(), ln.data_ptr(), isa.data_ptr(), tso.data_ptr(),
        _lib.ptr(d_drop), B, S, T,
        out.input_ids.data_ptr(), out.loss_mask.data_ptr(), out.position_ids.data_ptr(),
        out.traj_of_token.data_ptr(), out.cu_seqlens.data_ptr(), out.act_off.data_ptr(),
        out.act_idx.data_ptr(), ws.data_ptr(), ws_bytes, _lib.stream_handle(stream)))
    return out


def pack(trajectories: Sequence[Trajectory], device=None, stream=None, drop=None) -> PackedBatch:
    """Pack Trajectory objects (varlen, packed order) on the GPU."""
    return pack_table(segment_table(trajectories), device=device, stream=stream, drop=drop)


def pad(packed: PackedBatch, lmax: int | None = None, pad_id: int = 0, stream=None):
    """Padded [B, lmax] view: (input_ids, loss_mask, position_ids)."""
    import torch

    L = _lib.lib()
    lens = (packed.cu_seqlens[1:] - packed.cu_seqlens[:-1]).cpu()
    longest = int(lens.max()) if packed.n_traj else 0
    if lmax is None:
        lmax = longest
    if longest > lmax:
        raise ValueError(f"trajectory of {longest} tokens exceeds lmax={lmax}")
    dev = packed.cu_seqlens.device
    B = packed.n_traj
    ids = torch.empty((B, lmax), dtype=torch.int32, device=dev)
    mask = torch.empty((B, lmax), dtype=torch.uint8, device=dev)
    pos = torch.empty((B, lmax), dtype=torch.int32, device=dev)
    _lib.check(L.tl_pack_padded(
        packed.input_ids.data_ptr() if packed.n_tokens else packed.cu_seqlens.data_ptr(),
        packed.loss_mask.data_ptr() if packed.n_tokens else packed.cu_seqlens.data_ptr(),
        packed.cu_seqlens.data_ptr(), B, lmax, pad_id, ids.data_ptr(), mask.data_ptr(),
        pos.data_ptr(), _lib.stream_handle(stream)))
    return ids, mask, pos
