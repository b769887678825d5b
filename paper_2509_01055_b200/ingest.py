"""Native episode-log ingest (F1): JSONL episode log (+ sidecar) -> SoA
segment table and per-token log-probs, via tl_ingest_* (csrc/ingest.cpp).

Reference: rollout/episodes.read_episodes (episodes.py:132-147),
cli._read_sidecar / _flat_logps (cli.py:233-269), task_id grouping of
cli.loss (cli.py:309-311).  Host-only (no GPU needed); the arrays can be
allocated in pinned memory so the H2D copy of a step overlaps nothing else.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .packing import SegmentTable


@dataclass
class EpisodeBatch:
    table: SegmentTable
    group_off: np.ndarray   # int32 [n_groups+1], groups contiguous in table order
    rewards: np.ndarray     # float64 [B]
    logp_new: np.ndarray    # float64 [T] (packed order)
    logp_old: np.ndarray    # float64 [T]
    logp_ref: np.ndarray | None  # float64 [T], NaN where a row has no reference

    @property
    def n_episodes(self) -> int:
        return len(self.rewards)


def _empty(n, dtype, pinned):
    if pinned:
        import torch

        t = torch.empty(max(n, 1), dtype={np.int32: torch.int32, np.uint8: torch.uint8,
                                          np.float64: torch.float64}[dtype]).pin_memory()
        return t.numpy()[:n]
    return np.empty(max(n, 1), dtype=dtype)[:n]


def ingest(episodes_path, sidecar_path=None, pinned: bool = False) -> EpisodeBatch:
    L = _lib.load(require_device=False)
    h = C.c_void_p()
    _lib.check(L.tl_ingest_open(str(episodes_path).encode(),
                                None if sidecar_path is None else str(sidecar_path).encode(),
                                C.byref(h)))
    try:
        ne, ns, nt, ng = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        hr = C.c_int32()
        _lib.check(L.tl_ingest_sizes(h, C.byref(ne), C.byref(ns), C.byref(nt), C.byref(ng),
                                     C.byref(hr)))
        B, S, T, G = ne.value, ns.value, nt.value, ng.value
        pool = _empty(T, np.int32, pinned)
        src = _empty(S, np.int32, pinned)
        ln = _empty(S, np.int32, pinned)
        isa = _empty(S, np.uint8, pinned)
        tso = _empty(B + 1, np.int32, pinned)
        go = _empty(G + 1, np.int32, pinned)
        rw = _empty(B, np.float64, pinned)
        new = _empty(T, np.float64, pinned)
        old = _empty(T, np.float64, pinned)
        ref = _empty(T, np.float64, pinned) if hr.value else None
        p = lambda a: None if a is None else a.ctypes.data  # noqa: E731
        _lib.check(L.tl_ingest_fill(h, p(pool), p(src), p(ln), p(isa), p(tso), p(go), p(rw),
                                    p(new), p(old), p(ref)))
    finally:
        L.tl_ingest_free(h)
    return EpisodeBatch(SegmentTable(pool, src, ln, isa, tso), go, rw, new, old, ref)
