"""Data parallelism by trajectory group (one process per GPU).

Groups are independent units: advantages need only the group's rewards
(rl/loss.py:103-116) and the batch objective is a sum over groups
(cli.py:317-344), which SPEC.md:496 states is safe to evaluate in parallel.
So whole groups are assigned to ranks (LPT: longest-processing-time-first on
the group's action-token count, the LM head's work), every rank runs the
fused step on its shard with the GLOBAL normalisers (n_groups, action
tokens), and the only collectives are
  N1  all-reduce of the report's additive partials (~12 doubles), and
  N2  all-reduce of dW (the LM-head weight gradient) when it is trained, or
      its reduce-scatter into row shards when W is partitioned.
They run at the C ABI over the library's own NCCL communicator
(`NcclComm`, tl_nccl_* / tl_allreduce_* in include/toolloop_b200.h),
stream-ordered after the step on the caller's stream.  `allreduce_report` /
`allreduce_grad` are the same reductions through torch.distributed, for
process groups NCCL cannot serve (gloo: several ranks on one GPU, CPU tests).
"""

from __future__ import annotations

import heapq

import numpy as np

# indices into the TL_REPORT_LEN report (include/toolloop_b200.h)
_ADDITIVE = (2, 4, 5, 6, 7, 8, 9, 10, 11)


def shard_groups(work: np.ndarray, world: int) -> list[np.ndarray]:
    """LPT assignment of groups (by `work`) to `world` ranks.  Deterministic:
    ties broken by group index; each rank's groups are returned sorted."""
    work = np.asarray(work)
    order = sorted(range(len(work)), key=lambda g: (-work[g], g))
    heap = [(0, r) for r in range(world)]
    out: list[list[int]] = [[] for _ in range(world)]
    for g in order:
        load, r = heapq.heappop(heap)
        out[r].append(g)
        heapq.heappush(heap, (load + int(work[g]), r))
    return [np.asarray(sorted(o), dtype=np.int64) for o in out]


def finalize_report(rep: np.ndarray, agg: int = 0) -> np.ndarray:
    """Recompute the ratio fields (0 objective, 1 clip_fraction, 3 kl) from
    the additive partials after a cross-rank sum."""
    rep = np.array(rep, dtype=np.float64, copy=True)
    masked, groups = rep[2], rep[4]
    if agg == 1:
        rep[0] = rep[11] / masked if masked > 0 else 0.0
    else:
        rep[0] = rep[11] / groups if groups > 0 else 0.0
    rep[1] = rep[8] / masked if masked > 0 else 0.0
    rep[3] = rep[9] / masked if masked > 0 else 0.0
    return rep


def combine_reports(reports, agg: int = 0) -> np.ndarray:
    """Reports of disjoint micro-batches (or ranks) of one step -> the step's
    report: sum the additive partials, recompute the ratios."""
    reps = [np.asarray(r, dtype=np.float64) for r in reports]
    tot = reps[0].copy()
    for r in reps[1:]:
        tot[list(_ADDITIVE)] += r[list(_ADDITIVE)]
    return finalize_report(tot, agg)


def allreduce_report(rep_tensor, agg: int = 0, group=None):
    """N1: sum the additive report fields over ranks (in place) and recompute
    the ratios.  Works for NCCL (device tensor) and gloo (CPU tensor)."""
    import torch
    import torch.distributed as dist

    idx = torch.tensor(_ADDITIVE, device=rep_tensor.device)
    part = rep_tensor.index_select(0, idx)
    dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)
    rep_tensor.index_copy_(0, idx, part)
    masked, groups = rep_tensor[2], rep_tensor[4]
    if agg == 1:
        rep_tensor[0] = torch.where(masked > 0, rep_tensor[11] / masked.clamp_min(1), 0.0)
    else:
        rep_tensor[0] = torch.where(groups > 0, rep_tensor[11] / groups.clamp_min(1), 0.0)
    rep_tensor[1] = torch.where(masked > 0, rep_tensor[8] / masked.clamp_min(1), 0.0)
    rep_tensor[3] = torch.where(masked > 0, rep_tensor[9] / masked.clamp_min(1), 0.0)
    return rep_tensor


def allreduce_grad(t, group=None):
    """N2: sum a gradient tensor over ranks (the LM-head dW)."""
    import torch.distributed as dist

    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


class NcclComm:
    """An NCCL communicator owned by the C library (tl_nccl_comm_init), for
    the step's N1 / N2 collectives at the C ABI.  Build it collectively:
    rank 0 draws the unique id (tl_nccl_unique_id) and the existing
    torch.distributed group broadcasts it (`from_process_group`)."""

    def __init__(self, unique_id: bytes, nranks: int, rank: int):
        import ctypes

        from . import _lib

        L = _lib.lib()
        if not L.tl_nccl_available():
            from .errors import ToolloopError

            raise ToolloopError("NCCL (libnccl.so.2) is not loadable")
        buf = ctypes.create_string_buffer(bytes(unique_id), _lib.TL_NCCL_UNIQUE_ID_BYTES)
        h = ctypes.c_void_p()
        _lib.check(L.tl_nccl_comm_init(ctypes.byref(h), ctypes.addressof(buf), nranks, rank))
        self.handle = h.value
        self.nranks = nranks
        self.rank = rank

    @staticmethod
    def unique_id() -> bytes:
        import ctypes

        from . import _lib

        buf = ctypes.create_string_buffer(_lib.TL_NCCL_UNIQUE_ID_BYTES)
        _lib.check(_lib.lib().tl_nccl_unique_id(ctypes.addressof(buf)))
        return buf.raw

    @classmethod
    def from_process_group(cls, group=None) -> "NcclComm":
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(obj[0], world, rank)

    def size(self) -> int:
        import ctypes

        from . import _lib

        n = ctypes.c_int32()
        _lib.check(_lib.lib().tl_nccl_comm_size(self.handle, ctypes.byref(n)))
        return int(n.value)

    def allreduce_report(self, rep_tensor, agg: int = 0, stream=None):
        """N1 at the C ABI: the float64 [TL_REPORT_LEN] device report of this
        rank -> the global report, in place, stream-ordered."""
        from . import _lib

        _lib.check(_lib.lib().tl_allreduce_report(self.handle, rep_tensor.data_ptr(), agg,
                                                  _lib.stream_handle(stream)))
        return rep_tensor

    def allreduce_scalars(self, x, stream=None):
        from . import _lib

        _lib.check(_lib.lib().tl_allreduce_scalars(self.handle, x.data_ptr(), x.numel(),
                                                   _lib.stream_handle(stream)))
        return x

    def allreduce_grad(self, t, stream=None):
        """N2 at the C ABI: fp32 gradient summed over ranks, in place."""
        from . import _lib

        _lib.check(_lib.lib().tl_allreduce_f32(self.handle, t.data_ptr(), t.numel(),
                                               _lib.stream_handle(stream)))
        return t

    def reduce_scatter_grad(self, t, shard, stream=None):
        """N2 for a row-partitioned W: shard (numel = t.numel() / nranks)
        receives this rank's rows of the summed gradient."""
        from . import _lib

        if shard.numel() * self.nranks != t.numel():
            raise ValueError("shard must hold numel / nranks elements")
        _lib.check(_lib.lib().tl_reduce_scatter_f32(self.handle, t.data_ptr(), shard.data_ptr(),
                                                    shard.numel(), _lib.stream_handle(stream)))
        return shard

    def close(self) -> None:
        if self.handle:
            from . import _lib

            _lib.check(_lib.lib().tl_nccl_comm_destroy(self.handle))
            self.handle = None
