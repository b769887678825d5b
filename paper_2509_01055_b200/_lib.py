"""ctypes binding of the C-ABI library (include/toolloop_b200.h).

The library is the product: every operator in this package calls it.  If it
is missing (not built) or no CUDA device is present, `lib()` raises
ExtensionMissing — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import ExtensionMissing, GroupTooSmall, MaskMismatch, ToolloopError

LIB_PATH = Path(__file__).resolve().parent / "libtoolloop_b200.so"
# A/B builds of the same library (tools/*_ab.py) are selected by path
if os.environ.get("TOOLLOOP_B200_LIB"):
    LIB_PATH = Path(os.environ["TOOLLOOP_B200_LIB"])

TL_ABI_VERSION = 4  # include/toolloop_b200.h
TL_OK = 0
TL_ERR_INVALID_ARG = 1
TL_ERR_MASK_MISMATCH = 2
TL_ERR_GROUP_TOO_SMALL = 3
TL_ERR_CUDA = 4
TL_ERR_UNSUPPORTED = 5
TL_ERR_WORKSPACE = 6
TL_ERR_EPISODE_LOG = 7
TL_ERR_COMM = 8
TL_NCCL_UNIQUE_ID_BYTES = 128
TL_GROUP_OUT_LEN = 8
TL_REPORT_LEN = 12

# Every symbol include/toolloop_b200.h declares (checked by the CPU tests).
EXPORTS = [
    "tl_last_error", "tl_abi_version", "tl_launch_count",
    "tl_profile_enable", "tl_profile_read", "tl_profile_category",
    "tl_pack_workspace_bytes", "tl_pack_varlen", "tl_pack_padded",
    "tl_group_advantages", "tl_group_rewards_advantages",
    "tl_loss_f64_workspace_bytes", "tl_loss_f64", "tl_report_f64", "tl_token_ratio_f64",
    "tl_loss_f32_workspace_bytes", "tl_loss_f32",
    "tl_lmhead_workspace_bytes", "tl_lmhead_logprobs_workspace_bytes",
    "tl_lmhead_step_workspace_bytes", "tl_lmhead_logprobs",
    "tl_grpo_lmhead_step", "tl_grpo_lmhead_step_overlap",
    "tl_gemm_bf16",
    "tl_ingest_open", "tl_ingest_sizes", "tl_ingest_fill", "tl_ingest_free",
    "tl_tokenizer_create", "tl_tokenizer_free", "tl_tokenizer_vocab_size",
    "tl_tokenize_segments", "tl_tokenizer_decode",
    "tl_nccl_available", "tl_nccl_version", "tl_nccl_unique_id", "tl_nccl_comm_init",
    "tl_nccl_comm_destroy", "tl_nccl_comm_size", "tl_allreduce_scalars", "tl_allreduce_report",
    "tl_allreduce_f32", "tl_reduce_scatter_f32",
]


class LossConfigC(C.Structure):
    _fields_ = [
        ("eps_low", C.c_double), ("eps_high", C.c_double), ("kl_beta", C.c_double),
        ("entropy_coef", C.c_double), ("use_mask", C.c_int32), ("has_ref", C.c_int32),
        ("objective", C.c_int32), ("agg", C.c_int32), ("entropy_norm", C.c_double),
    ]


class StepOverlapC(C.Structure):
    _fields_ = [("dw_ready_event", C.c_void_p), ("reserve_sms", C.c_int32)]


class RewardParamsC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_int32), ("h", C.c_double),
                ("alpha", C.c_double), ("beta", C.c_double)]


_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_SZ = C.c_size_t
_D = C.c_double

_SIGS = {
    "tl_last_error": (C.c_char_p, []),
    "tl_abi_version": (C.c_int, []),
    "tl_launch_count": (_I64, []),
    "tl_profile_enable": (C.c_int, [_I32]),
    "tl_profile_read": (C.c_int, [_P, _P, _I32]),
    "tl_profile_category": (C.c_char_p, [_I32]),
    "tl_pack_workspace_bytes": (_SZ, [_I32, _I32]),
    "tl_pack_varlen": (C.c_int, [_P, _P, _P, _P, _P, _P, _I32, _I32, _I64, _P, _P, _P, _P, _P, _P, _P,
                                 _P, _SZ, _P]),
    "tl_pack_padded": (C.c_int, [_P, _P, _P, _I32, _I32, _I32, _P, _P, _P, _P]),
    "tl_group_advantages": (C.c_int, [_P, _P, _I32, _I32, _D, _P, _I32, _D, _D, _P, _P, _P, _P,
                                      _P]),
    "tl_group_rewards_advantages": (C.c_int, [C.POINTER(RewardParamsC), _P, _P, _P, _P, _P, _P,
                                              _I32, _I32, _D, _P, _P, _P, _P, _P, _P]),
    "tl_loss_f64_workspace_bytes": (_SZ, [_I64]),
    "tl_loss_f64": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _I32, _I32, _I64,
                              C.POINTER(LossConfigC), _P, _P, _P, _SZ, _P]),
    "tl_report_f64": (C.c_int, [_P, _I32, _I32, _P, _P]),
    "tl_token_ratio_f64": (C.c_int, [_P, _P, _I64, _P, _P]),
    "tl_loss_f32_workspace_bytes": (_SZ, [_I64, _I32, _I32]),
    "tl_loss_f32": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I32, _I32, _I64,
                              C.POINTER(LossConfigC), _P, _P, _P, _SZ, _P]),
    "tl_lmhead_workspace_bytes": (_SZ, [_I32, _I32, _I32, _I64, _I32, _I32]),
    "tl_lmhead_logprobs_workspace_bytes": (_SZ, [_I32, _I32, _I32]),
    "tl_lmhead_step_workspace_bytes": (_SZ, [_I32, _I32, _I32, _I64, _I32, _I32, _I32]),
    "tl_lmhead_logprobs": (C.c_int, [_P, _P, _P, _P, _I64, _I32, _I32, _P, _P, _P, _I32, _P, _SZ,
                                     _P]),
    "tl_grpo_lmhead_step": (C.c_int, [_P, _P, _P, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _I64,
                                      _I32, _I32, _I32, _I32, C.POINTER(LossConfigC), _P, _P, _P,
                                      _P, _P, _I32, _I32, _P, _SZ, _P]),
    "tl_grpo_lmhead_step_overlap": (C.c_int, [_P, _P, _P, _P, _P, _I64, _P, _P, _P, _P, _P, _P, _P,
                                              _I64, _I32, _I32, _I32, _I32,
                                              C.POINTER(LossConfigC), _P, _P, _P, _P, _P, _I32,
                                              _I32, _P, _SZ, _P, C.POINTER(StepOverlapC)]),
    "tl_gemm_bf16": (C.c_int, [_P, _I32, _I64, _P, _I32, _I64, _I32, _I32, _I32, _P, _I32, _I64,
                               _I32, _P]),
    "tl_ingest_open": (C.c_int, [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    "tl_ingest_sizes": (C.c_int, [_P, C.POINTER(_I64), C.POINTER(_I64), C.POINTER(_I64),
                                  C.POINTER(_I64), C.POINTER(_I32)]),
    "tl_ingest_fill": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "tl_ingest_free": (None, [_P]),
    "tl_tokenizer_create": (C.c_int, [_P, _P, _I32, C.POINTER(C.c_void_p)]),
    "tl_tokenizer_free": (None, [_P]),
    "tl_tokenizer_vocab_size": (_I32, [_P]),
    "tl_tokenize_segments": (C.c_int, [_P, _P, _P, _I64, _P, _P, _P, _I32]),
    "tl_tokenizer_decode": (C.c_int, [_P, _P, _I64, _P, _I64, C.POINTER(_I64)]),
    "tl_nccl_available": (C.c_int, []),
    "tl_nccl_version": (C.c_int, []),
    "tl_nccl_unique_id": (C.c_int, [_P]),
    "tl_nccl_comm_init": (C.c_int, [C.POINTER(C.c_void_p), _P, _I32, _I32]),
    "tl_nccl_comm_destroy": (C.c_int, [_P]),
    "tl_nccl_comm_size": (C.c_int, [_P, C.POINTER(_I32)]),
    "tl_allreduce_scalars": (C.c_int, [_P, _P, _I32, _P]),
    "tl_allreduce_report": (C.c_int, [_P, _P, _I32, _P]),
    "tl_allreduce_f32": (C.c_int, [_P, _P, _I64, _P]),
    "tl_reduce_scatter_f32": (C.c_int, [_P, _P, _P, _I64, _P]),
}

_lock = threading.Lock()
_lib: C.CDLL | None = None


def load(require_device: bool = True) -> C.CDLL:
    """Load the library (and, by default, insist on a CUDA device)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ExtensionMissing(
                    f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                )
            lib = C.CDLL(str(LIB_PATH))
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.tl_abi_version() != TL_ABI_VERSION:
                raise ExtensionMissing(
                    f"{LIB_PATH} has ABI {lib.tl_abi_version()}, this package needs "
                    f"{TL_ABI_VERSION}: rebuild it (__graft_entry__.build())")
            _lib = lib
    if require_device:
        import torch

        if not torch.cuda.is_available():
            raise ExtensionMissing("toolloop-b200 operators need a CUDA (sm_100a) device")
    return _lib


def lib() -> C.CDLL:
    return load(True)


def check(status: int) -> None:
    if status == TL_OK:
        return
    msg = (_lib.tl_last_error() or b"").decode(errors="replace")
    if status == TL_ERR_MASK_MISMATCH:
        raise MaskMismatch(msg)
    if status == TL_ERR_GROUP_TOO_SMALL:
        raise GroupTooSmall(msg)
    if status == TL_ERR_INVALID_ARG:
        raise ValueError(msg)
    if status == TL_ERR_EPISODE_LOG:
        from .errors import EpisodeLogError

        raise EpisodeLogError(msg)
    raise ToolloopError(f"toolloop-b200 status {status}: {msg}")


def ptr(t) -> int | None:
    """Device/host pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def launch_count() -> int:
    return int(load(False).tl_launch_count())


N_PROF = 13
LMHEAD_STORE_LOGITS = 0
LMHEAD_RECOMPUTE = 1
LMHEAD_STORE_LOGITS_PIPELINED = 2
LMHEAD_ACCUMULATE_DW = 0x100
LMHEAD_NO_SPLIT_TAIL = 0x200
LMHEAD_NO_FACTORED = 0x400
LMHEAD_DEBUG_FIXUP = 0x800


def profile_enable(on: bool = True) -> None:
    check(load(False).tl_profile_enable(1 if on else 0))


def profile_read() -> dict:
    """{category: (ms, launches)} for the kernels recorded since enable."""
    import numpy as np

    L = load(False)
    ms = np.zeros(N_PROF, dtype=np.float64)
    cnt = np.zeros(N_PROF, dtype=np.int64)
    check(L.tl_profile_read(ms.ctypes.data, cnt.ctypes.data, N_PROF))
    return {L.tl_profile_category(i).decode(): (float(ms[i]), int(cnt[i])) for i in range(N_PROF)}
