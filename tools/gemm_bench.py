"""Microbenchmark: tcgen05 GEMM (tl_gemm_bf16) and the fused LM-head forward
vs torch/cuBLAS on the LM-head shapes.  Device time via CUDA events."""

import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_01055_b200 import _lib, grpo  # noqa: E402


def timeit(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    dev = "cuda"
    shapes = [(8192, 8192, 8192, False, False), (37888, 152064 // 4, 3584, False, False),
              (37888, 3584, 152064 // 4, False, True), (152064 // 4, 3584, 37888, True, True)]
    for M, N, K, amn, bmn in shapes:
        A = torch.randn((K, M) if amn else (M, K), device=dev).bfloat16()
        B = torch.randn((K, N) if bmn else (N, K), device=dev).bfloat16()
        out = torch.empty((M, N), device=dev, dtype=torch.float32)
        ms = timeit(lambda: grpo.gemm(A, B, a_mn_major=amn, b_mn_major=bmn, out=out))
        Aop = A.t() if amn else A
        Bop = B if bmn else B.t()
        ms_ref = timeit(lambda: torch.matmul(Aop, Bop))
        fl = 2.0 * M * N * K
        print(f"gemm M={M} N={N} K={K} a_mn={amn} b_mn={bmn}: ours {fl / ms / 1e9:.1f} TF/s "
              f"({ms:.2f} ms)  cuBLAS(bf16 out) {fl / ms_ref / 1e9:.1f} TF/s", flush=True)
    # fused LM-head forward (online LSE epilogue)
    for T, H, V in [(37888, 3584, 152064), (18944, 3584, 152064)]:
        h = torch.randn(T, H, device=dev).bfloat16()
        W = (torch.randn(V, H, device=dev) * 0.02).bfloat16()
        y = torch.randint(0, V, (T,), device=dev, dtype=torch.int32)
        ms = timeit(lambda: grpo.lmhead_logprobs(h, W, y), iters=3)
        print(f"lmhead fwd T={T} H={H} V={V}: {2.0 * T * H * V / ms / 1e9:.1f} TF/s ({ms:.1f} ms)",
              flush=True)
        _lib.profile_enable(True)
        grpo.lmhead_logprobs(h, W, y)
        torch.cuda.synchronize()
        print("  profile:", {k: v for k, v in _lib.profile_read().items() if v[1]}, flush=True)
        _lib.profile_enable(False)
        del h, W


if __name__ == "__main__":
    main()
