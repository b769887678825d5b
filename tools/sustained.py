"""Steady-state power-capped GEMM throughput: cuBLAS vs our tcgen05 GEMM,
back-to-back for `secs` seconds each, reported per 2-second window with the
SM clock sampled by nvidia-smi (device time via CUDA events)."""

import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_01055_b200 import grpo  # noqa: E402


def run(name, fn, flops, secs):
    f = tempfile.NamedTemporaryFile("w+", delete=False)
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                          "-lms", "100"], stdout=f)
    t_end = time.time() + secs
    windows = []
    while time.time() < t_end:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 0
        e0.record()
        t0 = time.time()
        while time.time() - t0 < 2.0:
            fn()
            n += 1
            if n % 8 == 0:
                torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        windows.append(flops * n / (e0.elapsed_time(e1) / 1e3) / 1e12)
    p.terminate()
    p.wait()
    rows = [l.split(",") for l in Path(f.name).read_text().splitlines() if l.strip()]
    clk = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
    pw = [float(r[1]) for r in rows if len(r) > 1 and r[1].strip().replace(".", "").isdigit()]
    half = len(clk) // 2
    print(f"{name}: TF/s per 2s window {[round(w) for w in windows]}  "
          f"clock median(all/2nd half) {np.median(clk):.0f}/{np.median(clk[half:]):.0f} MHz  "
          f"power median {np.median(pw):.0f} W", flush=True)


def main():
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 20
    M = N = K = 8192
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(N, K, device="cuda").bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    fl = 2.0 * M * N * K
    run("cublas 8192^3", lambda: torch.matmul(A, B.t(), out=out), fl, secs)
    time.sleep(5)
    run("ours   8192^3", lambda: grpo.gemm(A, B, out=out), fl, secs)
    time.sleep(5)
    # dH-shaped: A = dS-like small values, B = W MN-major
    dS = (torch.randn(37888, 38016, device="cuda") * 1e-4).bfloat16()
    W = (torch.randn(38016, 3584, device="cuda") * 0.02).bfloat16()
    o2 = torch.empty(37888, 3584, device="cuda", dtype=torch.bfloat16)
    run("ours   dH-shape", lambda: grpo.gemm(dS, W, b_mn_major=True, out=o2),
        2.0 * 37888 * 38016 * 3584, secs)


if __name__ == "__main__":
    main()
