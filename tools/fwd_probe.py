"""Forward LM-head GEMM probe at the C2 chunk shape (37888 action rows,
H 3584, V 152064): event-timed launches of the fused log-prob kernel under
the wave-shape / L2-policy overrides in the environment (TL_FWD_*,
TL_SYNC_FWD).  Run under ncu for DRAM bytes; prints one JSON line."""

import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_01055_b200 import grpo  # noqa: E402


def main():
    C, H, V = int(os.environ.get("PROBE_ROWS", 37888)), 3584, 152064
    iters = int(os.environ.get("PROBE_ITERS", 4))
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    h = torch.randn((C, H), device=dev, dtype=torch.bfloat16, generator=g)
    W = (torch.randn((V, H), device=dev, generator=g) * 0.02).bfloat16()
    y = torch.randint(0, V, (C,), device=dev, dtype=torch.int32, generator=g)
    lp, _, _ = grpo.lmhead_logprobs(h, W, y, chunk_rows=C)
    torch.cuda.synchronize()
    ms = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lp2, _, _ = grpo.lmhead_logprobs(h, W, y, chunk_rows=C)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    env = {k: v for k, v in os.environ.items() if k.startswith("TL_")}
    tf = 2.0 * C * H * V / (min(ms) / 1e3) / 1e12 if ms else 0.0
    print(json.dumps({"env": env, "ms": ms, "tflops_best": tf,
                      "same": bool(torch.equal(lp, lp2))}), flush=True)


if __name__ == "__main__":
    main()
