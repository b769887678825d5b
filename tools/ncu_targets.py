"""Small, deterministic launch sequence for `ncu --set full` captures:
one GRPO step on a ~1-chunk C2-shaped batch (fwd LSE GEMM, dsoftmax, dH and
dW GEMMs, memory-bound pack / advantage / reduction kernels), then an
8192^3 GEMM from our kernel and from cuBLAS for comparison."""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_01055_b200 import grpo, packing  # noqa: E402
from paper_2509_01055_b200.rl.loss import LossConfig  # noqa: E402
from paper_2509_01055_b200.synthetic import CONFIGS, make_workload  # noqa: E402


def main():
    cfg = CONFIGS["c2"]
    wl = make_workload(cfg, group_ids=np.arange(2))
    dev = torch.device("cuda")
    T, H, V = wl.n_tokens, cfg.hidden, cfg.vocab
    hidden = torch.randn((T, H), device=dev, dtype=torch.bfloat16)
    weight = (torch.randn((V, H), device=dev) * 0.02).bfloat16()
    packed = packing.pack_table(wl.table, device=dev)
    lold = torch.from_numpy(wl.logp_old).to(dev)
    lref = torch.from_numpy(wl.logp_ref).to(dev)
    step = grpo.GRPOStep(H, V, LossConfig(kl_beta=0.04))
    for _ in range(2):
        step(packed, wl.group_off, wl.rewards, hidden, weight, lold, lref)
    torch.cuda.synchronize()
    A = torch.randn(8192, 8192, device=dev).bfloat16()
    B = torch.randn(8192, 8192, device=dev).bfloat16()
    for _ in range(2):
        grpo.gemm(A, B)
        torch.matmul(A, B.t())
    torch.cuda.synchronize()
    print("n_act", packed.n_act, "T", T)


if __name__ == "__main__":
    main()
