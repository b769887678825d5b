"""GEMM stall accounting at the C2 chunk shape (profiling build only):

    TL_GEMM_STATS=1 python -c "from paper_2509_01055_b200 import _build; _build.build(force=True)"
    python tools/gemm_stats.py

Runs one ~1-chunk GRPO step and reports, per GEMM kind (fwd / dH / dW), the
share of the MMA issuer's time spent waiting for operand data (full
barrier) and for a free TMEM accumulator (epilogue behind), the producer's
lockstep and ring-full waits, and the epilogue's busy / idle split."""

import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_01055_b200 import _lib, grpo, packing  # noqa: E402
from paper_2509_01055_b200.rl.loss import LossConfig  # noqa: E402
from paper_2509_01055_b200.synthetic import CONFIGS, make_workload  # noqa: E402

SLOTS = ["prod_sync", "prod_empty", "mma_full", "mma_tempty", "mma_total", "epi_tfull",
         "epi_tile", "epi_end"]


def main():
    L = _lib.lib()
    cfg = CONFIGS["c2"]
    wl = make_workload(cfg, group_ids=np.arange(2))
    dev = torch.device("cuda")
    T, H, V = wl.n_tokens, cfg.hidden, cfg.vocab
    hidden = torch.randn((T, H), device=dev, dtype=torch.bfloat16)
    weight = (torch.randn((V, H), device=dev) * 0.02).bfloat16()
    packed = packing.pack_table(wl.table, device=dev)
    lold = torch.from_numpy(wl.logp_old).to(dev)
    lref = torch.from_numpy(wl.logp_ref).to(dev)
    step = grpo.GRPOStep(H, V, LossConfig(kl_beta=0.04), chunk_rows=(packed.n_act + 255) // 256 * 256)
    step(packed, wl.group_off, wl.rewards, hidden, weight, lold, lref)  # warm-up
    torch.cuda.synchronize()
    buf = torch.zeros(_lib.N_PROF * 160 * 8, dtype=torch.int64, device=dev)
    fn = L.tl_debug_gemm_stats
    fn.argtypes = [ctypes.c_void_p]
    if fn(buf.data_ptr()) != 0:
        raise SystemExit("library not built with TL_GEMM_STATS=1")
    step(packed, wl.group_off, wl.rewards, hidden, weight, lold, lref)
    torch.cuda.synchronize()
    fn(None)
    st = buf.view(_lib.N_PROF, 160, 8).cpu().numpy().astype(np.float64)
    names = {L.tl_profile_category(i).decode(): i for i in range(_lib.N_PROF)}
    for k in ("gemm_fwd", "gemm_dh", "gemm_dw"):
        a = st[names[k]]
        live = a[:, 4] > 0  # MMA issuers (leader CTAs)
        tot = a[live, 4].mean()
        print(f"{k}: MMA loop {tot / 1e6:.2f} Mcyc/leader | "
              f"wait data {a[live, 2].mean() / tot:.1%}  wait acc {a[live, 3].mean() / tot:.1%} | "
              f"producer lockstep {a[:, 0].mean() / tot:.1%} ring-full {a[:, 1].mean() / tot:.1%} | "
              f"epilogue tile {a[:, 6].mean() / tot:.1%} idle {a[:, 5].mean() / tot:.1%} "
              f"end-unit {a[:, 7].mean() / tot:.1%}")


if __name__ == "__main__":
    main()
