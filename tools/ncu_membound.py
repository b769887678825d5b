"""One launch each of the memory-bound kernels at a full config's shape (default
C2), for `ncu --set full` captures of K1 (scan, scatter), K2 (advantages) and
K3 (standalone fp32 loss: streaming units + finalize):

    ncu --set full -k regex:"pack_|group_adv|loss_unit|loss_final" -o out python tools/ncu_membound.py [c2]

Each operation runs once untimed (lazy loads, allocations) and once more as
the captured launch; ncu replays the second one with flushed caches."""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_01055_b200 import grpo, packing  # noqa: E402
from paper_2509_01055_b200.rl.loss import LossConfig  # noqa: E402
from paper_2509_01055_b200.synthetic import CONFIGS, make_workload  # noqa: E402


def main():
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    wl = make_workload(cfg)
    tab = wl.table
    dev = torch.device("cuda")
    dtab = {k: torch.from_numpy(np.ascontiguousarray(getattr(tab, k))).to(dev)
            for k in ("token_pool", "seg_src_off", "seg_len", "seg_is_action", "traj_seg_off")}
    go = wl.group_off
    rw = torch.from_numpy(wl.rewards).to(dev)
    lnew = torch.from_numpy(wl.logp_old + 0.05).to(dev)
    lold = torch.from_numpy(wl.logp_old).to(dev)
    lref = torch.from_numpy(wl.logp_ref).to(dev)
    c = LossConfig(kl_beta=0.04)
    for _ in range(2):
        packed = packing.pack_table(tab, device=dev, validate=False, device_inputs=dtab)
        grpo.grpo_loss(packed, go, rw, lnew, lold, lref, c)
        torch.cuda.synchronize()
    print("T", tab.n_tokens, "T_act", tab.n_act, "segments", tab.n_seg, "trajectories", tab.n_traj)


if __name__ == "__main__":
    main()
