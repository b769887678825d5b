"""Per-kernel device durations (CUPTI via torch.profiler, kernels running
back to back as in production — not serialised like ncu) of the memory-bound
path: K1 pack, K2 advantages, K3 loss.  L2 is flushed before every iteration (256 MB write, then a
256 MB read so the kernels start on a clean L2).  Prints one JSON line: {op: {kernel name: {"us": median,
"n": launches per iteration}, "_span_us": first kernel start -> last end}}.

    python tools/kernel_times.py [c2]
"""

import json
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_01055_b200 import grpo, packing  # noqa: E402
from paper_2509_01055_b200.rl.loss import LossConfig  # noqa: E402
from paper_2509_01055_b200.synthetic import CONFIGS, make_workload  # noqa: E402


def kernel_spans(fn, iters=10):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flush_rd = torch.zeros(64 << 20, dtype=torch.float32, device="cuda")
    fn()
    torch.cuda.synchronize()
    per = defaultdict(list)
    spans = []
    for _ in range(iters):
        flush.fill_(1)       # > L2 (the bench rule) ...
        flush_rd.sum()       # ... then a read, so the dirty lines are written back before timing
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
        if not evs:
            continue
        t0 = min(e.time_range.start for e in evs)
        t1 = max(e.time_range.end for e in evs)
        spans.append(t1 - t0)
        for e in evs:
            per[e.name[:60]].append(e.time_range.end - e.time_range.start)
    out = {k: {"us": float(np.median(v)), "n": len(v) / iters} for k, v in per.items()}
    out["_span_us"] = float(np.median(spans)) if spans else None
    return out


def main():
    cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    wl = make_workload(cfg)
    tab = wl.table
    dev = torch.device("cuda")
    dtab = {k: torch.from_numpy(np.ascontiguousarray(getattr(tab, k))).to(dev)
            for k in ("token_pool", "seg_src_off", "seg_len", "seg_is_action", "traj_seg_off")}
    res = {"config": cfg.name, "T": tab.n_tokens, "T_act": tab.n_act, "B": tab.n_traj,
           "segments": tab.n_seg}
    packed = packing.pack_table(tab, device=dev, device_inputs=dtab)
    res["pack"] = kernel_spans(lambda: packing.pack_table(tab, device=dev, validate=False,
                                                          device_inputs=dtab))
    go = wl.group_off
    rw = torch.from_numpy(wl.rewards).to(dev)
    res["advantages"] = kernel_spans(lambda: grpo.advantages(rw, go, act_off=packed.act_off,
                                                             device=dev))
    lnew = torch.from_numpy(wl.logp_old + 0.05).to(dev)
    lold = torch.from_numpy(wl.logp_old).to(dev)
    lref = torch.from_numpy(wl.logp_ref).to(dev)
    c = LossConfig(kl_beta=0.04)
    res["loss"] = kernel_spans(lambda: grpo.grpo_loss(packed, go, rw, lnew, lold, lref, c))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
