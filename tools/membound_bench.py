"""Achieved HBM bandwidth of the memory-bound kernels at the C2 shape
(north star: "achieved HBM GB/s for the packer, advantage and loss kernels
against ~8 TB/s").  Each operation is timed alone, L2 flushed (256 MB
write) before every timed launch, two ways: CUDA events around the public
Python call (includes host work and allocations) and, for the rows marked
"device", the library's own events around its kernel launches;
GB/s = algorithmic bytes / median time.  Prints one JSON line."""

import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_01055_b200 import _lib, grpo, packing  # noqa: E402
from paper_2509_01055_b200.rl.loss import LossConfig  # noqa: E402
from paper_2509_01055_b200.synthetic import CONFIGS, make_workload  # noqa: E402

PEAK = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
    if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 6650.0
FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
FLUSH_RD = torch.zeros(64 << 20, dtype=torch.float32, device="cuda")  # 256 MB


def flush_l2():
    """Write a buffer larger than the 126 MB L2 (the bench rule), then read
    another one: the write's dirty lines are written back during the read,
    so the timed kernels start on a clean L2 (with the write alone they pay
    up to ~126 MB of write-backs of the flush buffer, as much DRAM traffic
    as K3 itself).  MEMBOUND_FLUSH=write keeps the write-only flush."""
    import os

    FLUSH.fill_(1)
    if os.environ.get("MEMBOUND_FLUSH", "write+read") != "write":
        FLUSH_RD.sum()


def timed(fn, iters=None):
    import os

    iters = int(os.environ.get("MEMBOUND_ITERS", "10")) if iters is None else iters
    ts = []
    for _ in range(iters + 2):
        flush_l2()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts[2:]))


def device_ms(fn, cat, iters=5):
    """Median device time of the kernels `fn` launches in profile category
    `cat` (CUDA events recorded by the library around its own launches);
    L2 flushed before each.  A ~1 ms spin kernel runs first so the host has
    queued every launch before the GPU reaches them: the kernels run back to
    back and the events measure device time, not host submission latency."""
    ts = []
    for _ in range(iters):
        flush_l2()
        torch.cuda.synchronize()
        torch.cuda._sleep(2_000_000)
        _lib.profile_enable(True)
        fn()
        torch.cuda.synchronize()
        ts.append(_lib.profile_read()[cat][0])
        _lib.profile_enable(False)
    return float(np.median(ts))


def main():
    cfg = CONFIGS["c2"]
    wl = make_workload(cfg)
    tab = wl.table
    dev = torch.device("cuda")
    dtab = {k: torch.from_numpy(np.ascontiguousarray(getattr(tab, k))).to(dev)
            for k in ("token_pool", "seg_src_off", "seg_len", "seg_is_action", "traj_seg_off")}
    T, A, B, S = tab.n_tokens, tab.n_act, tab.n_traj, tab.n_seg
    out = {"config": cfg.desc, "T": T, "T_act": A, "B": B, "segments": S, "peak_hbm_gbs": PEAK}
    res = {}

    packed = packing.pack_table(tab, device=dev, device_inputs=dtab)
    ms = timed(lambda: packing.pack_table(tab, device=dev, validate=False, device_inputs=dtab))
    # read ids 4 + write ids 4, mask 1, positions 4, traj 4 per token; act_idx 4 per action token
    by = 21 * T + 4 * A + 13 * S + 8 * (B + 1)
    res["pack_varlen (K1)"] = (ms, by)
    res["pack_varlen (K1) device"] = (device_ms(
        lambda: packing.pack_table(tab, device=dev, validate=False, device_inputs=dtab), "pack"), by)

    lmax = int((packed.cu_seqlens[1:] - packed.cu_seqlens[:-1]).max())
    ms = timed(lambda: packing.pad(packed, lmax=lmax))
    res["pack_padded (K1)"] = (ms, 5 * T + 9 * B * lmax)

    go = wl.group_off
    rw = torch.from_numpy(wl.rewards).to(dev)
    ms = timed(lambda: grpo.advantages(rw, go, act_off=packed.act_off, device=dev))
    res["group_advantages (K2)"] = (ms, 8 * B + 8 * B + 4 * B + 4 * B + 4 * (B + 1))

    lnew = torch.from_numpy(wl.logp_old + 0.05).to(dev)
    lold = torch.from_numpy(wl.logp_old).to(dev)
    lref = torch.from_numpy(wl.logp_ref).to(dev)
    c = LossConfig(kl_beta=0.04)
    ms = timed(lambda: grpo.grpo_loss(packed, go, rw, lnew, lold, lref, c))
    # mask 1 B/token, logp_new/old/ref 12 B per action token, grad 4 B/token
    res["grpo_loss fp32 (K3, incl. K2 + report)"] = (ms, 5 * T + 12 * A)
    res["grpo_loss fp32 (K3 + group/report reductions) device"] = (device_ms(
        lambda: grpo.grpo_loss(packed, go, rw, lnew, lold, lref, c), "loss"), 5 * T + 12 * A)

    # dsoftmax on one chunk and the row gather, via the fused step's profile
    H, V = cfg.hidden, cfg.vocab
    n = 37888
    idx = packed.act_idx[:n].contiguous()
    hidden = torch.randn((T, H), device=dev, dtype=torch.bfloat16)
    weight = (torch.randn((V, H), device=dev) * 0.02).bfloat16()
    sub = packing.PackedBatch(packed.input_ids, packed.loss_mask, packed.position_ids,
                              packed.traj_of_token, packed.cu_seqlens, packed.act_off, idx,
                              packed.n_traj, packed.n_tokens, n)
    def chunk_prof(factored):
        step = grpo.GRPOStep(H, V, c, chunk_rows=n, factored=factored)
        step(sub, go, rw, hidden, weight, lold, lref)
        torch.cuda.synchronize()
        _lib.profile_enable(True)
        step(sub, go, rw, hidden, weight, lold, lref)
        torch.cuda.synchronize()
        prof = _lib.profile_read()
        _lib.profile_enable(False)
        return prof

    prof = chunk_prof(False)  # fp16-logit store: the dS pass (kept for the entropy bonus)
    res["dsoftmax (K5, one chunk, fp16 store)"] = (prof["dsoftmax"][0], 4 * n * V)
    res["gather action rows (one chunk, fp16 store)"] = (prof["gather"][0], 4 * n * H + 8 * n)
    prof = chunk_prof(True)  # factored store (default without the entropy bonus)
    # gather + anchor: hidden rows and W[y] rows read, h_c written, ids / anchors
    res["gather + anchor (one chunk, factored)"] = (prof["gather"][0], 6 * n * H + 16 * n)
    # fixup (empty list) + h_c *= alpha in place
    res["rescale (one chunk, factored)"] = (prof["rescale"][0], 4 * n * H + 4 * n)
    for k, (ms, by) in res.items():
        gbs = by / (ms / 1e3) / 1e9
        out[k] = {"ms": round(ms, 4), "bytes": int(by), "GB_s": round(gbs, 1),
                  "frac_of_hbm": round(gbs / PEAK, 3)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
