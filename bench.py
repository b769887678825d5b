"""Benchmark: masked GRPO-step tokens/sec (pack + advantage + LM-head log-prob
+ surrogate loss + LM-head backward) on B200, vs the reference's CPU path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5]
                    [--impl ours|reference] [--mode store|pipelined|recompute]

One step = the whole trajectory-to-loss hot path over one synthetic batch of
BASELINE.json's config (default C2, Qwen2.5-7B shape: 256 prompts x 8
rollouts, <= 4 tool turns, seq 4k, H 3584, V 152064, bf16):
  K1 pack (segment table -> varlen batch) -> K2 group advantages ->
  K4 fused LM-head logp/entropy + GRPO surrogate epilogue (fp16 logits kept)
  -> K5 backward (dS pass, dH = dS W, dW += dS^T H) -> deterministic
  reductions [-> N1 report all-reduce, N2 dW all-reduce when N > 1].
Configs whose activations exceed one GPU's HBM (C3, C4) run each step as
micro-batches of whole groups with the step's global normalisers (dW
accumulated, reports combined); `config.micro_batches` says how many.
`value` = packed tokens (action + observation) per second over the whole job,
inputs resident in HBM; `e2e` = the same through the public API with the
step's host inputs (segment table, logp_old/logp_ref, rewards) copied from
pinned host memory and the report read back every step (hidden states and
the LM-head weight are device-resident model tensors).  Multi-GPU: weak
scaling, each rank owns a C2-sized shard of whole groups (LPT).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "masked GRPO-step tokens/sec (pack+adv+logprob+loss) at 1/2/4/8 B200 vs CPU ref"
UNIT = "tokens/s"
# ncu DRAM bytes of one C2 chunk (tools/profile_summary.py) for roofline.traffic
TRAFFIC_JSON = "r1f_gemm_traffic.json"


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("bf16_tflops_sustained", 1437.7), d.get("bf16_tflops", 1712.4), \
            d.get("hbm_gbs", 6452.5), "measured"
    return 1400.0, 1590.0, 6650.0, "fallback"


# --------------------------------------------------------------- clocks --
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.f = None

    def __enter__(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.f is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        self.f.flush()
        rows = [l.split(",") for l in Path(self.f.name).read_text().splitlines() if l.strip()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except ValueError:
                continue
            for n, v in zip(names, r[2:6]):
                if "Active" in v and "Not" not in v:
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(mx)) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------- CPU baseline --
def cpu_baseline(cfg, wl, target_s: float = 12.0, threads: int | None = None):
    """The reference's CPU path on a bounded sample of the same workload:
    the oracle port of token_records -> group_advantages ->
    grpo_multi_turn_loss (pure Python, as toolloop runs it) on one whole group,
    plus the fp32 numpy LM-head restatement (fwd + bwd, multithreaded BLAS) on
    a sample of action tokens; tokens/s extrapolated per token."""
    from oracle import grpo_oracle as O
    from oracle import lmhead_oracle as LH

    tab = wl.table
    # --- loss path on group 0
    b0, b1 = int(wl.group_off[0]), int(wl.group_off[1])
    segs_all = []
    pos_pool = tab.token_pool
    cu = 0
    starts = []
    for b in range(b0, b1):
        segs = []
        for s in range(tab.traj_seg_off[b], tab.traj_seg_off[b + 1]):
            o = int(tab.seg_src_off[s])
            n = int(tab.seg_len[s])
            segs.append(("action" if tab.seg_is_action[s] else "observation", pos_pool[o:o + n].tolist()))
        segs_all.append(segs)
    lens = [sum(len(t) for _, t in s) for s in segs_all]
    tg = sum(lens)
    new = (wl.logp_old[:tg] + 0.05).astype(np.float64)  # logp_new stand-in (LM head timed separately)
    old = wl.logp_old[:tg].astype(np.float64)
    ref = wl.logp_ref[:tg].astype(np.float64)
    t0 = time.perf_counter()
    recs, pos = [], 0
    for s, n in zip(segs_all, lens):
        recs.append(O.token_records(s, new[pos:pos + n].tolist(), old[pos:pos + n].tolist(),
                                    ref[pos:pos + n].tolist()))
        pos += n
    adv = O.group_advantages(wl.rewards[b0:b1].tolist())
    O.multi_turn(recs, adv, 0.2, 0.0)
    t_loss = time.perf_counter() - t0
    # --- LM head on a sample of action tokens
    H, V = cfg.hidden, cfg.vocab
    rng = np.random.default_rng(7)
    W = LH.to_bf16_f32((rng.standard_normal((V, H), dtype=np.float32) * 0.02))
    y = rng.integers(0, V, 4096)

    def run(n):
        h = LH.to_bf16_f32(rng.standard_normal((n, H), dtype=np.float32))
        t = time.perf_counter()
        LH.lmhead_forward(h, W, y[:n], chunk=128)
        LH.lmhead_backward(h, W, y[:n], np.full(n, -1e-3), None, chunk=128)
        return time.perf_counter() - t

    # time(n) = fixed (dW alloc/accumulate over V x H) + n * per_token: take the
    # slope between two sample sizes so the per-step fixed cost (amortised over
    # a whole batch in a real step) does not inflate the per-token figure.
    n1 = 64
    run(n1)  # warm BLAS / page in W
    t1 = run(n1)
    n = int(min(4096, max(4 * n1, n1 * target_s / max(t1, 1e-3))))
    dt = run(n)
    per_act = max((dt - t1) / (n - n1), dt / n * 0.5)
    f_act = wl.n_act / max(wl.n_tokens, 1)
    per_tok = t_loss / tg + f_act * per_act
    try:
        from threadpoolctl import threadpool_info

        blas_threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        blas_threads = os.cpu_count() or 1
    return {
        "value": 1.0 / per_tok,
        "unit": UNIT,
        "cores": int(blas_threads),
        "kind": "port",
        "sample": (f"oracle/ port: pure-Python token_records+group_advantages+multi_turn on group 0 "
                   f"({tg} tokens, {t_loss:.3f}s, 1 core) + numpy fp32 LM-head fwd+bwd on {n} action "
                   f"tokens at H={H} V={V} ({dt:.2f}s, {blas_threads} BLAS threads); "
                   f"per-token cost extrapolated with f_act={f_act:.3f}"),
        "host_cpu": _cpu_model(),
    }


def _cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip() + f" x{os.cpu_count()}"
    except Exception:
        pass
    return f"{os.cpu_count()} cpus"


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2509_01055_b200.synthetic import make_workload

    wl = make_workload(cfg, group_ids=np.arange(min(cfg.prompts, 2)))
    for _ in range(args.warmup):
        cpu_baseline(cfg, wl, target_s=3.0)
    vals, last = [], None
    t0 = time.perf_counter()
    for _ in range(args.steps):
        last = cpu_baseline(cfg, wl, target_s=args.ref_seconds)
        vals.append(last["value"])
    wall = time.perf_counter() - t0
    v = float(np.median(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall / max(args.steps, 1) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64 (loss path) / f32 (LM head)",
        "data": "synthetic", "config": {"workload": cfg.desc, "name": cfg.name},
        "cpu_baseline": {k: last[k] for k in ("kind", "cores", "sample")} | {"value": v, "unit": UNIT},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- GPU path --
def micro_batches(cfg, groups, max_tokens: int):
    """Split a rank's groups (in order) into contiguous micro-batches of at
    most max_tokens packed tokens (whole groups; at least one group each)."""
    from paper_2509_01055_b200.synthetic import group_tokens

    toks = group_tokens(cfg, groups)
    out, cur, n = [], [], 0
    for gid, t in zip(groups, toks):
        if cur and n + t > max_tokens:
            out.append(np.asarray(cur, dtype=np.int64))
            cur, n = [], 0
        cur.append(int(gid))
        n += int(t)
    if cur:
        out.append(np.asarray(cur, dtype=np.int64))
    return out


def combine_reports_device(reps, agg: int):
    """parallel.combine_reports on device tensors (no host sync)."""
    import torch

    from paper_2509_01055_b200 import parallel

    idx = torch.tensor(parallel._ADDITIVE, device=reps[0].device)
    tot = reps[0].clone()
    tot.index_copy_(0, idx, torch.stack([r.index_select(0, idx) for r in reps]).sum(0))
    masked, groups = tot[2], tot[4]
    if agg == 1:
        tot[0] = torch.where(masked > 0, tot[11] / masked.clamp_min(1), 0.0)
    else:
        tot[0] = torch.where(groups > 0, tot[11] / groups.clamp_min(1), 0.0)
    tot[1] = torch.where(masked > 0, tot[8] / masked.clamp_min(1), 0.0)
    tot[3] = torch.where(masked > 0, tot[9] / masked.clamp_min(1), 0.0)
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=8.0)
    ap.add_argument("--chunk-rows", type=int, default=None)
    ap.add_argument("--max-mb-tokens", type=int, default=7_000_000,
                    help="largest micro-batch (packed tokens) a rank holds at once")
    ap.add_argument("--mode", default="store", choices=["store", "pipelined", "recompute"],
                    help="LM-head backward schedule (TL_LMHEAD_* in include/toolloop_b200.h); "
                         "store is fastest on a power-capped B200 (DESIGN.md §3)")
    args = ap.parse_args()

    from paper_2509_01055_b200.synthetic import CONFIGS

    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import torch
    import torch.distributed as dist

    from paper_2509_01055_b200 import _lib, grpo, packing, parallel
    from paper_2509_01055_b200.rl.loss import AGG_TOKEN_MEAN, LossConfig
    from paper_2509_01055_b200.synthetic import group_act_tokens, make_workload

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TL_BENCH_ONE_DEVICE=1 + TL_BENCH_BACKEND=gloo: every rank on cuda:0 over
    # gloo — exercises the multi-rank path (sharding, N1/N2 all-reduces,
    # max-over-ranks timing) on a one-GPU box with a small --config.
    if os.environ.get("TL_BENCH_ONE_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("TL_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    # global batch = world x config (weak scaling); whole groups per rank by LPT
    n_groups_global = cfg.prompts * world
    work = group_act_tokens(cfg, np.arange(n_groups_global))
    shards = parallel.shard_groups(work, world)
    agg = 1 if cfg.loss_agg == AGG_TOKEN_MEAN else 0
    loss_cfg = LossConfig(epsilon_clip=0.2, kl_beta=0.04, loss_agg=cfg.loss_agg)
    norm_tokens = float(work.sum())
    H, V = cfg.hidden, cfg.vocab
    # Micro-batches of whole groups when a rank's hidden + dhidden would not
    # fit in HBM next to the LM head (C3-C5): each is one call of the fused
    # step with the step's global normalisers, dW accumulated across them.
    mb_groups = micro_batches(cfg, shards[rank], args.max_mb_tokens)
    wls = [make_workload(cfg, group_ids=gids) for gids in mb_groups]
    T_max = max(w.n_tokens for w in wls)
    T = sum(w.n_tokens for w in wls)
    n_act = sum(w.n_act for w in wls)
    wl = wls[0]

    # device-resident inputs (one hidden buffer sized for the largest micro-batch)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    hidden_buf = torch.randn((T_max, H), device=dev, dtype=torch.bfloat16, generator=g)
    gw = torch.Generator(device=dev).manual_seed(99)  # same W on every rank
    weight = (torch.randn((V, H), device=dev, dtype=torch.float32, generator=gw) * 0.02).to(torch.bfloat16)
    TAB_KEYS = ("token_pool", "seg_src_off", "seg_len", "seg_is_action", "traj_seg_off")
    gn = torch.Generator(device=dev).manual_seed(4321 + rank)
    mbs = []
    for w in wls:
        dtab = {k: torch.from_numpy(np.ascontiguousarray(getattr(w.table, k))).to(dev)
                for k in TAB_KEYS}
        lold = torch.from_numpy(w.logp_old).to(dev)
        lref = torch.from_numpy(w.logp_ref).to(dev)
        hidden = hidden_buf[:w.n_tokens]
        # Realistic behaviour-policy log-probs: the current policy's logp on
        # the action rows (forward-only fused LM head) plus a small drift, so
        # ratios, clip fraction and KL sit where a real GRPO step puts them.
        packed0 = packing.pack_table(w.table, device=dev, validate=True, vocab=V, device_inputs=dtab)
        lp_now, _, _ = grpo.lmhead_logprobs(hidden, weight, packed0.input_ids, rows=packed0.act_idx)
        act_rows = packed0.act_idx.long()
        lold[act_rows] = lp_now + 0.1 * torch.randn(lp_now.shape, device=dev, generator=gn)
        lref[act_rows] = lold[act_rows] + 0.05 * torch.randn(lp_now.shape, device=dev, generator=gn)
        w.logp_old = lold.cpu().numpy()
        w.logp_ref = lref.cpu().numpy()
        del packed0, lp_now, act_rows
        mbs.append({"wl": w, "dtab": dtab, "lold": lold, "lref": lref, "hidden": hidden,
                    "rewards": torch.from_numpy(w.rewards).to(dev),
                    "report": torch.empty(_lib.TL_REPORT_LEN, dtype=torch.float64, device=dev)})
    step = grpo.GRPOStep(H, V, loss_cfg, chunk_rows=args.chunk_rows,
                         recompute=args.mode == "recompute", pipelined=args.mode == "pipelined")
    dhidden_buf = torch.empty((T_max, H), dtype=torch.bfloat16, device=dev)
    dweight = torch.empty((V, H), dtype=torch.float32, device=dev)
    logp_buf = torch.empty(T_max, dtype=torch.float32, device=dev)
    ent_buf = torch.empty(T_max, dtype=torch.float32, device=dev)

    def one_step(inputs):
        """inputs[i] = (device segment table, logp_old, logp_ref, rewards) of micro-batch i"""
        reps = []
        for i, (mb, (dt, lo, lr, rw)) in enumerate(zip(mbs, inputs)):
            w = mb["wl"]
            packed = packing.pack_table(w.table, device=dev, validate=False, device_inputs=dt)
            out = {"logp": logp_buf[:w.n_tokens], "entropy": ent_buf[:w.n_tokens],
                   "dhidden": dhidden_buf[:w.n_tokens], "dweight": dweight,
                   "report": mb["report"]}
            res = step(packed, w.group_off, rw, mb["hidden"], weight, lo, lr,
                       norm_groups=n_groups_global, norm_tokens=norm_tokens, outputs=out,
                       sync_report=False, accumulate_dweight=i > 0)
            reps.append(res.report_tensor)
        rep = reps[0] if len(reps) == 1 else combine_reports_device(reps, agg)
        if world > 1:
            parallel.allreduce_report(rep, agg)
            parallel.allreduce_grad(dweight)
        return rep

    def device_inputs():
        return [(mb["dtab"], mb["lold"], mb["lref"], mb["rewards"]) for mb in mbs]

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- warm-up
    for _ in range(args.warmup):
        one_step(device_inputs())
    torch.cuda.synchronize()
    barrier()

    # ---- timed region (device-resident inputs; inputs >> L2: hidden is GBs)
    launches0 = _lib.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier()
        ev0.record()
        for _ in range(args.steps):
            rep_t = one_step(device_inputs())
        ev1.record()
        torch.cuda.synchronize()
        barrier()
    launches = _lib.launch_count() - launches0
    ms = ev0.elapsed_time(ev1) / args.steps
    t_max = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms = float(t_max.item())
    rep = grpo.report_dict(rep_t.cpu())
    tok_global = torch.tensor([T, n_act], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tok_global)
    T_all, A_all = (float(x) for x in tok_global.tolist())
    value = T_all / (ms / 1e3)

    # ---- per-kernel device timing (separate, untimed pass)
    prof = {}
    if not args.no_profile:
        _lib.profile_enable(True)
        one_step(device_inputs())
        torch.cuda.synchronize()
        prof = _lib.profile_read()
        _lib.profile_enable(False)

    # ---- end-to-end through the public API with host inputs
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        hosts = [({k: pin(getattr(mb["wl"].table, k)) for k in TAB_KEYS}, pin(mb["wl"].logp_old),
                  pin(mb["wl"].logp_ref), pin(mb["wl"].rewards)) for mb in mbs]
        h2d = sum(sum(v.numel() * v.element_size() for v in ht.values()) + lo.numel() * 4 +
                  lr.numel() * 4 + rw.numel() * 8 for ht, lo, lr, rw in hosts)
        host_rep = torch.empty(_lib.TL_REPORT_LEN, dtype=torch.float64).pin_memory()
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            inputs = [({k: v.to(dev, non_blocking=True) for k, v in ht.items()},
                       lo.to(dev, non_blocking=True), lr.to(dev, non_blocking=True),
                       rw.to(dev, non_blocking=True)) for ht, lo, lr, rw in hosts]
            r = one_step(inputs)
            host_rep.copy_(r, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        e1.record()
        torch.cuda.synchronize()
        barrier()
        ems = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e2e = {"value": T_all / (float(ems.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(host_rep.numel() * 8),
               "ms_per_step": float(ems.item()),
               "inputs": "segment table + logp_old/logp_ref + rewards from pinned host memory; "
                         "hidden states / LM-head weight device-resident (model tensors)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak_s, peak_b, hbm, peak_kind = _peaks()
    flops_alg = 6.0 * n_act * H * V      # fwd logp (2) + dH (2) + dW (2), action rows only
    # issued tensor FLOPs: the recompute mode runs the logits GEMM a second time
    flops_issued = (8.0 if args.mode == "recompute" else 6.0) * n_act * H * V
    gemm_ms = sum(prof.get(k, (0, 0))[0] for k in ("gemm_fwd", "gemm_dsoftmax", "gemm_dh", "gemm_dw"))
    gemm_launch = sum(prof.get(k, (0, 0))[1] for k in ("gemm_fwd", "gemm_dsoftmax", "gemm_dh", "gemm_dw"))
    roofline = None
    traffic, traffic_note = None, None
    tp = ROOT / "profiles" / TRAFFIC_JSON
    if tp.exists() and cfg.name == "c2":
        tj = json.loads(tp.read_text())
        per_chunk = sum(v["dram_read_GB"] + v["dram_write_GB"]
                        for k, v in tj["per_chunk"].items() if k.startswith("gemm"))
        traffic = per_chunk * 1e9 * n_act / tj["chunk_rows"]
        traffic_note = (f"bytes/step = ncu --set full DRAM read+write of the fwd/dH/dW GEMM launches "
                        f"of one {tj['chunk_rows']}-row chunk ({per_chunk:.1f} GB, {tp.name}) x chunks/step; "
                        f"per chunk each GEMM must read W (1.09 GB) and h_c or dS (0.27 / 11.5 GB) once")
    if gemm_ms > 0:
        ach = flops_alg / (gemm_ms / 1e3) / 1e12
        roofline = {
            "bound": "tensor", "achieved": ach, "peak": peak_s, "unit": "TFLOP/s",
            "frac": ach / peak_s, "traffic": traffic, "traffic_note": traffic_note,
            "kernel": "gemm_sm100_kernel (tcgen05 LM-head fwd / dS recompute / dH / dW), "
                      "algorithmic 6*T_act*H*V per step over their summed event time",
            "launches_per_step": gemm_launch,
            "issued_frac": flops_issued / (gemm_ms / 1e3) / 1e12 / peak_s,
            "frac_of_burst_peak": ach / peak_b,
            "step_frac": (flops_alg / (peak_s * 1e12)) / (ms / 1e3),
            "peak_kind": f"{peak_kind} bf16 sustained",
        }
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": cfg.desc, "name": cfg.name, "global_batch": cfg.prompts * cfg.n * world,
                   "seq_len": cfg.seq, "hidden": H, "vocab": V,
                   "tokens_per_step": int(T_all), "action_tokens_per_step": int(A_all),
                   "action_tokens_per_s": A_all / (ms / 1e3),
                   "parallelism": f"dp{world} (groups, LPT)", "l2": "inputs >> L2 (hidden is GBs)",
                   "chunk_rows": step.last_chunk, "loss_agg": cfg.loss_agg,
                   "micro_batches": len(mbs),
                   "lmhead_mode": args.mode},
        "roofline": roofline,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "kernel_ms_per_step": {k: v[0] for k, v in prof.items() if v[1]},
        "report": {k: rep[k] for k in ("objective", "clip_fraction", "masked_tokens", "kl")},
    }
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg, wl)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
