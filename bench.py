"""Benchmark: masked GRPO-step tokens/sec (pack + advantage + LM-head log-prob
+ surrogate loss + LM-head backward) on B200, vs the reference's CPU path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5]
                    [--impl ours|reference] [--mode store|store-fp16|pipelined|recompute]
                    [--n2-overlap SMS]

One step = the whole trajectory-to-loss hot path over one synthetic batch of
BASELINE.json's config (default C2, Qwen2.5-7B shape: 256 prompts x 8
rollouts, <= 4 tool turns, seq 4k, H 3584, V 152064, bf16):
  K1 pack (segment table -> varlen batch) -> K2 group advantages ->
  K4 fused LM-head logp/entropy + GRPO surrogate epilogue (keeps the chunk's
  bf16 q = e^(z - m0): dS = alpha_r q without an entropy bonus)
  -> K5 backward (dH = alpha (q W), dW += q^T (alpha H)) -> deterministic
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
TRAFFIC_JSON = "r2f_gemm_traffic.json"


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
              "clocks_event_reasons.sw_power_cap,power.draw,power.limit")

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
        sm, mx, pw, lim, reasons = [], [], [], [], set()
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except ValueError:
                continue
            for n, v in zip(names, r[2:6]):
                if "Active" in v and "Not" not in v:
                    reasons.add(n)
            try:  # board power (W): the step runs at the power limit
                pw.append(float(r[6]))
                lim.append(float(r[7]))
            except (IndexError, ValueError):
                pass
        out = {"sm_mhz": float(np.median(sm)) if sm else None,
               "sm_max_mhz": float(max(mx)) if mx else None,
               "samples": len(sm), "reasons": sorted(reasons)}
        if pw:
            out["power_w"] = float(np.median(pw))
            out["power_limit_w"] = float(max(lim))
        return out


# ---------------------------------------------------------- CPU baseline --
def workload_config(cfg, world: int, scaling: str) -> dict:
    """The `config` object of both arms' JSON lines (workload only; the GPU
    arm's implementation choices go to `impl_config`)."""
    from paper_2509_01055_b200.synthetic import group_act_tokens, group_tokens

    n_groups = cfg.prompts * (world if scaling == "weak" else 1)
    gids = np.arange(n_groups)
    return {"workload": cfg.desc, "name": cfg.name, "global_batch": n_groups * cfg.n,
            "seq_len": cfg.seq, "hidden": cfg.hidden, "vocab": cfg.vocab,
            "tokens_per_step": int(group_tokens(cfg, gids).sum()),
            "action_tokens_per_step": int(group_act_tokens(cfg, gids).sum()),
            "loss_agg": cfg.loss_agg, "parallelism": f"dp{world} (groups, LPT)",
            "l2": "inputs >> L2 (hidden is GBs)"}


def _calibrated_sampler(cfg, target_s: float):
    """ReferenceSampler whose LM-head block takes ~target_s per sample."""
    import bench_reference as R

    smp = R.ReferenceSampler(cfg, lm_rows=64)
    rate = 64 / smp.lm.run(64)
    smp.lm_rows = int(min(4096, max(64, round(rate * target_s / 64) * 64)))
    return smp


def cpu_baseline(cfg, target_s: float = 8.0) -> dict:
    """The reference's CPU path timed on a bounded sample (bench_reference):
    rank 0, N = 1, one ~10-30 s sample."""
    import bench_reference as R

    smp = _calibrated_sampler(cfg, target_s)
    try:
        st = smp.step()
    finally:
        smp.close()
    return {"value": st["value"], "unit": UNIT, "cores": R.n_cores(), "kind": smp.kind,
            "sample": smp.describe(st), "extrapolated_step_ms": st["extrapolated_step_ms"],
            "host_cpu": R.cpu_model()}


def run_reference(args, cfg):
    """--impl reference: the reference's own CPU implementation of the path
    (bench_reference.py) on the host cores, rank 0 only (other ranks exit
    0).  A step = one bounded sample of the workload (loss path on whole
    groups, single-process and fanned out over every core; the LM head on a
    block of action rows sized to ~--ref-seconds); `value` = the workload's
    tokens/s extrapolated from the sample's per-token costs (median over
    steps), `ms_per_step` = the measured wall time of one sample, and
    `extrapolated_step_ms` = the whole configured step at that rate."""
    import bench_reference as R

    if int(os.environ.get("RANK", "0")) != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    smp = _calibrated_sampler(cfg, args.ref_seconds)
    try:
        for _ in range(args.warmup):
            smp.step()
        res = []
        t0 = time.perf_counter()
        for _ in range(args.steps):
            res.append(smp.step())
        wall = time.perf_counter() - t0
        # the LM-head restatement on a 4096-row block once, for its GFLOP/s
        t_lm = smp.lm.run(4096)
    finally:
        smp.close()
    v = float(np.median([r["value"] for r in res]))
    last = res[-1]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall / max(args.steps, 1) * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f64 (reference loss path) / f32 (LM head restatement)", "data": "synthetic",
        "config": workload_config(cfg, world, args.scaling),
        "extrapolated_step_ms": float(np.median([r["extrapolated_step_ms"] for r in res])),
        "ms_per_step_note": "wall time of one bounded sample; extrapolated_step_ms = the whole "
                            "configured step at the sampled per-token rates",
        "lm_head_4096_rows": {"s": t_lm, "gflops": 6.0 * 4096 * cfg.hidden * cfg.vocab / t_lm / 1e9,
                              "threads": R.n_cores()},
        "cpu_baseline": {"kind": smp.kind, "cores": R.n_cores(), "sample": smp.describe(last),
                         "value": v, "unit": UNIT, "host_cpu": R.cpu_model()},
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


def _free_port() -> int:
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _relaunch(n: int) -> int:
    """`bench.py --gpus N` without a launcher: re-exec this command as N
    ranks under torch.distributed.run (one process per GPU, rendezvous on
    127.0.0.1) and return its exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           str(Path(__file__).resolve()), *sys.argv[1:]]
    print(f"[bench] launching {n} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: each rank owns a full config-sized batch (global batch = N x config); "
                         "strong: the config's batch is split across the N ranks")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=8.0)
    ap.add_argument("--chunk-rows", type=int, default=None)
    ap.add_argument("--max-mb-tokens", type=int, default=7_000_000,
                    help="largest micro-batch (packed tokens) a rank holds at once")
    ap.add_argument("--n2-overlap", type=int, default=0, metavar="SMS",
                    help="N > 1 with NCCL: run the dW all-reduce on a side stream beside the "
                         "last chunk's dH GEMM, which leaves SMS SMs free for it (0: after the "
                         "step; DESIGN.md section 6)")
    ap.add_argument("--mode", default="store",
                    choices=["store", "store-fp16", "pipelined", "recompute"],
                    help="LM-head backward schedule (TL_LMHEAD_* in include/toolloop_b200.h); "
                         "store is fastest on a power-capped B200 (DESIGN.md §3) and, without "
                         "an entropy bonus, runs factored (bf16 q, no dS pass); store-fp16 "
                         "forces the fp16-logit store + dS pass (TL_LMHEAD_NO_FACTORED)")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(_relaunch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

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

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TL_BENCH_ONE_DEVICE=1 + TL_BENCH_BACKEND=gloo: every rank on cuda:0 over
    # gloo — exercises the multi-rank path (sharding, N1/N2 all-reduces,
    # max-over-ranks timing) on a one-GPU box with a small --config.
    if os.environ.get("TL_BENCH_ONE_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    # TL_BENCH_FORCE_PG=1 (tests): a one-rank process group and NCCL
    # communicator, so the N1 / N2 collective path runs on a one-GPU box
    use_pg = world > 1 or os.environ.get("TL_BENCH_FORCE_PG") == "1"
    if use_pg:
        backend = os.environ.get("TL_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            # NCCL's init lines (nranks, NVLS / channels) go to stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=dev)
            # the step's own collectives (N1 report, N2 dW) go through the
            # library's NCCL communicator at the C ABI (tl_nccl_*)
            try:
                comm = parallel.NcclComm.from_process_group()
            except Exception as e:  # keep the run: same collectives through torch's NCCL group
                print(f"bench.py: NCCL at the C ABI unavailable ({e}); N1 / N2 via "
                      "torch.distributed", file=sys.stderr)
                comm = None
        else:
            dist.init_process_group(backend)

    # global batch: world x config (weak) or the config split across ranks
    # (strong); whole groups per rank by LPT
    n_groups_global = cfg.prompts * (world if args.scaling == "weak" else 1)
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
                         recompute=args.mode == "recompute", pipelined=args.mode == "pipelined",
                         factored=args.mode != "store-fp16")
    dhidden_buf = torch.empty((T_max, H), dtype=torch.bfloat16, device=dev)
    dweight = torch.empty((V, H), dtype=torch.float32, device=dev)
    logp_buf = torch.empty(T_max, dtype=torch.float32, device=dev)
    ent_buf = torch.empty(T_max, dtype=torch.float32, device=dev)

    dw_ready = torch.cuda.Event() if comm is not None and args.n2_overlap > 0 else None
    n2_stream = torch.cuda.Stream() if dw_ready is not None else None

    def one_step(inputs):
        """inputs[i] = (device segment table, logp_old, logp_ref, rewards) of micro-batch i"""
        reps = []
        for i, (mb, (dt, lo, lr, rw)) in enumerate(zip(mbs, inputs)):
            w = mb["wl"]
            packed = packing.pack_table(w.table, device=dev, validate=False, device_inputs=dt)
            out = {"logp": logp_buf[:w.n_tokens], "entropy": ent_buf[:w.n_tokens],
                   "dhidden": dhidden_buf[:w.n_tokens], "dweight": dweight,
                   "report": mb["report"]}
            last = i == len(mbs) - 1
            overlap = comm is not None and args.n2_overlap > 0 and last
            res = step(packed, w.group_off, rw, mb["hidden"], weight, lo, lr,
                       norm_groups=n_groups_global, norm_tokens=norm_tokens, outputs=out,
                       sync_report=False, accumulate_dweight=i > 0,
                       dw_ready=dw_ready if overlap else None,
                       reserve_sms=args.n2_overlap if overlap else 0)
            if overlap:  # N2 beside the last chunk's dH GEMM (tl_grpo_lmhead_step_overlap)
                n2_stream.wait_event(dw_ready)
                comm.allreduce_grad(dweight, stream=n2_stream)
            reps.append(res.report_tensor)
        rep = reps[0] if len(reps) == 1 else combine_reports_device(reps, agg)
        if comm is not None and args.n2_overlap > 0:
            comm.allreduce_report(rep, agg)
            torch.cuda.current_stream().wait_stream(n2_stream)
        elif comm is not None:   # N1 + N2 at the C ABI (NCCL), stream-ordered
            comm.allreduce_report(rep, agg)
            comm.allreduce_grad(dweight)
        elif use_pg:            # gloo process group (ranks sharing one GPU)
            parallel.allreduce_report(rep, agg)
            parallel.allreduce_grad(dweight)
        return rep

    def device_inputs():
        return [(mb["dtab"], mb["lold"], mb["lref"], mb["rewards"]) for mb in mbs]

    def barrier():
        if use_pg:
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
    if use_pg:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms = float(t_max.item())
    rep = grpo.report_dict(rep_t.cpu())
    tok_global = torch.tensor([T, n_act], device=dev, dtype=torch.float64)
    if use_pg:
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
        if use_pg:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e2e = {"value": T_all / (float(ems.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(host_rep.numel() * 8),
               "ms_per_step": float(ems.item()),
               "inputs": "segment table + logp_old/logp_ref + rewards from pinned host memory; "
                         "hidden states / LM-head weight device-resident (model tensors)"}

    if rank != 0:
        if comm is not None:
            comm.close()
        if use_pg:
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
                        f"reading every operand once would be 39.7 GB per chunk, but an output-stationary "
                        f"tile schedule on 74 CTA pairs re-reads W once per dH wave and h_c once per dW "
                        f"wave (TMEM holds one 256x512 fp32 tile per pair): 72.2 GB per chunk is "
                        f"compulsory for it (DESIGN.md section 3)")
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
    wcfg = workload_config(cfg, world, args.scaling)
    assert wcfg["tokens_per_step"] == int(T_all) and wcfg["action_tokens_per_step"] == int(A_all)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": wcfg,
        "impl_config": {"action_tokens_per_s": A_all / (ms / 1e3),
                        "collectives": ("NCCL at the C ABI (tl_allreduce_report, tl_allreduce_f32)"
                                        if comm is not None else
                                        ("torch.distributed " + dist.get_backend()) if use_pg
                                        else "none"),
                        "chunk_rows": step.last_chunk, "micro_batches": len(mbs),
                        "lmhead_mode": args.mode + (
                            " (factored: bf16 q = e^(z - m0), no dS pass)"
                            if args.mode in ("store", "pipelined") and loss_cfg.entropy_coef == 0
                            else "")},
        "roofline": roofline,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "kernel_ms_per_step": {k: v[0] for k, v in prof.items() if v[1]},
        "report": {k: rep[k] for k in ("objective", "clip_fraction", "masked_tokens", "kl")},
    }
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg)
    print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if use_pg:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
