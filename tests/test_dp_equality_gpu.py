"""Data parallelism by trajectory group: N ranks == 1 rank on the kernels'
own outputs ("verify that the N-rank report equals the 1-rank
report"; reference aggregation cli.py:317-344, parallel-safe per SPEC.md:496).

Two ranks (processes) share the box's one GPU over gloo: each runs the fused
GRPO step (K2 advantages -> K4 LM-head logp + surrogate -> K5 backward) on
its LPT shard of a global batch with the global normalisers, then N1 (report)
and N2 (dW) all-reduce.  Compared with one rank on the same global batch:

  * as micro-batches = the same shards in sequence (dW accumulated across
    calls, reports combined): per-token logp / entropy / dhidden bitwise, the
    report to fp64 summation order (rel 1e-12), dW to fp32 summation order
    (rel Frobenius 1e-6);
  * in one call over all groups: per-token logp / entropy / dS are bitwise
    too (the forward's K order is fixed per vocab tile, not per wave:
    GemmShape::serpentine == 2), the report rel 1e-12; dhidden to its dH GEMM
    K order (serpentine parity follows the wave; <= 1 bf16 ulp, rel
    Frobenius 1e-3), dW to chunk composition (rel Frobenius 1e-5).

The NCCL path of the same collectives (tl_allreduce_report /
tl_allreduce_f32 at the C ABI) is exercised with a 1-rank communicator
(NCCL refuses two ranks on one device).
"""

import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

H, V = 256, 3000
N_GROUPS, G = 12, 4
CHUNK = 512


def _global_batch():
    """Deterministic global batch: per-group trajectories (segment lists),
    rewards, per-token logp_old / logp_ref, hidden rows."""
    from paper_2509_01055_b200.synthetic import WorkloadConfig, make_workload

    cfg = WorkloadConfig("dp", N_GROUPS, G, (0, 3), 640, H, V, 0.3, "pm1")
    wl = make_workload(cfg)
    t = wl.table
    groups = []
    tok = 0
    for gi in range(N_GROUPS):
        trajs = []
        for b in range(gi * G, (gi + 1) * G):
            segs = []
            for s in range(t.traj_seg_off[b], t.traj_seg_off[b + 1]):
                o, n = int(t.seg_src_off[s]), int(t.seg_len[s])
                segs.append(("action" if t.seg_is_action[s] else "observation",
                             t.token_pool[o:o + n].tolist()))
            trajs.append(segs)
        n_tok = sum(len(x) for tr in trajs for _, x in tr)
        groups.append({"trajs": trajs, "rewards": wl.rewards[gi * G:(gi + 1) * G],
                       "tok": (tok, tok + n_tok),
                       "n_act": sum(len(x) for tr in trajs for o, x in tr if o == "action")})
        tok += n_tok
    gen = torch.Generator(device="cuda").manual_seed(77)
    hidden = torch.randn((tok, H), device="cuda", generator=gen).bfloat16()
    W = (torch.randn((V, H), device="cuda", generator=gen) * 0.05).bfloat16()
    return groups, wl.logp_old, wl.logp_ref, hidden, W


def _run(group_ids, groups, lold, lref, hidden, W, *, dw=None, accumulate=False):
    """One fused step over `group_ids` (in order) with the global normalisers."""
    from paper_2509_01055_b200 import grpo, packing
    from paper_2509_01055_b200.rl.loss import LossConfig
    from paper_2509_01055_b200.trajectory import Segment, Trajectory

    trajs, rewards, rows = [], [], []
    for g in group_ids:
        trajs += [Trajectory([Segment(o, "", x) for o, x in tr]) for tr in groups[g]["trajs"]]
        rewards.append(groups[g]["rewards"])
        rows.append(np.arange(*groups[g]["tok"]))
    rows = np.concatenate(rows)
    packed = packing.pack(trajs)
    go = np.arange(0, len(group_ids) * G + 1, G, dtype=np.int32)
    ridx = torch.from_numpy(rows).cuda()
    f = lambda a: torch.from_numpy(np.ascontiguousarray(a[rows])).cuda()  # noqa: E731
    cfg = LossConfig(epsilon_clip=0.2, kl_beta=0.05, entropy_coef=0.01)
    step = grpo.GRPOStep(H, V, cfg, chunk_rows=CHUNK)
    out = {"dweight": dw} if dw is not None else None
    n_act_global = sum(g["n_act"] for g in groups)
    res = step(packed, go, np.concatenate(rewards), hidden[ridx].contiguous(), W, f(lold), f(lref),
               norm_groups=N_GROUPS, norm_tokens=n_act_global, outputs=out,
               accumulate_dweight=accumulate)
    torch.cuda.synchronize()
    return res, rows


def _rank_main(rank, world, port, outdir):
    import torch.distributed as dist

    from paper_2509_01055_b200 import parallel

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    groups, lold, lref, hidden, W = _global_batch()
    shards = parallel.shard_groups(np.array([g["n_act"] for g in groups]), world)
    res, rows = _run(shards[rank], groups, lold, lref, hidden, W)
    rep = res.report_tensor
    parallel.allreduce_report(rep, 0)
    parallel.allreduce_grad(res.dweight)
    torch.save({"rows": rows, "report": rep.cpu(), "dweight": res.dweight.cpu(),
                "logp": res.logp.cpu(), "entropy": res.entropy.cpu(),
                "dhidden": res.dhidden.cpu(), "shard": shards[rank]},
               os.path.join(outdir, f"rank{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rel_fro(a, b):
    a, b = a.double(), b.double()
    return float(torch.linalg.norm(a - b) / torch.linalg.norm(b))


def _gather(parts, key, n_tok, width=None):
    shape = (n_tok,) if width is None else (n_tok, width)
    out = torch.zeros(shape, dtype=parts[0][key].dtype)
    for p in parts:
        out[torch.from_numpy(p["rows"])] = p[key][:len(p["rows"])]
    return out


def test_two_ranks_equal_one_rank():
    import torch.multiprocessing as mp

    from paper_2509_01055_b200 import parallel

    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank_main, args=(world, _free_port(), d), nprocs=world, join=True)
        parts = [torch.load(os.path.join(d, f"rank{r}.pt"), weights_only=False)
                 for r in range(world)]
    groups, lold, lref, hidden, W = _global_batch()
    n_tok = hidden.shape[0]
    assert sorted(np.concatenate([p["shard"] for p in parts]).tolist()) == list(range(N_GROUPS))
    assert all(len(p["shard"]) > 0 for p in parts)
    # the all-reduced report is identical on every rank
    assert torch.equal(parts[0]["report"], parts[1]["report"])
    rep_n = parts[0]["report"].double().numpy()
    dw_n = parts[0]["dweight"]
    assert torch.equal(dw_n, parts[1]["dweight"])

    # (a) one rank, the same shards as micro-batches in sequence
    dw = torch.empty((V, H), dtype=torch.float32, device="cuda")
    reps, seq = [], []
    for i, p in enumerate(parts):
        r, rows = _run(p["shard"], groups, lold, lref, hidden, W, dw=dw, accumulate=i > 0)
        reps.append(r.report_tensor.cpu().numpy())
        seq.append({"rows": rows, "logp": r.logp.cpu(), "entropy": r.entropy.cpu(),
                    "dhidden": r.dhidden.cpu()})
    rep_seq = parallel.combine_reports(reps, 0)
    np.testing.assert_allclose(rep_n, rep_seq, rtol=1e-12, atol=0)
    assert rep_n[2] == rep_seq[2] and rep_n[4] == N_GROUPS
    assert _rel_fro(dw_n, dw.cpu()) <= 1e-6
    for k, w in (("logp", None), ("entropy", None), ("dhidden", H)):
        assert torch.equal(_gather(parts, k, n_tok, w), _gather(seq, k, n_tok, w)), k

    # (b) one rank, one call over every group (global order)
    one, rows = _run(list(range(N_GROUPS)), groups, lold, lref, hidden, W)
    assert np.array_equal(rows, np.arange(n_tok))
    rep_1 = one.report_tensor.cpu().double().numpy()
    np.testing.assert_allclose(rep_n, rep_1, rtol=1e-12, atol=1e-15)
    assert rep_n[2] == rep_1[2] and rep_n[5] == rep_1[5]
    assert torch.equal(_gather(parts, "logp", n_tok), one.logp.cpu())
    assert torch.equal(_gather(parts, "entropy", n_tok), one.entropy.cpu())
    assert _rel_fro(_gather(parts, "dhidden", n_tok, H).float(), one.dhidden.cpu().float()) <= 1e-3
    assert _rel_fro(dw_n, one.dweight.cpu()) <= 1e-5


def test_nccl_collectives_at_the_c_abi():
    """tl_nccl_* / tl_allreduce_* with a one-rank NCCL communicator: the
    collectives run (NCCL kernels on the caller's stream), the report's
    ratio fields are recomputed from the additive partials, reduce-scatter
    with one rank is the identity."""
    from paper_2509_01055_b200 import _lib, parallel

    L = _lib.lib()
    assert L.tl_nccl_available() == 1 and L.tl_nccl_version() >= 22000
    comm = parallel.NcclComm(parallel.NcclComm.unique_id(), 1, 0)
    try:
        assert comm.size() == 1
        rep = torch.zeros(_lib.TL_REPORT_LEN, dtype=torch.float64, device="cuda")
        rep[2], rep[4], rep[8], rep[9], rep[11] = 40.0, 4.0, 3.0, 2.0, 1.0
        comm.allreduce_report(rep, 0)
        torch.cuda.synchronize()
        assert rep[0].item() == 0.25 and rep[1].item() == 3.0 / 40 and rep[3].item() == 2.0 / 40
        comm.allreduce_report(rep, 1)
        assert rep[0].item() == 1.0 / 40
        x = torch.randn(1 << 20, device="cuda")
        y = x.clone()
        comm.allreduce_grad(y)
        s = torch.empty_like(x)
        comm.reduce_scatter_grad(x, s)
        torch.cuda.synchronize()
        assert torch.equal(x, y) and torch.equal(s, x)
        d = torch.arange(5, dtype=torch.float64, device="cuda")
        comm.allreduce_scalars(d)
        assert d.tolist() == [0.0, 1.0, 2.0, 3.0, 4.0]
    finally:
        comm.close()


@pytest.mark.parametrize("factored", [True, False])
def test_n2_overlap_event_and_reserved_sms(factored):
    """tl_grpo_lmhead_step_overlap: the last chunk runs dW before dH, records
    dw_ready once dW is final and leaves SMs free for the dH GEMM's
    neighbour; a dW all-reduce issued on a side stream after the event
    (one-rank NCCL communicator: the identity) must see the final dW, and
    every output equals the plain step bitwise."""
    from paper_2509_01055_b200 import grpo, packing, parallel
    from paper_2509_01055_b200.rl.loss import LossConfig
    from paper_2509_01055_b200.trajectory import Segment, Trajectory

    groups, lold, lref, hidden, W = _global_batch()
    trajs = [Trajectory([Segment(o, "", x) for o, x in tr]) for g in groups for tr in g["trajs"]]
    rewards = np.concatenate([g["rewards"] for g in groups])
    go = np.arange(0, len(trajs) + 1, G, dtype=np.int32)
    packed = packing.pack(trajs)
    lo = torch.from_numpy(np.asarray(lold, dtype=np.float32)).cuda()
    lr = torch.from_numpy(np.asarray(lref, dtype=np.float32)).cuda()
    cfg = LossConfig(kl_beta=0.04, entropy_coef=0.0 if factored else 0.01)
    step = grpo.GRPOStep(H, V, cfg, chunk_rows=CHUNK)  # several chunks
    assert packed.n_act > 2 * CHUNK
    ref = step(packed, go, rewards, hidden, W, lo, lr)
    dh0, dw0 = ref.dhidden.clone(), ref.dweight.clone()
    comm = parallel.NcclComm(parallel.NcclComm.unique_id(), 1, 0)
    try:
        ev, side = torch.cuda.Event(), torch.cuda.Stream()
        res = step(packed, go, rewards, hidden, W, lo, lr, dw_ready=ev, reserve_sms=16)
        side.wait_event(ev)
        snap = torch.empty_like(res.dweight)
        with torch.cuda.stream(side):
            snap.copy_(res.dweight)               # what a collective after the event reads
        comm.allreduce_grad(res.dweight, stream=side)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        assert torch.equal(snap, dw0)
        assert torch.equal(res.dweight, dw0) and torch.equal(res.dhidden, dh0)
        assert res.report == ref.report
        assert torch.equal(res.logp, ref.logp)
    finally:
        comm.close()
