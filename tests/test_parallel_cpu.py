"""Data parallelism by trajectory group: LPT sharding and the N1 report
all-reduce, exercised with world_size 2 over gloo on CPU.  The per-shard
report partials come from the oracle (what each rank's kernels produce), and
the reduced report must equal the single-rank report of the whole batch
(cli.py:309-344 aggregation)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import grpo_oracle as O
from paper_2509_01055_b200 import parallel


def test_lpt_shard_balanced_and_deterministic():
    rng = np.random.default_rng(0)
    work = rng.lognormal(8, 1, 64).astype(np.int64)
    shards = parallel.shard_groups(work, 8)
    assert sorted(np.concatenate(shards).tolist()) == list(range(64))
    loads = [int(work[s].sum()) for s in shards]
    assert max(loads) - min(loads) <= work.max()  # LPT bound
    again = parallel.shard_groups(work, 8)
    assert all(np.array_equal(a, b) for a, b in zip(shards, again))
    assert [len(s) for s in parallel.shard_groups(work, 1)] == [64]


def _batch(seed=0, n_groups=10, G=4):
    rng = np.random.default_rng(seed)
    groups = []
    for _ in range(n_groups):
        trajs = []
        for _ in range(G):
            n = int(rng.integers(1, 12))
            trajs.append([(0, float(-rng.exponential()), float(-rng.exponential()),
                           int(rng.integers(0, 2)) if i else 1, float(-rng.exponential()))
                          for i in range(n)])
        groups.append((trajs, rng.choice([1.0, -1.0, 0.5], G).tolist()))
    return groups


def _report_partials(groups, eps=0.2, beta=0.1):
    """The additive TL_REPORT_LEN partials a rank's kernels emit for its groups."""
    rep = np.zeros(12)
    for trajs, rewards in groups:
        adv = O.group_advantages(rewards)
        obj, d = O.multi_turn(trajs, adv, eps, beta)
        rep[2] += d["masked_tokens"]
        rep[4] += 1
        rep[5] += len(trajs)
        rep[6] += d["total_tokens"]
        rep[7] += d["clamp_count"]
        rep[8] += round(d["clip_fraction"] * d["masked_tokens"])
        rep[9] += d["kl"] * d["masked_tokens"]
        rep[11] += obj
    return rep


def _worker(rank, world, port, groups, shards, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = [groups[g] for g in shards[rank]]
    t = torch.tensor(_report_partials(mine), dtype=torch.float64)
    parallel.allreduce_report(t, agg=0)
    out[rank] = t.numpy().copy()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_report_equals_single_rank():
    groups = _batch()
    work = np.asarray([sum(sum(r[3] for r in t) for t in g[0]) for g in groups])
    shards = parallel.shard_groups(work, 2)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), groups, shards, out), nprocs=2, join=True)
    ref = O.loss_report(groups, 0.2, 0.1)
    for r in range(2):
        rep = out[r]
        assert rep[2] == ref["masked_tokens"] and rep[4] == ref["groups"]
        assert rep[5] == ref["episodes"]
        assert abs(rep[0] - ref["objective"]) <= 1e-12
        assert abs(rep[1] - ref["clip_fraction"]) <= 1e-12
        assert abs(rep[3] - ref["kl"]) <= 1e-12
    assert np.array_equal(out[0], out[1])


def test_finalize_report_matches_allreduce():
    groups = _batch(3)
    a = _report_partials(groups[:5]) + _report_partials(groups[5:])
    fin = parallel.finalize_report(a)
    ref = O.loss_report(groups, 0.2, 0.1)
    assert abs(fin[0] - ref["objective"]) <= 1e-12
    assert abs(fin[3] - ref["kl"]) <= 1e-12


def test_combine_reports_micro_batches():
    """Micro-batches of whole groups: combining their reports (additive
    partials, then ratios) gives the one-shot report, in host and in device
    (bench.combine_reports_device) form."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench

    groups = _batch(5, n_groups=12)
    parts = [_report_partials(groups[a:b]) for a, b in ((0, 4), (4, 5), (5, 12))]
    for p in parts:  # the kernels also emit the ratios; combine must recompute them
        p[0] = p[11] / max(p[4], 1)
    ref = O.loss_report(groups, 0.2, 0.1)
    for rep in (parallel.combine_reports(parts, 0),
                bench.combine_reports_device([torch.tensor(p) for p in parts], 0).numpy()):
        assert rep[2] == ref["masked_tokens"] and rep[4] == ref["groups"]
        assert abs(rep[0] - ref["objective"]) <= 1e-12
        assert abs(rep[1] - ref["clip_fraction"]) <= 1e-12
        assert abs(rep[3] - ref["kl"]) <= 1e-12


def test_micro_batches_cover_groups_in_order():
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    from paper_2509_01055_b200.synthetic import CONFIGS, group_tokens

    cfg = CONFIGS["c3"]
    groups = np.arange(0, cfg.prompts, 3)
    mbs = bench.micro_batches(cfg, groups, 2_000_000)
    assert np.array_equal(np.concatenate(mbs), groups)
    toks = [int(group_tokens(cfg, m).sum()) for m in mbs]
    assert len(mbs) > 1 and all(t <= 2_000_000 or len(m) == 1 for t, m in zip(toks, mbs))
