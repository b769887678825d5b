"""The multi-rank bench path (one process per rank: LPT group sharding, N1
report all-reduce, N2 dW all-reduce, barriers, max-over-ranks timing, rank-0
JSON line) run end to end with two ranks sharing the one GPU of a gpurun box
over gloo, on the small `tiny` workload, launched exactly as a user would:
`bench.py --gpus 2` with no launcher spawns its own ranks.  The report must
cover the whole global batch (weak: 2 x config; strong: the config split)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = Path(__file__).resolve().parents[1]


def _bench(*extra):
    env = dict(os.environ, TL_BENCH_ONE_DEVICE="1", TL_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    # no launcher: bench.py --gpus 2 spawns its own two ranks (torch.distributed.run)
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--config", "tiny", "--steps", "2",
           "--warmup", "3", "--no-cpu", *extra]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 only
    return json.loads(lines[0])


def test_two_rank_bench_tiny():
    from paper_2509_01055_b200.synthetic import CONFIGS, group_act_tokens

    d = _bench()
    cfg = CONFIGS["tiny"]
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["config"]["global_batch"] == 2 * cfg.prompts * cfg.n
    want = int(np.sum(group_act_tokens(cfg, np.arange(2 * cfg.prompts))))
    assert d["report"]["masked_tokens"] == want
    assert d["config"]["action_tokens_per_step"] == want
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0


def test_two_rank_bench_strong_scaling():
    from paper_2509_01055_b200.synthetic import CONFIGS, group_act_tokens

    d = _bench("--scaling", "strong")
    cfg = CONFIGS["tiny"]
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["global_batch"] == cfg.prompts * cfg.n
    want = int(np.sum(group_act_tokens(cfg, np.arange(cfg.prompts))))
    assert d["report"]["masked_tokens"] == want


def test_bench_rejects_world_mismatch():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "tiny"], cwd=ROOT,
                         env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode != 0 and "WORLD_SIZE=1" in out.stderr


@pytest.mark.parametrize("overlap", [0, 2])
def test_one_rank_nccl_bench_path(overlap):
    """The collective path the driver's N-GPU run takes — NCCL process group,
    the library's NCCL communicator, N1 report / N2 dW at the C ABI, optional
    N2 overlap with the last dH GEMM — on a one-rank group (every gpurun box
    has one GPU), launched under torch.distributed.run like the driver."""
    import socket

    from paper_2509_01055_b200.synthetic import CONFIGS, group_act_tokens

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, TL_BENCH_FORCE_PG="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "1",
           "--config", "tiny", "--steps", "2", "--warmup", "3", "--no-cpu",
           "--n2-overlap", str(overlap)]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert "NCCL at the C ABI" in d["impl_config"]["collectives"]
    cfg = CONFIGS["tiny"]
    assert d["report"]["masked_tokens"] == int(np.sum(group_act_tokens(cfg, np.arange(cfg.prompts))))
    assert d["value"] > 0 and d["e2e"]["value"] > 0
