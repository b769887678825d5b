"""The multi-rank bench path (one process per rank: LPT group sharding, N1
report all-reduce, N2 dW all-reduce, barriers, max-over-ranks timing, rank-0
JSON line) run end to end with two ranks sharing the one GPU of a gpurun box
over gloo, on the small `tiny` workload.  The report must cover the whole
global batch: masked_tokens == action tokens of all groups of both ranks."""

import json
import os
import socket
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


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_bench_tiny():
    from paper_2509_01055_b200.synthetic import CONFIGS, group_act_tokens

    env = dict(os.environ, TL_BENCH_ONE_DEVICE="1", TL_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--gpus", "2", "--config", "tiny", "--steps", "2", "--warmup", "3", "--no-cpu"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 only
    d = json.loads(lines[0])
    cfg = CONFIGS["tiny"]
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 2 * cfg.prompts * cfg.n
    want = int(np.sum(group_act_tokens(cfg, np.arange(2 * cfg.prompts))))
    assert d["report"]["masked_tokens"] == want
    assert d["config"]["action_tokens_per_step"] == want
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
