"""A/B of library builds on the LM-head step's kernels at the C2 shape.

    python tools/dsoftmax_ab.py [lib.so ...]     (default: the product build)

Each library (an A/B build from paper_2509_01055_b200/_build.build(variant=...))
runs in its own process: a fused GRPO step over 4 C2 groups (~76 k action
rows, chunks of 37 888 rows) with the library's per-category CUDA-event
timing; prints one JSON line per library with ms per category and the dS
pass's HBM GB/s (4 bytes per logit: fp16 u in, bf16 dS out)."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

CHILD = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, %r)
from paper_2509_01055_b200 import _lib, grpo, packing
from paper_2509_01055_b200.rl.loss import LossConfig
from paper_2509_01055_b200.synthetic import CONFIGS, make_workload
cfg = CONFIGS["c2"]
wl = make_workload(cfg, group_ids=np.arange(4))
packed = packing.pack_table(wl.table)
H, V = cfg.hidden, cfg.vocab
g = torch.Generator(device="cuda").manual_seed(1)
h = torch.randn((wl.n_tokens, H), device="cuda", generator=g).bfloat16()
W = (torch.randn((V, H), device="cuda", generator=g) * 0.02).bfloat16()
lo = torch.from_numpy(wl.logp_old).cuda(); lr = torch.from_numpy(wl.logp_ref).cuda()
step = grpo.GRPOStep(H, V, LossConfig(kl_beta=0.04, entropy_coef=0.01), chunk_rows=37888)
for _ in range(2):
    step(packed, wl.group_off, wl.rewards, h, W, lo, lr)
res = []
for _ in range(3):
    torch.cuda.synchronize(); _lib.profile_enable(True)
    step(packed, wl.group_off, wl.rewards, h, W, lo, lr)
    torch.cuda.synchronize(); res.append(_lib.profile_read()); _lib.profile_enable(False)
out = {k: float(np.median([r[k][0] for r in res])) for k in res[0] if res[0][k][1]}
vld = (V + 7) // 8 * 8
out["dsoftmax_GBs"] = packed.n_act * vld * 4 / (out["dsoftmax"] / 1e3) / 1e9
out["n_act"] = packed.n_act
out["lib"] = str(_lib.LIB_PATH)
print(json.dumps(out))
"""


def main():
    libs = sys.argv[1:] or [str(ROOT / "paper_2509_01055_b200" / "libtoolloop_b200.so")]
    for lib in libs:
        env = dict(os.environ, TOOLLOOP_B200_LIB=lib)
        r = subprocess.run([sys.executable, "-c", CHILD % str(ROOT)], env=env, capture_output=True,
                           text=True, timeout=900)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        print(line[-1] if line else json.dumps({"lib": lib, "error": r.stderr[-2000:]}), flush=True)


if __name__ == "__main__":
    main()
