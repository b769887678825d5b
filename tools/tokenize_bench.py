"""F4 throughput: rollout segment texts -> token ids, the reference's
ToyMergeTokenizer (pure Python, per segment, as trajectory.append_* calls it)
vs the native batched encoder (csrc/tokenize.cpp).  Runs in the build
container (imports the reference from /root/reference); identical ids
asserted.

    PYTHONPATH=/root/reference/pkg/src python tools/tokenize_bench.py [n_traj]
"""

import random
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main(n_traj: int = 2000):
    from toolloop.tokenizer import ToyMergeTokenizer as RefTok

    from paper_2509_01055_b200 import tokenizer as T

    rng = random.Random(1)
    alphabet = "abcdefghijklmnopqrstuvwxyz <>/\n`=()[]{}.,0123456789"
    texts = []
    for _ in range(n_traj):
        for s in range(2 * rng.randrange(0, 5) + 1):
            n = rng.randrange(200, 1200)
            texts.append("".join(rng.choice(alphabet) for _ in range(n)) + ("</python>" if s % 2 == 0 else ""))
    nbytes = sum(len(t.encode()) for t in texts)
    ref = RefTok()
    t0 = time.perf_counter()
    ref_ids = [ref.encode(t) for t in texts]
    t_ref = time.perf_counter() - t0
    tok = T.ToyMergeTokenizer()
    res = {}
    for nt in (1, 0):
        tok.encode_segments(texts[:10], n_threads=nt)
        t0 = time.perf_counter()
        pool, off, lens = tok.encode_segments(texts, n_threads=nt)
        res[nt] = time.perf_counter() - t0
    assert all(pool[o:o + n].tolist() == r for o, n, r in zip(off, lens, ref_ids))
    ntok = int(sum(len(r) for r in ref_ids))
    import os
    print(f"{len(texts)} segments, {nbytes / 1e6:.1f} MB text, {ntok / 1e6:.2f} M tokens")
    print(f"reference ToyMergeTokenizer.encode (Python, 1 core): {t_ref:.2f} s  ({ntok / t_ref / 1e6:.2f} M tok/s)")
    print(f"native, 1 thread: {res[1]:.3f} s  ({ntok / res[1] / 1e6:.1f} M tok/s, x{t_ref / res[1]:.0f})")
    print(f"native, {os.cpu_count()} threads: {res[0]:.3f} s  ({ntok / res[0] / 1e6:.1f} M tok/s, x{t_ref / res[0]:.0f})")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2000)
