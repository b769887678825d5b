"""End-to-end `loss` over an episode log: native ingest + GPU kernels
(paper_2509_01055_b200.cli) vs the reference's CPU path (oracle port of
read_episodes -> token_records -> group_advantages -> grpo_multi_turn_loss ->
aggregation, pure Python, as `toolloop loss` runs).  Synthetic C2-shaped
episodes written as the reference's JSONL schema + a log-prob sidecar."""

import json
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import grpo_oracle as O  # noqa: E402
from paper_2509_01055_b200 import cli  # noqa: E402
from paper_2509_01055_b200.synthetic import CONFIGS, make_workload  # noqa: E402


def write_log(wl, d: Path):
    tab = wl.table
    ep, sc = d / "ep.jsonl", d / "sc.jsonl"
    pos = 0
    with ep.open("w") as fe, sc.open("w") as fs:
        for g in range(len(wl.group_off) - 1):
            for b in range(wl.group_off[g], wl.group_off[g + 1]):
                segs, alog = [], []
                n_tok = 0
                for s in range(tab.traj_seg_off[b], tab.traj_seg_off[b + 1]):
                    o, n = int(tab.seg_src_off[s]), int(tab.seg_len[s])
                    toks = tab.token_pool[o:o + n].tolist()
                    origin = "action" if tab.seg_is_action[s] else "observation"
                    segs.append({"origin": origin, "text": "", "tokens": toks})
                    if origin == "action":
                        alog.append(wl.logp_old[pos + n_tok:pos + n_tok + n].tolist())
                    n_tok += n
                turns = sum(1 for s in segs if s["origin"] == "observation")
                rec = {"task_id": f"task{int(wl.group_ids[g])}", "policy_id": "p",
                       "trajectory": {"segments": segs, "turn_count": turns, "terminated": True,
                                      "termination_cause": "answer"},
                       "timings": [{} for _ in segs], "reward": float(wl.rewards[b]),
                       "reward_breakdown": {}, "limits": {"max_turns": 6},
                       "answer": None, "prompt_tokens": 0, "action_logprobs": alog}
                fe.write(json.dumps(rec) + "\n")
                new = (wl.logp_old[pos:pos + n_tok] + 0.05).tolist()
                fs.write(json.dumps({"logp_new": new, "logp_old": wl.logp_old[pos:pos + n_tok].tolist(),
                                     "logp_ref": wl.logp_ref[pos:pos + n_tok].tolist()}) + "\n")
                pos += n_tok
    return ep, sc


def reference_cpu(ep, sc, cfg):
    """cli.loss restated in pure Python (oracle), with the reference's JSON parsing."""
    recs = [json.loads(l) for l in ep.read_text().splitlines() if l.strip()]
    side = [json.loads(l) for l in sc.read_text().splitlines() if l.strip()]
    groups, order = {}, []
    for r, s in zip(recs, side):
        segs = [(x["origin"], x["tokens"]) for x in r["trajectory"]["segments"]]
        tr = O.token_records(segs, s["logp_new"], s.get("logp_old", s["logp_new"]), s.get("logp_ref"))
        if r["task_id"] not in groups:
            groups[r["task_id"]] = ([], [])
            order.append(r["task_id"])
        groups[r["task_id"]][0].append(tr)
        groups[r["task_id"]][1].append(float(r["reward"]))
    return O.loss_report([groups[k] for k in order], cfg["eps"], cfg["beta"])


def main():
    n_groups = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    wl = make_workload(CONFIGS["c2"], group_ids=np.arange(n_groups))
    with tempfile.TemporaryDirectory() as d:
        d = Path(d)
        ep, sc = write_log(wl, d)
        cfgp = d / "cfg.yaml"
        cfgp.write_text("loss:\n  epsilon_clip: 0.2\n  kl_beta: 0.04\n")
        mb = (ep.stat().st_size + sc.stat().st_size) / 1e6
        cli.loss_report(ep, sc, cfgp)  # warm-up (CUDA context, build caches)
        t0 = time.perf_counter()
        ours = cli.loss_report(ep, sc, cfgp)
        t_ours = time.perf_counter() - t0
        t0 = time.perf_counter()
        ref = reference_cpu(ep, sc, {"eps": 0.2, "beta": 0.04})
        t_ref = time.perf_counter() - t0
    T = wl.n_tokens
    rel = abs(ours["objective"] - ref["objective"]) / max(abs(ref["objective"]), 1e-300)
    print(json.dumps({"episodes": len(wl.rewards), "tokens": T, "log_MB": round(mb, 1),
                      "ours_s": t_ours, "ours_tok_per_s": T / t_ours,
                      "reference_cpu_s": t_ref, "reference_tok_per_s": T / t_ref,
                      "speedup": t_ref / t_ours, "objective_rel_diff": rel,
                      "masked_equal": ours["masked_tokens"] == ref["masked_tokens"]}))


if __name__ == "__main__":
    main()
