"""Generate golden vectors by running the REAL reference (`toolloop`) here.

Run in the build container only (the reference tree does not exist on the
GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/*.json.  Floats are stored as float.hex() strings so
fp64 comparisons against the fixtures can be bitwise.  Every vector is the
output of the reference's own functions:
  toolloop.rl.loss.{group_advantages, grpo_multi_turn_loss,
                    grpo_single_turn_loss, unclipped_objective, token_ratio}
  toolloop.trajectory.{flatten, action_mask} over ToyMergeTokenizer ids
  toolloop.cli `loss` report over an episode log (+ sidecar)
  toolloop.tokenizer.ToyMergeTokenizer / trajectory._tokenize (tokenizer.json;
  `--only tokenizer` regenerates just that file)
"""

from __future__ import annotations

import json
import math
import random
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent

from toolloop.rl.loss import (  # noqa: E402  (reference, this container only)
    GroupBatch,
    LossConfig,
    TokenRecord,
    group_advantages,
    grpo_multi_turn_loss,
    grpo_single_turn_loss,
    token_ratio,
    unclipped_objective,
)
from toolloop.tokenizer import ToyMergeTokenizer  # noqa: E402
from toolloop.trajectory import (  # noqa: E402
    Trajectory,
    action_mask,
    append_action,
    append_observation,
    flatten,
    terminate,
)


def hx(x: float) -> str:
    return float(x).hex()


def enc_recs(recs):
    return [[r.token, hx(r.logp_new), hx(r.logp_old), r.action_bit,
             None if r.logp_ref is None else hx(r.logp_ref)] for r in recs]


# ------------------------------------------------------------- advantages ----

def gen_advantages():
    rng = random.Random(250901055)
    cases = []
    for i in range(400):
        g = rng.randint(2, 64)
        kind = i % 5
        if kind == 0:
            r = [rng.uniform(-5, 5) for _ in range(g)]
        elif kind == 1:      # all-equal non-dyadic (fsum matters)
            v = rng.choice([0.1, 1.1, -1.25, 0.3, 2.0 / 3.0, 1e-7])
            r = [v] * g
        elif kind == 2:      # binary rewards (SWE-style {0,1}, match +-1)
            r = [float(rng.random() < 0.2) for _ in range(g)]
        elif kind == 3:      # math TIR {1, -1.25}
            r = [rng.choice([1.0, -1.25]) for _ in range(g)]
        else:                # wide dynamic range
            r = [rng.uniform(-1, 1) * 10 ** rng.randint(-12, 12) for _ in range(g)]
        floor = 1e-6 if i % 7 else rng.choice([1e-3, 0.5, 1e-12])
        cases.append({"rewards": [hx(x) for x in r], "std_floor": hx(floor),
                      "adv": [hx(a) for a in group_advantages(r, floor)]})
    return cases


# ------------------------------------------------------------------ losses ----

def rand_batch(rng, with_refs, single_turn=False, big=False):
    g = rng.randint(2, 8)
    trajs, rewards = [], []
    for _ in range(g):
        recs = []
        turns = rng.randint(1, 6 if big else 4)
        for _t in range(turns):
            for _ in range(rng.randint(1, 16 if big else 6)):
                recs.append(TokenRecord(rng.randrange(32000), rng.uniform(-3, 0),
                                        rng.uniform(-3, 0), 1,
                                        rng.uniform(-3, 0) if with_refs else None))
            if single_turn:
                continue
            for _ in range(rng.randint(0, 16 if big else 5)):
                recs.append(TokenRecord(rng.randrange(32000), rng.uniform(-50, 50),
                                        rng.uniform(-50, 50), 0,
                                        rng.uniform(-50, 50) if with_refs else None))
        if rng.random() < 0.05 and not single_turn:
            recs = [TokenRecord(r.token, r.logp_new, r.logp_old, 0, r.logp_ref) for r in recs]
        trajs.append(recs)
        rewards.append(rng.choice([rng.uniform(-2, 2), 1.0, -1.0, 0.0]))
    return GroupBatch("g", trajs, rewards)


def gen_losses():
    rng = random.Random(20250901)
    cases = []
    for i in range(160):
        with_refs = i % 2 == 1
        single = i % 5 == 0
        batch = rand_batch(rng, with_refs, single_turn=single, big=(i % 3 == 0))
        # a few tokens with pathological gaps to hit the +-20 clamp
        if i % 4 == 0:
            t = batch.trajectories[0]
            k = rng.randrange(len(t))
            r = t[k]
            t[k] = TokenRecord(r.token, r.logp_new - 60.0 * rng.choice([1, -1]), r.logp_old,
                               r.action_bit, r.logp_ref)
        eps = rng.choice([0.2, 0.1, 0.28, 0.5])
        beta = rng.choice([0.0, 0.1, 0.3]) if with_refs else 0.0
        cfg = LossConfig(epsilon_clip=eps, kl_beta=beta)
        adv = group_advantages(batch.rewards, cfg.std_floor)
        obj, diag = grpo_multi_turn_loss(batch, adv, cfg)
        single_v = grpo_single_turn_loss(batch, adv, cfg)
        uval, ugrads = unclipped_objective(batch, adv, cfg)
        cases.append({
            "eps": hx(eps), "beta": hx(beta),
            "rewards": [hx(x) for x in batch.rewards],
            "adv": [hx(a) for a in adv],
            "trajectories": [enc_recs(t) for t in batch.trajectories],
            "multi": hx(obj),
            "diag": {"masked_tokens": diag.masked_tokens, "total_tokens": diag.total_tokens,
                     "clip_fraction": hx(diag.clip_fraction), "clamp_count": diag.clamp_count,
                     "kl": hx(diag.kl)},
            "single": hx(single_v),
            "unclipped": hx(uval),
            "unclipped_grads": [[hx(g) for g in row] for row in ugrads],
        })
    ratios = []
    for _ in range(200):
        a, b = rng.uniform(-40, 0), rng.uniform(-40, 0)
        ratios.append([hx(a), hx(b), hx(token_ratio(TokenRecord(0, a, b, 1)))])
    return cases, ratios


# ----------------------------------------------------------------- packing ----

def gen_pack():
    tok = ToyMergeTokenizer()
    rng = random.Random(4242)
    alphabet = "abcdefr <>/\n`otuhpyns"
    trajs = []
    for i in range(60):
        traj = Trajectory()
        turns = rng.randint(0, 6)
        for t in range(turns + 1):
            txt = "".join(rng.choice(alphabet) for _ in range(rng.randrange(0, 40)))
            if t == 0 and not txt:
                txt = "x"
            if rng.random() < 0.3:
                txt += "</python>"
            append_action(traj, txt, tok)
            if t < turns:
                obs = "".join(rng.choice(alphabet) for _ in range(rng.randrange(0, 60)))
                if rng.random() < 0.5:
                    obs = "\n" + obs
                append_observation(traj, obs, tok)
        if i % 3 == 0:
            terminate(traj, "answer")
        trajs.append({
            "segments": [[s.origin, list(s.tokens)] for s in traj.segments],
            "flatten": flatten(traj),
            "action_mask": action_mask(traj),
            "joint_encode": tok.encode(traj.text()),
        })
    return trajs


# ------------------------------------------------------------- CLI report ----

def gen_cli_report():
    """Run `toolloop loss` (cli.py:272-345) on a synthetic episode log with a
    sidecar and record its JSON report."""
    from click.testing import CliRunner
    from toolloop.cli import main
    from toolloop.rollout.episodes import EpisodeRecord, RolloutLimits, write_episodes

    rng = random.Random(77)
    tok = ToyMergeTokenizer()
    records, sidecar = [], []
    for p in range(5):
        for s in range(rng.randint(2, 5)):
            traj = Trajectory()
            alog = []
            turns = rng.randint(0, 3)
            for t in range(turns + 1):
                txt = "".join(rng.choice("abc <>/\n") for _ in range(rng.randint(1, 20)))
                seg = append_action(traj, txt, tok)
                alog.append([-abs(rng.gauss(0, 1)) for _ in seg.tokens])
                if t < turns:
                    append_observation(traj, "".join(rng.choice("xyz\n") for _ in range(rng.randint(0, 15))), tok)
            terminate(traj, "answer")
            rec = EpisodeRecord(task_id=f"task{p}", policy_id="scripted", trajectory=traj,
                                timings=[{} for _ in traj.segments],
                                reward=rng.choice([1.0, -1.0, 0.5]), reward_breakdown={},
                                limits=RolloutLimits(), action_logprobs=alog)
            records.append(rec)
            n = len(flatten(traj))
            new = [-abs(rng.gauss(0, 1)) for _ in range(n)]
            old = [x + rng.gauss(0, 0.3) for x in new]
            ref = [x + rng.gauss(0, 0.1) for x in new]
            sidecar.append({"logp_new": new, "logp_old": old, "logp_ref": ref})
    with tempfile.TemporaryDirectory() as d:
        ep = Path(d) / "ep.jsonl"
        sc = Path(d) / "sc.jsonl"
        cfgp = Path(d) / "cfg.yaml"
        write_episodes(ep, records)
        sc.write_text("".join(json.dumps(r) + "\n" for r in sidecar), encoding="utf-8")
        cfgp.write_text("loss:\n  epsilon_clip: 0.2\n  kl_beta: 0.1\n", encoding="utf-8")
        runner = CliRunner()
        out_embedded = runner.invoke(main, ["loss", "--episodes", str(ep)])
        out_sidecar = runner.invoke(main, ["loss", "--episodes", str(ep), "--logprobs", str(sc),
                                           "--config", str(cfgp)])
        assert out_embedded.exit_code == 0, out_embedded.output
        assert out_sidecar.exit_code == 0, out_sidecar.output
        episodes_text = ep.read_text(encoding="utf-8")
    return {
        "episodes_jsonl": episodes_text,
        "sidecar": sidecar,
        "config": {"epsilon_clip": 0.2, "kl_beta": 0.1, "std_floor": 1e-6},
        "report_embedded": json.loads(out_embedded.output),
        "report_sidecar": json.loads(out_sidecar.output),
        "report_sidecar_text": out_sidecar.output,
    }


# --------------------------------------------------------------- tokenizer ----

def gen_tokenizer():
    """ToyMergeTokenizer.encode / decode and trajectory._tokenize (token cap)
    over fuzzed texts (ASCII tool markup + multi-byte characters) for several
    merge tables, plus the tables the reference rejects."""
    from toolloop.trajectory import _tokenize

    rng = random.Random(2509)
    alphabet = "abcdefr <>/\n`otuhpyns" + "πé≈—\u00a0"
    tables = [None, [], [["a", "b"]], [["a", "b"], ["ab", "c"]],
              [["<", "/"], ["</", "r"], ["e", "r"], ["er", ">"], [">", "\n"], ["\n", "\n"]]]
    cases = []
    for ti, merges in enumerate(tables):
        tok = ToyMergeTokenizer() if merges is None else ToyMergeTokenizer([tuple(m) for m in merges])
        for _ in range(150):
            text = "".join(rng.choice(alphabet) for _ in range(rng.randrange(0, 120)))
            cap = rng.choice([None, 0, 1, 3, 10, 40])
            t_text, t_ids = _tokenize(tok, text, cap)
            cases.append({"table": ti, "text": text, "ids": tok.encode(text), "cap": cap,
                          "cap_text": t_text, "cap_ids": t_ids})
        cases.append({"table": ti, "text": "", "ids": tok.encode(""), "cap": None,
                      "cap_text": "", "cap_ids": []})
    rejected = []
    for merges in ([["ab", "c"]], [["a", "b"], ["abc", "d"]], [["é", "a"]]):
        try:
            ToyMergeTokenizer([tuple(m) for m in merges])
        except ValueError as e:
            rejected.append({"merges": merges, "error": str(e)})
    return {"tables": tables, "vocab_sizes": [
        (ToyMergeTokenizer() if m is None else ToyMergeTokenizer([tuple(x) for x in m])).vocab_size
        for m in tables], "cases": cases, "rejected": rejected}


def main() -> None:
    if "--only" in sys.argv:  # regenerate one fixture, leave the others untouched
        which = sys.argv[sys.argv.index("--only") + 1]
        gen = {"tokenizer": gen_tokenizer}[which]
        (HERE / f"{which}.json").write_text(json.dumps(gen()))
        return
    adv = gen_advantages()
    losses, ratios = gen_losses()
    pack = gen_pack()
    cli = gen_cli_report()
    (HERE / "advantages.json").write_text(json.dumps(adv))
    (HERE / "losses.json").write_text(json.dumps({"cases": losses, "ratios": ratios}))
    (HERE / "pack.json").write_text(json.dumps(pack))
    (HERE / "cli_report.json").write_text(json.dumps(cli))
    (HERE / "tokenizer.json").write_text(json.dumps(gen_tokenizer()))
    for p in sorted(HERE.glob("*.json")):
        print(p.name, p.stat().st_size, "bytes", file=sys.stderr)


if __name__ == "__main__":
    main()
