"""Parity against the unmodified reference package itself, at a larger scale
than the committed golden vectors.

The reference (`toolloop`, pure Python) is installed into baseline/_ref by
tools/install_reference.sh (git-ignored; it travels to the GPU box with the
snapshot; these tests skip without it).  On 48 random groups of 4-8
multi-turn trajectories (empty segments, all-observation trajectories,
degenerate reward groups, missing reference log-probs) the drop-in operators
are compared with the reference's own functions on the same inputs:

  flatten / action_mask / token ids + mask      bit-exact (K1)
  group_advantages                               <= 2 ulp, >= 95 % bitwise
  grpo_multi_turn_loss objective + diagnostics   rel 1e-12, integers exact
  grpo_single_turn_loss, unclipped_objective     rel 1e-12 (value and gradient)
  cli.loss report (the reference's aggregation,   rel 1e-5 (kl 1e-5 of max(1e-3, kl),
  cli.py:317-344) vs the batched fp32 K3          clip fraction 2e-3), counts exact
(The fp64 CLI report is checked against the reference CLI's own JSON in
tests/test_cli.py.)
"""

import math
import random
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"
if not (REF / "toolloop").is_dir():  # pragma: no cover
    pytest.skip("reference package not installed (tools/install_reference.sh)", allow_module_level=True)
sys.path.insert(0, str(REF))

import toolloop.rl.loss as RL  # noqa: E402
import toolloop.trajectory as RT  # noqa: E402

from paper_2509_01055_b200 import grpo, packing  # noqa: E402
from paper_2509_01055_b200.rl import loss as L  # noqa: E402
from paper_2509_01055_b200.trajectory import Segment, Trajectory  # noqa: E402


def _case(seed=2509, n_groups=48):
    """Per group: segment lists, rewards, per-token logp_new / old / ref (ref
    None for some trajectories)."""
    rng = random.Random(seed)
    groups = []
    for g in range(n_groups):
        G = rng.randrange(4, 9)
        trajs = []
        for _ in range(G):
            segs = []
            for s in range(rng.randrange(0, 5) * 2 + 1):
                n = 0 if rng.random() < 0.1 else rng.randrange(1, 40)
                origin = "action" if s % 2 == 0 else "observation"
                if g % 7 == 3 and origin == "action" and s > 0:
                    origin = "observation"  # some trajectories are nearly all observation
                segs.append((origin, [rng.randrange(0, 50000) for _ in range(n)]))
            n_tok = sum(len(t) for _, t in segs)
            old = [-rng.expovariate(1.0) for _ in range(n_tok)]
            new = [o + rng.gauss(0.0, 0.2) for o in old]
            ref = None if rng.random() < 0.25 else [o + rng.gauss(0.0, 0.05) for o in old]
            trajs.append({"segs": segs, "new": new, "old": old, "ref": ref})
        if g % 5 == 0:
            rewards = [1.0] * G  # degenerate group: zero advantages
        else:
            rewards = [rng.choice([1.0, -1.0, 0.5, 0.0, -1.25]) for _ in range(G)]
        groups.append((trajs, rewards))
    return groups


def _ulps(a, b):
    return 0 if a == b else abs(a - b) / max(math.ulp(a), math.ulp(b))


def _rel(a, b, rel):
    return abs(a - b) <= rel * max(1.0, abs(b))


def _ref_traj(segs):
    return RT.Trajectory([RT.Segment(o, "", list(t)) for o, t in segs])


def _our_traj(segs):
    return Trajectory([Segment(o, "", list(t)) for o, t in segs])


def _records(mod, traj, t):
    return mod.token_records(traj, t["new"], t["old"], t["ref"])


def test_flatten_mask_and_records_match_the_reference():
    groups = _case(7, 12)
    trajs = [t for g, _ in groups for t in g]
    packed = packing.pack([_our_traj(t["segs"]) for t in trajs])
    ids = packed.input_ids.cpu().numpy().tolist()
    mask = packed.loss_mask.cpu().numpy().tolist()
    want_ids, want_mask = [], []
    for t in trajs:
        rt = _ref_traj(t["segs"])
        want_ids += RT.flatten(rt)
        want_mask += RT.action_mask(rt)
        got = _records(L, _our_traj(t["segs"]), t)
        ref = _records(RL, rt, t)
        assert [(r.token, r.action_bit) for r in got] == [(r.token, r.action_bit) for r in ref]
    assert ids == want_ids and mask == want_mask


def test_advantages_and_losses_match_the_reference():
    cfg_ref = RL.LossConfig(epsilon_clip=0.2, kl_beta=0.05)
    cfg = L.LossConfig(epsilon_clip=0.2, kl_beta=0.05)
    n_adv = n_bitwise = 0
    for trajs, rewards in _case():
        adv_ref = RL.group_advantages(rewards, cfg_ref.std_floor)
        adv = L.group_advantages(rewards, cfg.std_floor)
        for a, b in zip(adv, adv_ref):
            assert _ulps(a, b) <= 2
            n_adv += 1
            n_bitwise += a == b
        rb = RL.GroupBatch("g", [_records(RL, _ref_traj(t["segs"]), t) for t in trajs], rewards)
        ob = L.GroupBatch("g", [_records(L, _our_traj(t["segs"]), t) for t in trajs], rewards)
        obj_ref, d_ref = RL.grpo_multi_turn_loss(rb, adv_ref, cfg_ref)
        obj, d = L.grpo_multi_turn_loss(ob, adv_ref, cfg)
        assert _rel(obj, obj_ref, 1e-12), (obj, obj_ref)
        assert (d.masked_tokens, d.total_tokens, d.clamp_count) == \
            (d_ref.masked_tokens, d_ref.total_tokens, d_ref.clamp_count)
        assert _rel(d.clip_fraction, d_ref.clip_fraction, 1e-12)
        assert _rel(d.kl, d_ref.kl, 1e-12)
        # unclipped objective and its per-token gradient (the reference's only gradient)
        u_ref, g_ref = RL.unclipped_objective(rb, adv_ref, cfg_ref)
        u, g = L.unclipped_objective(ob, adv_ref, cfg)
        assert _rel(u, u_ref, 1e-12)
        for row, row_ref in zip(g, g_ref):
            assert len(row) == len(row_ref)
            for x, y in zip(row, row_ref):
                assert abs(x - y) <= 1e-12 * max(abs(y), 1e-12)
        # single-turn objective on all-action copies of the records
        import dataclasses

        sb_ref = RL.GroupBatch("g", [[dataclasses.replace(r, action_bit=1) for r in tr]
                                     for tr in rb.trajectories], rewards)
        sb = L.GroupBatch("g", [[dataclasses.replace(r, action_bit=1) for r in tr]
                                for tr in ob.trajectories], rewards)
        assert _rel(L.grpo_single_turn_loss(sb, adv_ref, cfg),
                    RL.grpo_single_turn_loss(sb_ref, adv_ref, cfg_ref), 1e-12)
    assert n_bitwise >= 0.95 * n_adv


def _ref_report(groups, cfg_ref):
    """The reference's cli.loss aggregation (cli.py:317-344)."""
    objective_sum, masked_total, clipped_weighted, kl_weighted = 0.0, 0, 0.0, 0.0
    for trajs, rewards in groups:
        batch = RL.GroupBatch("g", [_records(RL, _ref_traj(t["segs"]), t) for t in trajs], rewards)
        adv = RL.group_advantages(batch.rewards, cfg_ref.std_floor)
        objective, diag = RL.grpo_multi_turn_loss(batch, adv, cfg_ref)
        objective_sum += objective
        masked_total += diag.masked_tokens
        clipped_weighted += diag.clip_fraction * diag.masked_tokens
        kl_weighted += diag.kl * diag.masked_tokens
    return {"objective": objective_sum / len(groups),
            "clip_fraction": clipped_weighted / masked_total if masked_total else 0.0,
            "masked_tokens": masked_total,
            "kl": kl_weighted / masked_total if masked_total else 0.0,
            "groups": len(groups), "episodes": sum(len(t) for t, _ in groups)}


def test_batched_report_matches_the_reference_cli():
    groups = _case(11)
    cfg_ref = RL.LossConfig(epsilon_clip=0.2, kl_beta=0.05)
    want = _ref_report(groups, cfg_ref)
    trajs = [t for g, _ in groups for t in g]
    rewards = np.array([r for _, rw in groups for r in rw], dtype=np.float64)
    go = np.cumsum([0] + [len(g) for g, _ in groups]).astype(np.int32)
    packed = packing.pack([_our_traj(t["segs"]) for t in trajs])
    lnew = np.concatenate([t["new"] for t in trajs])
    lold = np.concatenate([t["old"] for t in trajs])
    lref = np.concatenate([t["ref"] if t["ref"] is not None else [float("nan")] * len(t["old"])
                           for t in trajs])
    f = lambda a: torch.from_numpy(a.astype(np.float32)).cuda()  # noqa: E731
    rep, _ = grpo.grpo_loss(packed, go, rewards, f(lnew), f(lold), f(lref),
                            L.LossConfig(epsilon_clip=0.2, kl_beta=0.05))
    # the fp32 path sees fp32-rounded log-probs: compare with the reference on those
    groups32 = [([dict(t, new=np.float32(t["new"]).astype(float).tolist(),
                       old=np.float32(t["old"]).astype(float).tolist(),
                       ref=None if t["ref"] is None else np.float32(t["ref"]).astype(float).tolist())
                  for t in g], rw) for g, rw in groups]
    want32 = _ref_report(groups32, cfg_ref)
    assert rep["masked_tokens"] == want32["masked_tokens"] == want["masked_tokens"]
    assert rep["groups"] == want["groups"] and rep["episodes"] == want["episodes"]
    assert _rel(rep["objective"], want32["objective"], 1e-5)
    assert abs(rep["kl"] - want32["kl"]) <= 1e-5 * max(1e-3, abs(want32["kl"]))
    assert abs(rep["clip_fraction"] - want32["clip_fraction"]) <= 2e-3
