"""Pure-Python restatement of the reference's trajectory-to-loss arithmetic.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain Python floats
(IEEE fp64), fixed sequential order, stdlib math only — exactly the number
system of the reference, so fp64 comparisons can be bitwise.

Data shapes used here (deliberately plain, independent of the product):
  segments : list[(origin, tokens)]   origin in {"action", "observation"}
  record   : (token, logp_new, logp_old, action_bit, logp_ref_or_None)

Reference anchors are relative to /root/reference/pkg/src/toolloop/.
"""

from __future__ import annotations

import math
from typing import Sequence

ACTION = "action"
OBSERVATION = "observation"
# rl/loss.py:22-24 — log-ratio clamp before exponentiation.
CLAMP = 20.0


class OracleMaskMismatch(Exception):
    """Mirror of errors.MaskMismatch (errors.py:28)."""


class OracleGroupTooSmall(Exception):
    """Mirror of errors.GroupTooSmall (errors.py:32)."""


# ---------------------------------------------------------------- packing ----

def flatten(segments) -> list[int]:
    """trajectory.py:154-159 — per-segment token lists concatenated in order
    (no re-tokenisation)."""
    ids: list[int] = []
    for _, toks in segments:
        ids += list(toks)
    return ids


def action_mask(segments) -> list[int]:
    """trajectory.py:162-167 — 1 per action token, 0 per observation token."""
    bits: list[int] = []
    for origin, toks in segments:
        bits += [int(origin == ACTION)] * len(toks)
    return bits


def token_records(segments, logp_new, logp_old, logp_ref=None):
    """rl/loss.py:76-100 — zip ids, mask and log-probs; length checks first."""
    ids = flatten(segments)
    bits = action_mask(segments)
    n = len(ids)
    if len(logp_new) != n or len(logp_old) != n:
        raise OracleMaskMismatch(f"{n} tokens vs {len(logp_new)} new / {len(logp_old)} old")
    if logp_ref is not None and len(logp_ref) != n:
        raise OracleMaskMismatch(f"{n} tokens vs {len(logp_ref)} ref")
    out = []
    for j in range(n):
        ref = None if logp_ref is None else float(logp_ref[j])
        out.append((ids[j], float(logp_new[j]), float(logp_old[j]), bits[j], ref))
    return out


# -------------------------------------------------------------- advantage ----

def group_advantages(rewards: Sequence[float], std_floor: float = 1e-6) -> list[float]:
    """rl/loss.py:103-116 — correctly-rounded (fsum) mean and population
    variance, divisor max(std, floor) (the code, not SPEC.md:463's std+floor)."""
    g = len(rewards)
    if g < 2:
        raise OracleGroupTooSmall(f"need >= 2 rewards, got {g}")
    mu = math.fsum(rewards) / g
    var = math.fsum([(x - mu) ** 2 for x in rewards]) / g
    div = max(math.sqrt(var), std_floor)
    return [(x - mu) / div for x in rewards]


# ------------------------------------------------------------ token terms ----

def _clamp(d: float) -> float:
    if d > CLAMP:
        return CLAMP
    if d < -CLAMP:
        return -CLAMP
    return d


def token_ratio(logp_new: float, logp_old: float) -> float:
    """rl/loss.py:119-126."""
    return math.exp(_clamp(logp_new - logp_old))


def k3(logp_ref: float, logp_new: float) -> float:
    """rl/loss.py:139-147 — exp(d) - d - 1 with d = clamp(ref - new)."""
    d = _clamp(logp_ref - logp_new)
    return math.exp(d) - d - 1.0


def _check(trajs, advs):
    """rl/loss.py:129-136."""
    if len(advs) != len(trajs):
        raise OracleMaskMismatch(f"{len(advs)} advantages vs {len(trajs)} trajectories")
    if not trajs:
        raise OracleGroupTooSmall("empty group")


# ----------------------------------------------------------------- losses ----

def multi_turn(trajs, advs, eps: float = 0.2, beta: float = 0.0, eps_high: float | None = None):
    """rl/loss.py:150-201 — masked clipped objective of one group.

    Returns (objective, diag) with diag keys masked_tokens, total_tokens,
    clip_fraction, clamp_count, kl (loss.py:67-73, :194-200).  `eps_high` is the
    build's DAPO clip-higher extension (unpinned; None = reference behaviour).
    """
    _check(trajs, advs)
    lo = 1.0 - eps
    hi = 1.0 + (eps if eps_high is None else eps_high)
    total = 0.0
    masked = total_tokens = clipped = clamps = 0
    kl_sum = 0.0
    for recs, a in zip(trajs, advs):
        total_tokens += len(recs)
        n_act = sum(r[3] for r in recs)
        if n_act == 0:
            continue                        # still counted in G (:193)
        acc = 0.0
        for (_, new, old, bit, ref) in recs:
            if not bit:
                continue
            masked += 1
            d = new - old
            if d > CLAMP or d < -CLAMP:
                clamps += 1
            r = token_ratio(new, old)
            term = min(r * a, min(max(r, lo), hi) * a)
            if (r > hi and a > 0.0) or (r < lo and a < 0.0):
                clipped += 1
            if ref is not None:
                kk = k3(ref, new)
                kl_sum += kk
                term -= beta * kk
            acc += term
        total += acc / n_act
    obj = total / len(trajs)
    diag = {
        "masked_tokens": masked,
        "total_tokens": total_tokens,
        "clip_fraction": clipped / masked if masked else 0.0,
        "clamp_count": clamps,
        "kl": kl_sum / masked if masked else 0.0,
    }
    return obj, diag


def single_turn(trajs, advs, eps: float = 0.2, beta: float = 0.0):
    """rl/loss.py:204-227 — same term, mask ignored, normaliser len(recs)."""
    _check(trajs, advs)
    lo, hi = 1.0 - eps, 1.0 + eps
    total = 0.0
    for recs, a in zip(trajs, advs):
        if not recs:
            continue
        acc = 0.0
        for (_, new, old, _bit, ref) in recs:
            r = token_ratio(new, old)
            term = min(r * a, min(max(r, lo), hi) * a)
            if ref is not None:
                term -= beta * k3(ref, new)
            acc += term
        total += acc / len(recs)
    return total / len(trajs)


def unclipped(trajs, advs, eps: float = 0.2, beta: float = 0.0):
    """rl/loss.py:230-270 — unclipped arm value and d value / d logp_new."""
    _check(trajs, advs)
    g = len(trajs)
    value = 0.0
    grads = []
    for recs, a in zip(trajs, advs):
        row = [0.0] * len(recs)
        grads.append(row)
        n_act = sum(r[3] for r in recs)
        if n_act == 0:
            continue
        scale = 1.0 / (n_act * g)
        acc = 0.0
        for t, (_, new, old, bit, ref) in enumerate(recs):
            if not bit:
                continue
            d = new - old
            r = token_ratio(new, old)
            term = r * a
            grad = 0.0 if (d > CLAMP or d < -CLAMP) else r * a
            if ref is not None:
                e = ref - new
                if -CLAMP <= e <= CLAMP:
                    term -= beta * (math.exp(e) - e - 1.0)
                    grad += beta * (math.exp(e) - 1.0)
                else:
                    ec = _clamp(e)
                    term -= beta * (math.exp(ec) - ec - 1.0)
            acc += term
            row[t] = grad * scale
        value += acc / n_act
    return value / g, grads


def clipped_grad(trajs, advs, eps: float = 0.2, beta: float = 0.0, eps_high: float | None = None):
    """Gradient of multi_turn's objective w.r.t. logp_new (build restatement,
    parity unpinned: the reference only differentiates the unclipped arm,
    loss.py:230-270).  The min selects the r*A arm when r*A <= clip(r)*A
    (derivative r*A), else the constant clip arm (0); clamped ratio -> 0; the
    k3 term contributes beta*(exp(d)-1) inside the clamp window."""
    _check(trajs, advs)
    lo = 1.0 - eps
    hi = 1.0 + (eps if eps_high is None else eps_high)
    g = len(trajs)
    grads = []
    for recs, a in zip(trajs, advs):
        row = [0.0] * len(recs)
        grads.append(row)
        n_act = sum(r[3] for r in recs)
        if n_act == 0:
            continue
        scale = 1.0 / (n_act * g)
        for t, (_, new, old, bit, ref) in enumerate(recs):
            if not bit:
                continue
            d = new - old
            r = token_ratio(new, old)
            unclipped_arm = r * a
            clip_arm = min(max(r, lo), hi) * a
            gr = 0.0
            if not (d > CLAMP or d < -CLAMP) and unclipped_arm <= clip_arm:
                gr = r * a
            if ref is not None:
                e = ref - new
                if -CLAMP <= e <= CLAMP:
                    gr += beta * (math.exp(e) - 1.0)
            row[t] = gr * scale
    return grads


def term_and_grad(new, old, ref, a, eps: float = 0.2, beta: float = 0.0,
                  eps_high: float | None = None):
    """One action token's A11 term (loss.py:179-190) and d term / d logp_new
    (clipped-arm restatement, as clipped_grad without the 1/(n_i G) scale)."""
    lo = 1.0 - eps
    hi = 1.0 + (eps if eps_high is None else eps_high)
    d = new - old
    r = token_ratio(new, old)
    ua, ca = r * a, min(max(r, lo), hi) * a
    term = min(ua, ca)
    g = r * a if (not (d > CLAMP or d < -CLAMP) and ua <= ca) else 0.0
    if ref is not None:
        term -= beta * k3(ref, new)
        e = ref - new
        if -CLAMP <= e <= CLAMP:
            g += beta * (math.exp(e) - 1.0)
    return term, g


def token_mean(trajs_by_group, advs_by_group, eps: float = 0.2, beta: float = 0.0,
               eps_high: float | None = None):
    """DAPO token-mean aggregation (build extension, parity unpinned; SPEC.md:500
    lists it as a reference non-goal): objective = sum of A11 per-token terms
    over every action token of the batch / number of action tokens."""
    lo = 1.0 - eps
    hi = 1.0 + (eps if eps_high is None else eps_high)
    s = 0.0
    n = 0
    for trajs, advs in zip(trajs_by_group, advs_by_group):
        for recs, a in zip(trajs, advs):
            for (_, new, old, bit, ref) in recs:
                if not bit:
                    continue
                r = token_ratio(new, old)
                term = min(r * a, min(max(r, lo), hi) * a)
                if ref is not None:
                    term -= beta * k3(ref, new)
                s += term
                n += 1
    return (s / n if n else 0.0), n


# ---------------------------------------------------- batch aggregation ----

def loss_report(groups, eps: float = 0.2, beta: float = 0.0, std_floor: float = 1e-6):
    """cli.py:309-344 — per-group advantages + multi_turn, aggregated.

    `groups` is a list of (records_per_trajectory, rewards) in first-appearance
    order of task_id (cli.py:309-311).
    """
    obj_sum = 0.0
    masked_total = 0
    clip_w = 0.0
    kl_w = 0.0
    for trajs, rewards in groups:
        if len(trajs) != len(rewards):
            raise OracleMaskMismatch("trajectories vs rewards")
        advs = group_advantages(rewards, std_floor)
        obj, diag = multi_turn(trajs, advs, eps, beta)
        obj_sum += obj
        masked_total += diag["masked_tokens"]
        clip_w += diag["clip_fraction"] * diag["masked_tokens"]
        kl_w += diag["kl"] * diag["masked_tokens"]
    return {
        "objective": obj_sum / len(groups),
        "clip_fraction": clip_w / masked_total if masked_total else 0.0,
        "masked_tokens": masked_total,
        "kl": kl_w / masked_total if masked_total else 0.0,
        "groups": len(groups),
        "episodes": sum(len(t) for t, _ in groups),
    }


def flat_logps(segments, action_logprobs):
    """cli.py:233-252 — per-action-segment rows expanded to per-token logps,
    0.0 on observation positions."""
    out: list[float] = []
    rows = iter(action_logprobs)
    for origin, toks in segments:
        if origin == ACTION:
            row = next(rows, None)
            if row is None or len(row) != len(toks):
                raise OracleMaskMismatch("action_logprobs do not align with action segments")
            out += [float(x) for x in row]
        else:
            out += [0.0] * len(toks)
    return out
