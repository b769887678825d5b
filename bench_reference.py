"""bench.py's reference arm and CPU baseline: the reference's own CPU path of
the trajectory-to-loss step, timed on the host cores of the box.

Loss path (pack + advantage + masked clipped surrogate) — the UNMODIFIED
reference package `toolloop`, installed into baseline/_ref/ by
tools/install_reference.sh, through its public API exactly as `toolloop
loss` drives it (cli.py:292-328): per group, `token_records` per trajectory
(flatten + action_mask + zip, rl/loss.py:76-100) -> `group_advantages`
(:103-116) -> `grpo_multi_turn_loss` (:150-201) on a `GroupBatch`, then the
cli aggregation sum_g obj_g / n_groups (cli.py:337-344).  Timed
  (i)  single process (the reference is single-threaded), and
  (ii) fanned out over every host core by group, one worker process per core
       (groups are safe to evaluate in parallel); each worker
       builds its groups' inputs before the clock starts, the wall time from
       "go" to the last result is the fan-out time.
LM head (logp_new, entropy and their gradient): the reference has no LM head
(the policy supplies log-probs, rollout/policy.py:25-28), so
its CPU cost is a torch fp32 restatement of the same equations as
oracle/lmhead_oracle.py — z = h W^T once per row block, log-sum-exp, p,
dZ = g (onehot - p) - c p (z - E_p z), dH = dZ W, dW += dZ^T h: 6 H V FLOPs
per action token, on all host cores (torch threads = cores), its achieved
GFLOP/s stated.

A step of this arm is a bounded sample of the configured workload: groups
for the loss path, a block of action rows for the LM head; tokens/s for the
whole workload is extrapolated from the per-token costs (loss path per
packed token fanned out, LM head per action token), and the full step's
time at that rate is reported as `extrapolated_step_ms`.
"""

from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
REF_DIR = ROOT / "baseline" / "_ref"


def load_reference():
    """(toolloop.rl.loss, toolloop.trajectory) of the installed reference, or
    — when baseline/_ref is absent — the same API over the oracle's
    restatement of those functions (kind "port")."""
    if (REF_DIR / "toolloop").is_dir():
        if str(REF_DIR) not in sys.path:
            sys.path.insert(0, str(REF_DIR))
        import toolloop.rl.loss as L
        import toolloop.trajectory as T

        return L, T
    return _port()


def reference_kind() -> str:
    return "reference" if (REF_DIR / "toolloop").is_dir() else "port"


def _port():
    import types
    from dataclasses import dataclass, field

    if str(ROOT) not in sys.path:
        sys.path.insert(0, str(ROOT))
    from oracle import grpo_oracle as O

    @dataclass
    class Segment:
        origin: str
        text: str
        tokens: list

    @dataclass
    class Trajectory:
        segments: list = field(default_factory=list)

    @dataclass(frozen=True)
    class LossConfig:
        epsilon_clip: float = 0.2
        kl_beta: float = 0.0
        std_floor: float = 1e-6

    @dataclass
    class GroupBatch:
        group_id: str
        trajectories: list
        rewards: list

    def token_records(traj, new, old, ref=None):
        return O.token_records([(s.origin, s.tokens) for s in traj.segments], new, old, ref)

    def grpo_multi_turn_loss(batch, adv, cfg):
        obj, d = O.multi_turn(batch.trajectories, adv, cfg.epsilon_clip, cfg.kl_beta)
        return obj, types.SimpleNamespace(**d)

    L = types.SimpleNamespace(LossConfig=LossConfig, GroupBatch=GroupBatch,
                              token_records=token_records, group_advantages=O.group_advantages,
                              grpo_multi_turn_loss=grpo_multi_turn_loss)
    return L, types.SimpleNamespace(Segment=Segment, Trajectory=Trajectory)


def n_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip() + f" x{n_cores()}"
    except OSError:
        pass
    return f"{n_cores()} cpus"


# ---------------------------------------------------------------- loss path --
def group_inputs(cfg, gid: int, ref):
    """One group of the synthetic workload as the reference's own objects:
    Trajectory/Segment lists plus per-token log-prob lists and rewards
    (logp_new = logp_old + N(0, 0.05): the LM head's output, costed
    separately)."""
    from paper_2509_01055_b200.synthetic import make_workload

    L, T = ref
    wl = make_workload(cfg, group_ids=[gid])
    tab = wl.table
    rng = np.random.default_rng([7, gid])
    new = (wl.logp_old + rng.normal(0, 0.05, wl.n_tokens)).astype(np.float64)
    trajs, pos = [], 0
    for b in range(tab.n_traj):
        segs = []
        for s in range(tab.traj_seg_off[b], tab.traj_seg_off[b + 1]):
            o, n = int(tab.seg_src_off[s]), int(tab.seg_len[s])
            segs.append(T.Segment("action" if tab.seg_is_action[s] else "observation", "",
                                  tab.token_pool[o:o + n].tolist()))
        n_b = sum(len(s.tokens) for s in segs)
        trajs.append((T.Trajectory(segments=segs), new[pos:pos + n_b].tolist(),
                      wl.logp_old[pos:pos + n_b].astype(np.float64).tolist(),
                      wl.logp_ref[pos:pos + n_b].astype(np.float64).tolist()))
        pos += n_b
    return {"gid": gid, "trajs": trajs, "rewards": wl.rewards.tolist(), "tokens": wl.n_tokens,
            "act": wl.n_act}


def run_groups(groups, ref, eps=0.2, beta=0.04):
    """The reference path (cli.py:292-328) over prepared groups -> (sum of
    group objectives, masked tokens)."""
    L, _ = ref
    lc = L.LossConfig(epsilon_clip=eps, kl_beta=beta)
    obj, masked = 0.0, 0
    for g in groups:
        recs = [L.token_records(tr, new, old, lref) for tr, new, old, lref in g["trajs"]]
        adv = L.group_advantages(g["rewards"], lc.std_floor)
        o, d = L.grpo_multi_turn_loss(L.GroupBatch(str(g["gid"]), recs, g["rewards"]), adv, lc)
        obj += o
        masked += d.masked_tokens
    return obj, masked


def _worker(conn, cfg, gids):
    ref = load_reference()
    groups = [group_inputs(cfg, g, ref) for g in gids]
    conn.send("ready")
    while conn.recv() == "go":
        t0 = time.perf_counter()
        obj, masked = run_groups(groups, ref)
        conn.send((time.perf_counter() - t0, obj, masked, sum(g["tokens"] for g in groups)))
    conn.close()


class FanOut:
    """One worker process per host core, each owning `per_worker` whole
    groups (inputs built before timing)."""

    def __init__(self, cfg, per_worker: int = 2, first_group: int = 0):
        import multiprocessing as mp

        ctx = mp.get_context("spawn")
        self.n = n_cores()
        self.procs, self.conns = [], []
        for w in range(self.n):
            a, b = ctx.Pipe()
            gids = [(first_group + w * per_worker + k) % cfg.prompts for k in range(per_worker)]
            p = ctx.Process(target=_worker, args=(b, cfg, gids), daemon=True)
            p.start()
            self.procs.append(p)
            self.conns.append(a)
        for c in self.conns:
            assert c.recv() == "ready"

    def run(self):
        """-> (wall s, packed tokens, masked tokens)."""
        t0 = time.perf_counter()
        for c in self.conns:
            c.send("go")
        res = [c.recv() for c in self.conns]
        wall = time.perf_counter() - t0
        return wall, sum(r[3] for r in res), sum(r[2] for r in res)

    def close(self):
        for c in self.conns:
            try:
                c.send("stop")
            except (BrokenPipeError, OSError):
                pass
        for p in self.procs:
            p.join(timeout=10)


# ------------------------------------------------------------------ LM head --
def lmhead_cpu(h, W, y, g, c, chunk: int = 256):
    """fp32 CPU LM head forward + backward (oracle/lmhead_oracle.py's
    equations; logits formed once per row block).  h [n, H], W [V, H] fp32
    torch tensors; g, c [n] upstream grads.  Returns (logp, dH, dW)."""
    import torch

    n = h.shape[0]
    logp = torch.empty(n)
    dH = torch.empty_like(h)
    dW = torch.zeros_like(W)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        hs = h[s:e]
        z = hs @ W.T
        lse = torch.logsumexp(z, 1, keepdim=True)
        p = torch.exp(z - lse)
        ez = (p * z).sum(1, keepdim=True)
        idx = torch.arange(e - s)
        logp[s:e] = z[idx, y[s:e]] - lse[:, 0]
        dz = p.mul_(-g[s:e, None] - c[s:e, None] * (z - ez))
        dz[idx, y[s:e]] += g[s:e]
        dH[s:e] = dz @ W
        dW.addmm_(dz.T, hs)
    return logp, dH, dW


class LmHeadCPU:
    def __init__(self, H: int, V: int, seed: int = 7):
        import torch

        torch.set_num_threads(n_cores())
        gen = torch.Generator().manual_seed(seed)
        self.W = (torch.randn((V, H), generator=gen) * 0.02).bfloat16().float()
        self.H, self.V = H, V
        self.gen = gen

    def run(self, n: int) -> float:
        """Seconds for fwd + bwd over n action rows."""
        import torch

        h = torch.randn((n, self.H), generator=self.gen).bfloat16().float()
        y = torch.randint(0, self.V, (n,), generator=self.gen)
        g = torch.randn(n, generator=self.gen) * 1e-3
        c = torch.full((n,), -1e-6)
        t0 = time.perf_counter()
        lmhead_cpu(h, self.W, y, g, c)
        return time.perf_counter() - t0


# ------------------------------------------------------------- one sample --
class ReferenceSampler:
    """Times the reference's CPU path on bounded samples of `cfg`."""

    def __init__(self, cfg, lm_rows: int = 1024, loss_groups: int = 2):
        self.cfg = cfg
        self.ref = load_reference()
        self.kind = reference_kind()
        self.lm_rows = lm_rows
        self.loss_groups = [group_inputs(cfg, g, self.ref) for g in range(loss_groups)]
        self.fan = FanOut(cfg)
        self.lm = LmHeadCPU(cfg.hidden, cfg.vocab)
        from paper_2509_01055_b200.synthetic import group_act_tokens, group_tokens

        gids = np.arange(cfg.prompts)
        self.T = int(group_tokens(cfg, gids).sum())
        self.T_act = int(group_act_tokens(cfg, gids).sum())

    def step(self, lm_rows: int | None = None) -> dict:
        lm_rows = lm_rows or self.lm_rows
        out = {}
        t0 = time.perf_counter()
        run_groups(self.loss_groups, self.ref)
        t1 = time.perf_counter() - t0
        tok1 = sum(g["tokens"] for g in self.loss_groups)
        fw, ftok, _ = self.fan.run()
        out.update(loss_single_tok_s=tok1 / t1, loss_fanout_tok_s=ftok / fw,
                   loss_sample=f"{len(self.loss_groups)} groups / {tok1} tokens single-process; "
                               f"{self.fan.n} workers x 2 groups / {ftok} tokens fanned out")
        t_lm = self.lm.run(lm_rows)
        flops = 6.0 * lm_rows * self.cfg.hidden * self.cfg.vocab
        out.update(lm_rows=lm_rows, lm_s=t_lm, lm_gflops=flops / t_lm / 1e9,
                   lm_act_tok_s=lm_rows / t_lm)
        # whole-workload rate: fanned-out loss path per packed token, then the
        # LM head per action token (both phases use every core)
        per_tok = 1.0 / out["loss_fanout_tok_s"] + (self.T_act / self.T) / out["lm_act_tok_s"]
        out["value"] = 1.0 / per_tok
        out["extrapolated_step_ms"] = self.T * per_tok * 1e3
        return out

    def describe(self, s: dict) -> str:
        return (f"{'unmodified reference toolloop (baseline/_ref)' if self.kind == 'reference' else 'oracle port'}"
                f" loss path: {s['loss_sample']}: {s['loss_single_tok_s']:.3g} tok/s on 1 core, "
                f"{s['loss_fanout_tok_s']:.3g} tok/s on {n_cores()} cores; LM head (absent from the "
                f"reference; torch fp32 CPU restatement, 6HV FLOP/token) on {s['lm_rows']} action rows "
                f"at H={self.cfg.hidden} V={self.cfg.vocab}: {s['lm_s']:.2f} s = {s['lm_gflops']:.0f} "
                f"GFLOP/s on {n_cores()} threads; tokens/s extrapolated to the {self.T}-token step "
                f"(f_act {self.T_act / self.T:.3f}): {s['extrapolated_step_ms'] / 3.6e6:.2f} h per step")

    def close(self):
        if self.fan is not None:
            self.fan.close()
