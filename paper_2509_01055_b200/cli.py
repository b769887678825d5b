"""`loss` command — drop-in for `toolloop loss` (toolloop/cli.py:272-345).

    python -m paper_2509_01055_b200.cli loss --episodes E [--logprobs S] [--config C]

Reads the episode log (JSON lines, rollout/episodes.py:132-147) and an
optional log-prob sidecar (cli.py:255-269), packs every trajectory on the GPU
(K1), computes group advantages (K2) and the masked clipped objective (K3)
with the fp64 parity kernels for all task_id groups at once, and prints the
same JSON report as the reference (objective, clip_fraction, masked_tokens,
kl, groups, episodes).  Errors exit 1 with the reference's messages
(GroupTooSmall gets the "--samples" hint, cli.py:329-333).
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

from .errors import EpisodeLogError, GroupTooSmall, MaskMismatch

_LOSS_KEYS = {"epsilon_clip", "kl_beta", "std_floor"}


def load_loss_config(path):
    from .rl.loss import LossConfig

    if path is None:
        return LossConfig()
    import yaml

    data = yaml.safe_load(Path(path).read_text(encoding="utf-8")) or {}
    sec = data.get("loss", {}) or {}
    bad = set(sec) - _LOSS_KEYS
    if bad:
        raise ValueError(f"unknown loss config keys: {sorted(bad)}")
    return LossConfig(**sec)


def loss_report(episodes_path, logprobs_path=None, config_path=None) -> dict:
    """Episode log (+ sidecar) -> native ingest (F1, C++) -> K1 pack -> K2
    advantages -> K3 fp64 loss -> cli.loss report."""
    import torch

    from . import grpo, packing
    from .ingest import ingest

    cfg = load_loss_config(config_path)
    b = ingest(episodes_path, logprobs_path, pinned=True)
    sizes = np.diff(b.group_off)
    if np.any(sizes < 2):
        raise GroupTooSmall(f"need at least 2 rewards, got {int(sizes[np.argmax(sizes < 2)])}")
    packed = packing.pack_table(b.table)
    d = lambda a: torch.from_numpy(a if len(a) else np.zeros(1)).to("cuda", non_blocking=True)  # noqa: E731
    lref = None if b.logp_ref is None else d(b.logp_ref)
    rep = grpo.report_f64(packed, b.group_off, b.rewards, d(b.logp_new), d(b.logp_old), lref, cfg)
    return {"objective": rep["objective"], "clip_fraction": rep["clip_fraction"],
            "masked_tokens": rep["masked_tokens"], "kl": rep["kl"], "groups": rep["groups"],
            "episodes": rep["episodes"]}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="toolloop-b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    lp = sub.add_parser("loss", help="masked clipped objective over an episode log; print JSON")
    lp.add_argument("--episodes", required=True)
    lp.add_argument("--logprobs", default=None)
    lp.add_argument("--config", default=None)
    args = ap.parse_args(argv)
    if not Path(args.episodes).is_file():
        print(f"Error: episodes file {args.episodes!r} does not exist", file=sys.stderr)
        return 2
    try:
        report = loss_report(args.episodes, args.logprobs, args.config)
    except GroupTooSmall as exc:
        print(f"Error: {exc}; groups need at least 2 episodes per task_id "
              f"(roll out with --samples 2 or more)")
        return 1
    except (MaskMismatch, EpisodeLogError, ValueError) as exc:
        print(f"Error: {exc}")
        return 1
    print(json.dumps(report, indent=2))
    return 0


if __name__ == "__main__":
    sys.exit(main())
