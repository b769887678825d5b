"""Python restatement of the reference's episode-log / sidecar readers
(TEST INFRASTRUCTURE ONLY — the product path is the C++ ingest,
csrc/ingest.cpp, tl_ingest_*).  The checker the ingest tests compare the
C++ reader against; follows /root/reference/pkg/src/toolloop/:
  read_episodes   rollout/episodes.py:132-147 (+ EpisodeRecord.from_dict :95-120)
  flat_logps      cli.py:233-252 (_flat_logps)
  read_sidecar    cli.py:255-269 (_read_sidecar)
"""

from __future__ import annotations

import json
from pathlib import Path

from paper_2509_01055_b200.errors import EpisodeLogError, MaskMismatch
from paper_2509_01055_b200.trajectory import ACTION, trajectory_from_dict


def read_episodes(path) -> list[dict]:
    """rollout/episodes.py:132-147 — one record per non-blank line; any defect
    raises EpisodeLogError citing path:line."""
    path = Path(path)
    out = []
    with path.open("r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            if not line.strip():
                continue
            try:
                data = json.loads(line)
                traj = trajectory_from_dict(data["trajectory"])
                timings = data["timings"]
                if len(timings) != len(traj.segments):
                    raise ValueError(f"timings has {len(timings)} entries for "
                                     f"{len(traj.segments)} segments")
                logps = data.get("action_logprobs")
                if logps is not None:
                    logps = [[float(x) for x in row] for row in logps]
                out.append({"task_id": str(data["task_id"]), "reward": float(data["reward"]),
                            "trajectory": traj, "action_logprobs": logps})
            except EpisodeLogError:
                raise
            except Exception as exc:
                raise EpisodeLogError(f"{path}:{lineno}: {exc}") from exc
    return out


def flat_logps(record: dict) -> list[float]:
    """cli.py:233-252 — per-action-segment rows expanded to per-token logps,
    0.0 on observation positions."""
    if record["action_logprobs"] is None:
        raise MaskMismatch(f"episode {record['task_id']!r} has no action_logprobs; supply --logprobs")
    flat: list[float] = []
    rows = iter(record["action_logprobs"])
    for seg in record["trajectory"].segments:
        if seg.origin == ACTION:
            row = next(rows, None)
            if row is None or len(row) != len(seg.tokens):
                raise MaskMismatch(f"episode {record['task_id']!r}: action_logprobs do not align "
                                   f"with action segments")
            flat.extend(row)
        else:
            flat.extend(0.0 for _ in seg.tokens)
    return flat


def read_sidecar(path: Path, count: int) -> list[dict]:
    """cli.py:255-269."""
    rows = []
    for lineno, line in enumerate(path.read_text(encoding="utf-8").splitlines(), start=1):
        if not line.strip():
            continue
        try:
            data = json.loads(line)
        except json.JSONDecodeError as exc:
            raise EpisodeLogError(f"{path}:{lineno}: {exc}")
        if not isinstance(data, dict) or "logp_new" not in data:
            raise EpisodeLogError(f"{path}:{lineno}: expected an object with 'logp_new'")
        rows.append(data)
    if len(rows) != count:
        raise MaskMismatch(f"{path}: {len(rows)} sidecar rows for {count} episodes")
    return rows
