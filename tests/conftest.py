import json
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run under gpurun)")


def fx(s):
    """Decode a float.hex() fixture entry (None passes through)."""
    return None if s is None else float.fromhex(s)


def load_golden(name: str):
    return json.loads((GOLDEN / name).read_text())


def decode_records(traj):
    """[[tok, new_hex, old_hex, bit, ref_hex|None], ...] -> oracle tuples."""
    return [(t, fx(n), fx(o), b, fx(r)) for (t, n, o, b, r) in traj]


@pytest.fixture(scope="session")
def golden_losses():
    return load_golden("losses.json")


@pytest.fixture(scope="session")
def golden_adv():
    return load_golden("advantages.json")


@pytest.fixture(scope="session")
def golden_pack():
    return load_golden("pack.json")


@pytest.fixture(scope="session")
def golden_cli():
    return load_golden("cli_report.json")


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False
