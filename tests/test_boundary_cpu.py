"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every symbol include/toolloop_b200.h declares; host-side validation
raises the reference's exception types before any launch; the product path
fails loudly without a GPU (no CPU fallback)."""

import re
from pathlib import Path

import numpy as np
import pytest

from conftest import cuda_available

ROOT = Path(__file__).resolve().parents[1]


def _header_symbols():
    text = (ROOT / "include" / "toolloop_b200.h").read_text()
    return sorted(set(re.findall(r"\b(tl_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2509_01055_b200 import _lib

    lib = _lib.load(require_device=False)
    syms = _header_symbols()
    assert syms, "no declarations parsed"
    for s in syms:
        assert hasattr(lib, s), f"missing export {s}"
    assert set(syms) == set(_lib.EXPORTS)
    assert lib.tl_abi_version() == _lib.TL_ABI_VERSION == 4
    assert lib.tl_launch_count() >= 0


def test_workspace_queries_are_host_only():
    from paper_2509_01055_b200 import _lib

    lib = _lib.load(require_device=False)
    assert lib.tl_pack_workspace_bytes(10, 100) > 0
    assert lib.tl_loss_f64_workspace_bytes(1000) >= 1000 * 25
    big = lib.tl_lmhead_workspace_bytes(37888, 3584, 152064, 6_000_000, 2048, 256)
    assert big > 37888 * 152064 * 2  # holds the bf16 dS chunk
    # forward-only (F3) workspace: no dS chunk, ~ the gathered rows only
    fwd = lib.tl_lmhead_logprobs_workspace_bytes(4 * 37888, 3584, 152064)
    assert 4 * 37888 * 3584 * 2 <= fwd < 4 * 37888 * 3584 * 2 * 1.1


def test_config_validation_matches_reference():
    from paper_2509_01055_b200.rl.loss import LossConfig

    with pytest.raises(ValueError):
        LossConfig(epsilon_clip=0.0)
    with pytest.raises(ValueError):
        LossConfig(kl_beta=-0.1)
    with pytest.raises(ValueError):
        LossConfig(std_floor=0.0)
    with pytest.raises(ValueError):
        LossConfig(loss_agg="nope")


def test_host_validation_errors():
    from paper_2509_01055_b200.errors import GroupTooSmall, MaskMismatch
    from paper_2509_01055_b200.rl.loss import GroupBatch, LossConfig, TokenRecord, grpo_multi_turn_loss

    with pytest.raises(MaskMismatch):
        GroupBatch("g", [[TokenRecord(0, -1.0, -1.0, 1)]], [1.0, 2.0])
    batch = GroupBatch("g", [[TokenRecord(0, -1.0, -1.0, 1)]], [0.0])
    with pytest.raises(MaskMismatch):
        grpo_multi_turn_loss(batch, [1.0, 2.0], LossConfig())
    with pytest.raises(GroupTooSmall):
        grpo_multi_turn_loss(GroupBatch("g", [], []), [], LossConfig())


def test_segment_table_layout():
    from paper_2509_01055_b200.packing import segment_table
    from paper_2509_01055_b200.trajectory import Segment, Trajectory

    t1 = Trajectory([Segment("action", "", [1, 2]), Segment("observation", "", [3]),
                     Segment("action", "", [4])])
    t2 = Trajectory([Segment("action", "", [])])
    tab = segment_table([t1, t2, Trajectory()])
    assert tab.token_pool.tolist() == [1, 2, 3, 4]
    assert tab.seg_len.tolist() == [2, 1, 1, 0]
    assert tab.seg_is_action.tolist() == [1, 0, 1, 1]
    assert tab.traj_seg_off.tolist() == [0, 3, 4, 4]
    assert tab.n_tokens == 4 and tab.n_act == 3
    assert tab.traj_lengths().tolist() == [4, 0, 0]
    tab.validate(vocab=5)
    with pytest.raises(ValueError):
        tab.validate(vocab=4)


@pytest.mark.skipif(cuda_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    from paper_2509_01055_b200.errors import ExtensionMissing
    from paper_2509_01055_b200.rl.loss import group_advantages

    with pytest.raises(ExtensionMissing):
        group_advantages([1.0, 0.0])


def test_struct_mirrors_match_the_header():
    """ctypes mirrors of the header's structs: same field names, order and
    size as the C declarations (tl_loss_config, tl_step_overlap)."""
    import ctypes

    from paper_2509_01055_b200 import _lib

    text = (ROOT / "include" / "toolloop_b200.h").read_text()
    for cname, py in (("tl_step_overlap", _lib.StepOverlapC), ("tl_loss_config", _lib.LossConfigC)):
        body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (cname, cname), text, re.S).group(1)
        fields = re.findall(r"\b(?:void\s*\*|double|int32_t|float)\s*\*?\s*(\w+)\s*;", body)
        assert fields == [f for f, _ in py._fields_], cname
    assert ctypes.sizeof(_lib.StepOverlapC) == 16
    assert _lib.StepOverlapC.reserve_sms.offset == 8
