"""F4: the native incremental tokenizer (csrc/tokenize.cpp) against the
reference's golden vectors, its own unit tests (test_tokenizer.py), and the
oracle restatement (oracle/tokenizer_oracle.py).  Host code: runs without a
GPU."""

import json
import random
from pathlib import Path

import numpy as np
import pytest

from oracle import pack_oracle as P
from oracle import tokenizer_oracle as TO
from paper_2509_01055_b200 import tokenizer as T

GOLD = json.loads((Path(__file__).parent / "golden" / "tokenizer.json").read_text())


def _tok(table):
    m = GOLD["tables"][table]
    return T.ToyMergeTokenizer() if m is None else T.ToyMergeTokenizer([tuple(x) for x in m])


def _merges(table):
    m = GOLD["tables"][table]
    return TO.DEFAULT_MERGES if m is None else [tuple(x) for x in m]


@pytest.fixture
def tok():
    return T.ToyMergeTokenizer()


# --------------------------------------------------- pin the oracle first --
def test_oracle_matches_reference_golden():
    for c in GOLD["cases"]:
        m = _merges(c["table"])
        assert TO.encode(c["text"], m) == c["ids"]
        assert TO.tokenize(c["text"], c["cap"], m) == (c["cap_text"], c["cap_ids"])


# ------------------------------------------------ native vs golden vectors --
def test_native_encode_and_cap_golden():
    toks = {i: _tok(i) for i in range(len(GOLD["tables"]))}
    for i, t in toks.items():
        assert t.vocab_size == GOLD["vocab_sizes"][i]
    for c in GOLD["cases"]:
        t = toks[c["table"]]
        assert t.encode(c["text"]) == c["ids"]
        assert T.tokenize(t, c["text"], c["cap"]) == (c["cap_text"], c["cap_ids"])
        assert t.decode(c["ids"]) == c["text"]


def test_native_batch_equals_per_segment_golden():
    for table in range(len(GOLD["tables"])):
        t = _tok(table)
        cases = [c for c in GOLD["cases"] if c["table"] == table]
        pool, off, lens = t.encode_segments([c["text"] for c in cases],
                                            [c["cap"] for c in cases], n_threads=4)
        for c, o, n in zip(cases, off, lens):
            assert pool[o:o + n].tolist() == c["cap_ids"]


def test_rejected_tables_same_error():
    for r in GOLD["rejected"]:
        with pytest.raises(ValueError) as e:
            T.ToyMergeTokenizer([tuple(m) for m in r["merges"]])
        assert str(e.value) == r["error"]


# ------------------------- the reference's own tokenizer tests, restated --
def test_empty_roundtrip(tok):
    assert tok.encode("") == []
    assert tok.decode([]) == ""


def test_vocab_size_counts_merges(tok):
    assert tok.vocab_size == 260


def test_plain_ascii_is_bytes():
    t = T.ToyMergeTokenizer(merges=[])
    assert t.encode("abc") == [97, 98, 99]
    assert t.decode([97, 98, 99]) == "abc"


def test_default_merge_gt_newline(tok):
    assert tok.encode(">\n") == [256]
    assert tok.decode([256]) == ">\n"


def test_merge_pass_is_single_left_to_right():
    t = T.ToyMergeTokenizer(merges=[("a", "b")])
    assert t.encode("aab") == [97, 256]
    assert t.encode("abab") == [256, 256]


def test_later_rule_consumes_earlier_merge():
    t = T.ToyMergeTokenizer(merges=[("a", "b"), ("ab", "c")])
    assert t.encode("abc") == [257]
    assert t.decode([257]) == "abc"


ACTION_TEXT = "x</python>"
OBS_TEXT = "\n<result>ok</result>"
ACTION_IDS = [120, 257, 112, 121, 116, 104, 111, 110, 62]
OBS_IDS = [258, 114, 101, 115, 117, 108, 116, 62, 111, 107, 257, 114, 101, 115, 117, 108, 116, 62]
JOINT_IDS = [120, 257, 112, 121, 116, 104, 111, 110, 256, 60, 114, 101, 115, 117, 108, 116, 62,
             111, 107, 257, 114, 101, 115, 117, 108, 116, 62]


def test_boundary_divergence_witness(tok):
    """test_tokenizer.py:52-65: incremental != joint encoding at the boundary."""
    assert tok.encode(ACTION_TEXT) == ACTION_IDS
    assert tok.encode(OBS_TEXT) == OBS_IDS
    assert tok.encode(ACTION_TEXT + OBS_TEXT) == JOINT_IDS
    assert tok.decode(ACTION_IDS + OBS_IDS) == tok.decode(JOINT_IDS)


def test_encode_decode_roundtrip_fuzz(tok):
    rng = random.Random(7)
    alphabet = "abcdefr <>/\n`otuhpyns"
    for _ in range(500):
        text = "".join(rng.choice(alphabet) for _ in range(rng.randrange(0, 60)))
        assert tok.decode(tok.encode(text)) == text


def test_roundtrip_multibyte(tok):
    text = "π ≈ 3.14159 — naïve café"
    assert tok.decode(tok.encode(text)) == text


def test_decode_out_of_range_raises(tok):
    with pytest.raises(IndexError):
        tok.decode([tok.vocab_size])


# ------------------------------------------ batch -> packer segment table --
def test_segment_table_feeds_the_packer_incrementally(tok):
    """Rollout texts -> SegmentTable in one call: ids per segment are the
    incremental encodings (never the joint one), caps keep leading ids, and
    the CPU restatement of K1 over it gives flatten/action_mask of the
    per-segment token lists; many threads == one thread."""
    rng = random.Random(11)
    alphabet = "abcdefr <>/\n`otuhpyns é"
    trajs, caps = [], []
    for _ in range(200):
        k = rng.randrange(0, 6)
        segs, cs = [], []
        for s in range(2 * k + 1):
            txt = "".join(rng.choice(alphabet) for _ in range(rng.randrange(1 if s == 0 else 0, 80)))
            if s % 2 == 0 and rng.random() < 0.3:
                txt += "</python>"
            if s % 2 == 1 and rng.random() < 0.5:
                txt = "\n<result>" + txt
            segs.append(("action" if s % 2 == 0 else "observation", txt))
            cs.append(rng.choice([None, 5, 30]))
        trajs.append(segs)
        caps.append(cs)
    tab = T.segment_table(tok, trajs, caps, n_threads=8)
    tab1 = T.segment_table(tok, trajs, caps, n_threads=1)
    assert np.array_equal(tab.seg_len, tab1.seg_len)
    expect = []
    i = 0
    for segs, cs in zip(trajs, caps):
        lists = []
        for (origin, txt), cap in zip(segs, cs):
            ids = TO.tokenize(txt, cap)[1]
            o, n = int(tab.seg_src_off[i]), int(tab.seg_len[i])
            assert tab.token_pool[o:o + n].tolist() == ids
            assert tab.seg_is_action[i] == (origin == "action")
            lists.append((origin, ids))
            i += 1
        expect.append(lists)
    ref = P.pack_varlen(expect)
    got = np.concatenate([tab.token_pool[o:o + n] for o, n in zip(tab.seg_src_off, tab.seg_len)])
    assert got.tolist() == ref["input_ids"].tolist()
