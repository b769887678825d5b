"""Drop-in for toolloop.tokenizer (F4): the byte-level
ordered-merge tokenizer, backed by the native C++ encoder (csrc/tokenize.cpp,
`tl_tokenizer_*`), plus the batched, per-segment encoder a rollout uses to
turn collected texts into the packer's segment table.

Reference: ToyMergeTokenizer (tokenizer.py:36-87), DEFAULT_MERGES
(:27-33), trajectory._tokenize (trajectory.py:97-104) and the token caps of
orchestrator.feed_action / feed_response (orchestrator.py:112-117, :156-161).
Host code: needs the library, not a GPU.
"""

from __future__ import annotations

import ctypes as C
from typing import Protocol, Sequence

import numpy as np

from . import _lib


class Tokenizer(Protocol):
    """Minimal tokenizer surface the trajectory layer depends on (tokenizer.py:13-21)."""

    def encode(self, text: str) -> list[int]: ...

    def decode(self, tokens: Sequence[int]) -> str: ...

    @property
    def vocab_size(self) -> int: ...


DEFAULT_MERGES: tuple[tuple[str, str], ...] = (
    (">", "\n"),
    ("<", "/"),
    ("\n", "<"),
    ("e", "r"),
)


class ToyMergeTokenizer:
    """Byte-level tokenizer (ids 0..255) plus an ordered merge table: rule k
    makes one left-to-right pass merging every adjacent (left, right) pair
    into id 256 + k (tokenizer.py:36-87)."""

    def __init__(self, merges: Sequence[tuple[str, str]] = DEFAULT_MERGES):
        L = _lib.load(require_device=False)
        self._L = L
        known = {bytes([i]) for i in range(256)}
        parts, off = [], [0]
        for left, right in merges:
            lb, rb = left.encode("utf-8"), right.encode("utf-8")
            if lb not in known or rb not in known:  # same check and message as the reference
                raise ValueError(
                    f"merge ({left!r}, {right!r}) references a token that does not exist yet"
                )
            known.add(lb + rb)
            parts += [lb, rb]
            off += [off[-1] + len(lb), off[-1] + len(lb) + len(rb)]
        blob = b"".join(parts)
        self._blob = (C.c_uint8 * max(len(blob), 1)).from_buffer_copy(blob or b"\0")
        offs = np.asarray(off, dtype=np.int64)
        h = C.c_void_p()
        _lib.check(L.tl_tokenizer_create(C.addressof(self._blob), offs.ctypes.data,
                                         len(merges), C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._L.tl_tokenizer_free(h)
            self._h = None

    @property
    def vocab_size(self) -> int:
        return int(self._L.tl_tokenizer_vocab_size(self._h))

    def encode(self, text: str) -> list[int]:
        pool, off, lens = self.encode_segments([text])
        return pool[:lens[0]].tolist()

    def decode(self, tokens: Sequence[int]) -> str:
        ids = np.ascontiguousarray(np.asarray(list(tokens), dtype=np.int64))
        if ids.size and (ids.min() < 0 or ids.max() >= self.vocab_size):
            raise IndexError("list index out of range")  # the reference indexes a list
        ids32 = ids.astype(np.int32)
        n = C.c_int64()
        _lib.check(self._L.tl_tokenizer_decode(self._h, ids32.ctypes.data, ids32.size, None, 0,
                                               C.byref(n)))
        buf = (C.c_uint8 * max(n.value, 1))()
        _lib.check(self._L.tl_tokenizer_decode(self._h, ids32.ctypes.data, ids32.size,
                                               C.addressof(buf), n.value, C.byref(n)))
        # errors="replace": a cut through a multi-byte character degrades gracefully
        return bytes(buf)[:n.value].decode("utf-8", errors="replace")

    def encode_segments(self, texts: Sequence[str], max_tokens=None, n_threads: int = 0):
        """Encode every text on its own (never across a segment boundary),
        keeping the first max_tokens[i] ids (None / negative: no cap).
        Returns (token_pool int32, seg_src_off int64, seg_len int32): segment
        i is token_pool[seg_src_off[i] : seg_src_off[i] + seg_len[i]], the
        layout packing.SegmentTable / tl_pack_varlen consume."""
        enc = [t.encode("utf-8") for t in texts]
        off = np.zeros(len(enc) + 1, dtype=np.int64)
        np.cumsum([len(b) for b in enc], out=off[1:])
        blob = np.frombuffer(b"".join(enc), dtype=np.uint8) if off[-1] else np.zeros(1, np.uint8)
        pool = np.zeros(max(int(off[-1]), 1), dtype=np.int32)
        lens = np.zeros(len(enc), dtype=np.int32)
        caps = None
        if max_tokens is not None:
            caps = np.asarray([-1 if m is None else int(m) for m in (
                max_tokens if hasattr(max_tokens, "__len__") else [max_tokens] * len(enc))],
                dtype=np.int32)
        _lib.check(self._L.tl_tokenize_segments(
            self._h, blob.ctypes.data, off.ctypes.data, len(enc),
            None if caps is None else caps.ctypes.data, pool.ctypes.data, lens.ctypes.data,
            int(n_threads)))
        return pool, off[:-1], lens


def tokenize(tokenizer: ToyMergeTokenizer, text: str,
             max_tokens: int | None) -> tuple[str, list[int]]:
    """trajectory._tokenize (trajectory.py:97-104): encode, keep the first
    max_tokens ids and the text they decode to (never re-encode the cut)."""
    toks = tokenizer.encode(text)
    if max_tokens is not None and len(toks) > max_tokens:
        toks = toks[:max_tokens]
        text = tokenizer.decode(toks)
    return text, toks


def segment_table(tokenizer: ToyMergeTokenizer, trajectories, max_tokens=None,
                  n_threads: int = 0):
    """Rollout texts -> the packer's SegmentTable in one native call.

    trajectories: sequence of [(origin, text), ...] (origin "action" /
    "observation", alternating, action first as trajectory.append_segment
    enforces).  max_tokens: None, an int cap for every segment, or a
    parallel nested sequence of caps."""
    from .packing import SegmentTable

    texts, is_act, caps, nseg = [], [], [], []
    for i, segs in enumerate(trajectories):
        nseg.append(len(segs))
        for j, (origin, text) in enumerate(segs):
            texts.append(text)
            is_act.append(1 if origin == "action" else 0)
            if max_tokens is None:
                caps.append(None)
            elif isinstance(max_tokens, int):
                caps.append(max_tokens)
            else:
                caps.append(max_tokens[i][j])
    pool, off, lens = tokenizer.encode_segments(texts, caps, n_threads=n_threads)
    traj_seg_off = np.zeros(len(nseg) + 1, dtype=np.int32)
    np.cumsum(nseg, out=traj_seg_off[1:])
    if len(pool) >= 2 ** 31:
        raise ValueError("token pool exceeds int32 offsets")
    return SegmentTable(pool, off.astype(np.int32), lens, np.asarray(is_act, dtype=np.uint8),
                        traj_seg_off)
