"""Restatement of the reference tokenizer (TEST INFRASTRUCTURE ONLY: imported
by tests/ as the checker for the native encoder, never by the product).

Follows toolloop.tokenizer.ToyMergeTokenizer (tokenizer.py:36-87): ids
0..255 are bytes; merge k = (left, right) -> id 256 + k, and rule k makes a
single left-to-right pass over the current sequence merging every adjacent
(left, right) pair; rules apply in table order.  `tokenize` follows
trajectory._tokenize (trajectory.py:97-104): keep the first max_tokens ids and
the text they decode to.  Pinned to tests/golden/tokenizer.json (outputs of
the reference itself).
"""

from __future__ import annotations

DEFAULT_MERGES = ((">", "\n"), ("<", "/"), ("\n", "<"), ("e", "r"))


def build(merges=DEFAULT_MERGES):
    table = [bytes([i]) for i in range(256)]
    ids = {b: i for i, b in enumerate(table)}
    rules = []
    for left, right in merges:  # tokenizer.py:49-62
        lb, rb = left.encode("utf-8"), right.encode("utf-8")
        if lb not in ids or rb not in ids:
            raise ValueError(f"merge ({left!r}, {right!r}) references a token that does not exist yet")
        rules.append((ids[lb], ids[rb], len(table)))
        table.append(lb + rb)
        ids[lb + rb] = len(table) - 1
    return table, rules


def encode(text, merges=DEFAULT_MERGES):
    _, rules = build(merges)
    seq = list(text.encode("utf-8"))
    for left, right, new in rules:  # tokenizer.py:68-81
        out, i = [], 0
        while i < len(seq):
            if i + 1 < len(seq) and seq[i] == left and seq[i + 1] == right:
                out.append(new)
                i += 2
            else:
                out.append(seq[i])
                i += 1
        seq = out
    return seq


def decode(tokens, merges=DEFAULT_MERGES):
    table, _ = build(merges)
    return b"".join(table[t] for t in tokens).decode("utf-8", errors="replace")


def tokenize(text, max_tokens, merges=DEFAULT_MERGES):
    toks = encode(text, merges)
    if max_tokens is not None and len(toks) > max_tokens:  # trajectory.py:100-103
        toks = toks[:max_tokens]
        text = decode(toks, merges)
    return text, toks
