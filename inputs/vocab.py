"""Synthetic vocabulary and greedy tokenizer (reading R17).

The paper's models ship trained tokenizers we do not have (no network), so both sides
receive the same seeded table T: id -> bytes (|T[id]| <= 16):
  * byte-level (tiny config, V = 256): T[i] = bytes([i]);
  * V > 259: ids 0..2 are specials (unk, BOS, EOS) with empty byte strings, ids 3..258
    are the 256 single bytes (byte fallback), ids 259..V-1 are the most frequent 2..16
    byte substrings of the seeded workload corpus (so delimiters occur mid-token, e.g.
    ")\\n", ":\\n    ", "},\\n"), filled up with seeded random byte strings if needed.
Tokenization is greedy longest match.  This is input preparation, not method arithmetic.
"""
from __future__ import annotations

import random
from collections import Counter
from functools import lru_cache

from .workloads import corpus

MAX_TOKEN_BYTES = 16
SPECIALS = 3  # 0 unk, 1 BOS, 2 EOS
BOS, EOS = 1, 2


def byte_level_vocab(V: int = 256) -> list[bytes]:
    assert V == 256
    return [bytes([i]) for i in range(256)]


@lru_cache(maxsize=4)
def synthetic_vocab(V: int, seed: int = 7) -> tuple:
    if V == 256:
        return tuple(byte_level_vocab())
    assert V > SPECIALS + 256
    text = corpus(seed).encode()
    counts = Counter()
    n = len(text)
    for L in range(2, MAX_TOKEN_BYTES + 1):
        step = 1 if L <= 6 else 2
        for i in range(0, n - L + 1, step):
            counts[text[i:i + L]] += 1
    # gain of merging a substring: (len - 1) * count; deterministic tie-break on bytes
    cands = sorted(((c * (len(s) - 1), s) for s, c in counts.items() if c >= 2),
                   key=lambda x: (-x[0], x[1]))
    vocab = [b"", b"", b""] + [bytes([i]) for i in range(256)]
    seen = set(vocab[SPECIALS:])
    for _, s in cands:
        if len(vocab) >= V:
            break
        if s not in seen:
            seen.add(s)
            vocab.append(s)
    rng = random.Random(seed)
    while len(vocab) < V:
        s = bytes(rng.randrange(32, 127) for _ in range(rng.randint(2, 8)))
        if s not in seen:
            seen.add(s)
            vocab.append(s)
    return tuple(vocab)


class Tokenizer:
    """Greedy longest-match tokenizer over a vocab table."""

    def __init__(self, vocab):
        self.vocab = list(vocab)
        self.index = {}
        for i, s in enumerate(self.vocab):
            if s and s not in self.index:
                self.index[s] = i
        self.maxlen = max(len(s) for s in self.vocab)

    def encode(self, text) -> list[int]:
        b = text.encode() if isinstance(text, str) else bytes(text)
        out = []
        i = 0
        n = len(b)
        while i < n:
            for L in range(min(self.maxlen, n - i), 0, -1):
                t = self.index.get(b[i:i + L])
                if t is not None:
                    out.append(t)
                    i += L
                    break
            else:  # pragma: no cover - every single byte is in the vocab
                raise ValueError("untokenizable byte")
        return out

    def decode(self, ids) -> bytes:
        return b"".join(self.vocab[i] for i in ids)


def table(vocab) -> tuple[bytes, bytes]:
    """Flattened [V][16] byte table + [V] lengths, the layout the C ABI copies."""
    V = len(vocab)
    tb = bytearray(V * MAX_TOKEN_BYTES)
    ln = bytearray(V)
    for i, s in enumerate(vocab):
        assert len(s) <= MAX_TOKEN_BYTES
        tb[i * MAX_TOKEN_BYTES:i * MAX_TOKEN_BYTES + len(s)] = s
        ln[i] = len(s)
    return bytes(tb), bytes(ln)
