"""Pins for oracle O-2 (segmentation) against things other than itself.

 * Single-byte delimiters: textbook regex `[^D]*[D]` (Python `re`), every string up to
   length 10 over {a, ;, \\n}.
 * Overlapping multi-byte delimiters: an independently written match-set matcher
   (enumerate every delimiter occurrence, then take leftmost-ending ones that start at
   or after the previous cut), every string up to length 9.
 * token_index ("emit ... immediately"): for every tokenization
   (all 2^(L-1) splits) the index is the token whose byte range holds the cut's last byte.
 * JSON: member/object boundaries computed from per-member json.dumps serialisations; an
   independent stack-based bracket/string scanner on brute-force strings.
 * Invariants (north star): concat(segments) + tail = S; every non-final, non-overflow
   segment ends with a registered delimiter; no proper prefix does.
 * Paper structure: a 13-line script gives 13 segments; a 4-stage plan
   gives 4 object cuts.
"""
import itertools
import json
import random
import re

import pytest

import oracle
from oracle.scan import NO_TOKEN, round_length, round_records
from inputs.workloads import SINE_SCRIPT_13, plan_stages

LIT, MEM, OBJ = oracle.PARSER_LITERAL, oracle.PARSER_JSON_MEMBER, oracle.PARSER_JSON_OBJECT
BIG = 1 << 20


def all_strings(alpha, max_len):
    for L in range(0, max_len + 1):
        for t in itertools.product(alpha, repeat=L):
            yield b"".join(t)


def matchset_cuts(S: bytes, delims):
    """Independent: all occurrences (start, end, i), then repeatedly choose the
    occurrence with the smallest end among those starting at/after the last cut;
    ties on end -> smallest delimiter index."""
    occ = []
    for i, d in enumerate(delims):
        for s in range(len(S) - len(d) + 1):
            if S[s:s + len(d)] == d:
                occ.append((s, s + len(d), i))
    cuts, c = [], 0
    while True:
        cand = [(e, i) for (s, e, i) in occ if s >= c]
        if not cand:
            return cuts
        e, i = min(cand)
        cuts.append((e, i, 0))
        c = e


def test_single_byte_delims_equal_regex():
    n = 0
    for S in all_strings([b"a", b";", b"\n"], 10):
        got = oracle.segment(LIT, [b"\n", b";"], BIG, S)
        segs = re.findall(rb"[^;\n]*[;\n]", S)
        ends = list(itertools.accumulate(len(x) for x in segs))
        assert [g[0] for g in got] == ends
        assert [g[1] for g in got] == [0 if x.endswith(b"\n") else 1 for x in segs]
        n += 1
    assert n == sum(3 ** k for k in range(11))  # 88,573 strings


def test_newline_only_equals_findall():
    rng = random.Random(3)
    for _ in range(500):
        S = bytes(rng.choice(b"ab\n;{") for _ in range(rng.randint(0, 60)))
        got = [g[0] for g in oracle.segment(LIT, [b"\n"], BIG, S)]
        exp = list(itertools.accumulate(len(x) for x in re.findall(rb"[^\n]*\n", S)))
        assert got == exp


@pytest.mark.parametrize("delims,alpha", [
    ([b";;", b"\n", b"a;"], [b"a", b";", b"\n"]),
    ([b";;", b"\r\n", b"\n"], [b"a", b";", b"\r", b"\n"]),
    ([b"ab", b"b", b"aab"], [b"a", b"b"]),
])
def test_overlapping_delims_equal_matchset(delims, alpha):
    maxlen = 9 if len(alpha) <= 3 else 7
    for S in all_strings(alpha, maxlen):
        assert oracle.segment(LIT, delims, BIG, S) == matchset_cuts(S, delims)


def check_invariants(S, cuts, delims):
    segs, c = [], 0
    for (e, did, fl) in cuts:
        segs.append(S[c:e])
        c = e
    tail = S[c:]
    assert b"".join(segs) + tail == S
    for seg, (e, did, fl) in zip(segs, cuts):
        if fl == 0:
            assert seg.endswith(delims[did])
            # no proper prefix of the segment ends with a delimiter lying inside it
            for p in range(1, len(seg)):
                assert not any(len(d) <= p and seg[:p].endswith(d) for d in delims)
            # smallest matching index
            assert did == min(i for i, d in enumerate(delims) if seg.endswith(d))


def test_invariants_random():
    rng = random.Random(11)
    for _ in range(300):
        delims = list({bytes(rng.choice(b"ab;\n") for _ in range(rng.randint(1, 4)))
                       for _ in range(rng.randint(1, 5))})
        S = bytes(rng.choice(b"ab;\nc") for _ in range(rng.randint(0, 80)))
        check_invariants(S, oracle.segment(LIT, delims, BIG, S), delims)


def test_overflow_cut():
    S = b"x" * 10 + b"\n" + b"y" * 3
    got = oracle.segment(LIT, [b"\n"], 4, S)
    assert got == [(4, oracle.DELIM_NONE, oracle.FLAG_OVERFLOW), (8, oracle.DELIM_NONE, oracle.FLAG_OVERFLOW),
                   (11, 0, 0)]
    # a match and the overflow length at the same byte: the match wins
    assert oracle.segment(LIT, [b"\n"], 3, b"ab\ncd") == [(3, 0, 0)]


@pytest.mark.parametrize("L", range(1, 9))
def test_token_index_every_tokenization(L):
    vocab = {}
    delims = [b";;", b"\n"]
    rng = random.Random(L)
    strings = list(all_strings([b"a", b";", b"\n"], L))
    strings = [s for s in strings if len(s) == L]
    if len(strings) > 200:
        strings = rng.sample(strings, 200)
    for S in strings:
        base = oracle.segment(LIT, delims, BIG, S)
        for mask in range(1 << (L - 1)):
            pieces, cur = [], S[:1]
            for i in range(1, L):
                if mask >> (i - 1) & 1:
                    pieces.append(cur)
                    cur = S[i:i + 1]
                else:
                    cur += S[i:i + 1]
            pieces.append(cur)
            ids = []
            for p in pieces:
                ids.append(vocab.setdefault(p, len(vocab)))
            table = {v: k for k, v in vocab.items()}
            recs, stream = round_records(ids, table, LIT, delims, BIG)
            assert stream == S
            assert [(r.byte_offset + r.byte_len, r.delim_id, r.flags) for r in recs[:-1]] == base
            starts = list(itertools.accumulate([0] + [len(p) for p in pieces]))
            for r in recs[:-1]:
                last = r.byte_offset + r.byte_len - 1
                t = max(i for i in range(len(pieces)) if starts[i] <= last)
                assert r.token_index == t
            assert recs[-1].flags == oracle.FLAG_FINAL and recs[-1].token_index == len(pieces) - 1
            assert [r.seq for r in recs] == list(range(len(recs)))


def test_specials_and_empty_round():
    table = {0: b"", 1: b"", 2: b"", 3: b"x;", 4: b";"}
    recs, S = round_records([3, 2], table, LIT, [b";"], BIG)
    assert S == b"x;" and recs[0].token_index == 0 and recs[0].byte_len == 2
    assert recs[1].flags == oracle.FLAG_FINAL and recs[1].byte_len == 0 and recs[1].token_index == 1
    recs, S = round_records([], table, LIT, [b";"], BIG, cancelled=True)
    assert len(recs) == 1 and recs[0].token_index == NO_TOKEN
    assert recs[0].flags == oracle.FLAG_FINAL | oracle.FLAG_CANCELLED
    assert round_length([5, 6, 2, 7], eos=2, max_new=10) == 3
    assert round_length([5, 6, 7], eos=2, max_new=2) == 2


# ---------------------------------------------------------------- JSON


def rand_value(rng, depth=0):
    r = rng.random()
    if depth < 2 and r < 0.2:
        return {f"k{i}": rand_value(rng, depth + 1) for i in range(rng.randint(0, 3))}
    if depth < 2 and r < 0.35:
        return [rand_value(rng, depth + 1) for _ in range(rng.randint(0, 3))]
    if r < 0.7:
        return "".join(rng.choice('ab,{}[]":\\ ') for _ in range(rng.randint(0, 8)))
    return rng.randint(-1000, 1000)


@pytest.mark.parametrize("seps", [(",", ":"), (", ", ": ")])
def test_json_member_cuts_from_serialisation(seps):
    rng = random.Random(5)
    for _ in range(400):
        obj = {f"key{i}": rand_value(rng) for i in range(rng.randint(1, 6))}
        S = json.dumps(obj, separators=seps).encode()
        members = [json.dumps(k) + seps[1] + json.dumps(v, separators=seps) for k, v in obj.items()]
        exp, pos = [], 1
        for j, m in enumerate(members):
            pos += len(m.encode())
            exp.append(pos + 1)  # the ',' after the member, or the closing '}'
            pos += len(seps[0].encode()) if j + 1 < len(members) else 0
        got = oracle.segment(MEM, [], BIG, b"prose " + S + b" tail")
        assert [g[0] - 6 for g in got] == exp
        assert [g[1] for g in got] == [0] * (len(exp) - 1) + [1]
        got_o = oracle.segment(OBJ, [], BIG, S)
        assert got_o == [(len(S), 1, 0)]


def stack_cuts(S: bytes, member: bool):
    """Independent definition: find string literals and brackets with an explicit stack
    of open brackets; strings only exist inside a bracket; prose outside is ignored."""
    stack, cuts, i, n = [], [], 0, len(S)
    while i < n:
        ch = S[i:i + 1]
        if stack and ch == b'"':
            j = i + 1
            while j < n and S[j:j + 1] != b'"':
                j += 2 if S[j:j + 1] == b"\\" else 1
            if j >= n:
                return cuts
            i = j + 1
            continue
        if ch in (b"{", b"["):
            stack.append(ch)
        elif stack and ch in (b"}", b"]"):
            stack.pop()
            if not stack:
                cuts.append((i + 1, 1, 0))
        elif member and ch == b"," and len(stack) == 1:
            cuts.append((i + 1, 0, 0))
        i += 1
    return cuts


def test_json_bruteforce_vs_stack_definition():
    alpha = [b"{", b"}", b"[", b"]", b'"', b",", b"a", b"\\"]
    for S in all_strings(alpha, 6):
        for kind, member in ((MEM, True), (OBJ, False)):
            assert oracle.segment(kind, [], BIG, S) == stack_cuts(S, member), S


# ---------------------------------------------------------------- paper structure


def test_13_line_script_gives_13_segments():
    S = SINE_SCRIPT_13.encode()
    cuts = oracle.segment(LIT, [b"\n"], BIG, S)
    assert len(cuts) == 13 and cuts[-1][0] == len(S)
    lines = SINE_SCRIPT_13.splitlines(keepends=True)
    assert [e for e, _, _ in cuts] == list(itertools.accumulate(len(x) for x in lines))


def test_four_stage_plan_gives_four_object_cuts():
    rng = random.Random(1)
    S = plan_stages(rng).encode()
    cuts = oracle.segment(OBJ, [], BIG, S)
    assert len(cuts) == 4
    for (e, did, fl), line in zip(cuts, S.split(b"\n")):
        assert did == 1 and fl == 0
    assert [json.loads(x) for x in S.decode().strip().split("\n")][3]["id"] == 4
