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


def stack_cuts_capped(S: bytes, member: bool, cap: int = 127):
    """stack_cuts with the bounded nesting of reading R10: an opening bracket beyond `cap`
    open brackets is not pushed (the automaton's depth saturates at 127)."""
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
            if len(stack) < cap:
                stack.append(ch)
        elif stack and ch in (b"}", b"]"):
            stack.pop()
            if not stack:
                cuts.append((i + 1, 1, 0))
        elif member and ch == b"," and len(stack) == 1:
            cuts.append((i + 1, 0, 0))
        i += 1
    return cuts


def overflow_merge(natural, n: int, M: int):
    """Independent reading of the OVERFLOW rule (R13) for the JSON parsers, whose automaton
    state is not reset by an OVERFLOW cut: every natural cut stays a cut, and any run of M
    bytes since the previous cut that reaches no natural cut is cut with OVERFLOW (delim NONE).
    A natural cut exactly M bytes after the previous one stays natural."""
    out, c = [], 0
    for (p, did, fl) in natural:
        while p - c > M:
            c += M
            out.append((c, oracle.DELIM_NONE, oracle.FLAG_OVERFLOW))
        out.append((p, did, fl))
        c = p
    while n - c >= M:
        c += M
        out.append((c, oracle.DELIM_NONE, oracle.FLAG_OVERFLOW))
    return out


@pytest.mark.parametrize("M", [1, 2, 3, 5])
def test_json_overflow_bruteforce_vs_merge_reading(M):
    """JSON_MEMBER / JSON_OBJECT with a short max_segment_bytes: every string up to length 5
    over 8 symbols equals the natural stack cuts with OVERFLOW cuts merged in."""
    alpha = [b"{", b"}", b"[", b"]", b'"', b",", b"a", b"\\"]
    for S in all_strings(alpha, 5):
        for kind, member in ((MEM, True), (OBJ, False)):
            exp = overflow_merge(stack_cuts(S, member), len(S), M)
            assert oracle.segment(kind, [], M, S) == exp, (S, M)


def test_json_overflow_random_long_members():
    """Validation-shaped objects with members longer than max_segment_bytes (16..64)."""
    rng = random.Random(31)
    for _ in range(300):
        obj = {f"k{i}": "".join(rng.choice('ab ,{}":\\') for _ in range(rng.randint(0, 90)))
               for i in range(rng.randint(1, 8))}
        S = b"x " + json.dumps(obj).encode() + b" tail"
        M = rng.randint(16, 64)
        for kind, member in ((MEM, True), (OBJ, False)):
            assert oracle.segment(kind, [], M, S) == overflow_merge(stack_cuts(S, member), len(S), M)


def test_json_depth_cap_127():
    """Nesting deeper than 127 (R10): the depth saturates, so the object cut lands on the
    127th closing bracket after the saturation -- equal to a stack that stops pushing at 127."""
    S = b"[" * 130 + b"]" * 130
    assert oracle.segment(OBJ, [], BIG, S) == [(130 + 127, 1, 0)] == stack_cuts_capped(S, False)
    rng = random.Random(8)
    for _ in range(200):
        parts = []
        for _ in range(rng.randint(1, 6)):
            k = rng.randint(100, 140)
            parts.append(b"{" * k + b'"a,]"' + b"," * rng.randint(0, 2) + b"]" * rng.randint(k - 5, k + 5))
        S = b"".join(parts)
        for kind, member in ((MEM, True), (OBJ, False)):
            assert oracle.segment(kind, [], BIG, S) == stack_cuts_capped(S, member)
            assert oracle.segment(kind, [], 50, S) == overflow_merge(stack_cuts_capped(S, member), len(S), 50)


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


# ------------------------------------------------------------------ FENCE region grammar (NEXT-2)
FEN = oracle.PARSER_FENCE


def regex_fence(S: bytes, tag: bytes):
    """Independent reading of the fence grammar without overflow: split S into '\\n'-terminated
    lines with a regex, then pair markers with a running flag."""
    recs, inside = [], False
    for m in re.finditer(rb"[^\n]*\n", S):
        a, b, line = m.start(), m.end(), m.group(0)
        if not inside and line == b"```" + tag + b"\n":
            recs.append((a, b, 0, oracle.FLAG_OPEN))
            inside = True
        elif inside and line == b"```\n":
            recs.append((a, b, 0, oracle.FLAG_CLOSE))
            inside = False
        elif inside:
            recs.append((a, b, 0, 0))
    tail = S.rfind(b"\n") + 1
    return recs, tail


def test_fence_bruteforce_equals_regex_reading():
    """Every string up to length 9 over {`, p, \\n, a} (tag 'p': markers "```p\\n" / "```\\n")."""
    n = 0
    for S in all_strings([b"`", b"p", b"\n", b"a"], 9):
        assert oracle.fence_records(b"p", BIG, S) == regex_fence(S, b"p"), S
        n += 1
    assert n == sum(4 ** k for k in range(10))


def test_fence_paper_codegen_script_13_pieces():
    """the ```python / ``` indicators delimit the tool; lines 1-13 of the
    script are pieces; prose before/after the block is not tool input."""
    S = ("Here is the code.\n```python\n" + SINE_SCRIPT_13 + "```\nIt saves sine.png").encode()
    recs, tail = oracle.fence_records(b"python", 4096, S)
    assert [f for (_, _, _, f) in recs] == [oracle.FLAG_OPEN] + [0] * 13 + [oracle.FLAG_CLOSE]
    lines = SINE_SCRIPT_13.encode().splitlines(keepends=True)
    assert [S[a:b] for (a, b, _, f) in recs if f == 0] == lines
    assert S[tail:] == b"It saves sine.png"


def test_fence_other_tags_and_nesting_are_text():
    S = b"```bash\nls\n```\n```python\nx=1\n```python\n```\ny\n"
    recs, _ = oracle.fence_records(b"python", 4096, S)
    # the bash block is prose; inside the python block a second opener is just a line
    assert [(S[a:b], f) for (a, b, _, f) in recs] == [
        (b"```python\n", oracle.FLAG_OPEN), (b"x=1\n", 0), (b"```python\n", 0), (b"```\n", oracle.FLAG_CLOSE)]


def test_fence_overflow_inside_and_outside():
    S = b"aaaaaaa\n```p\nbbbbbbbbbbbbb\n```\ncc"
    recs, tail = oracle.fence_records(b"p", 6, S)
    # outside: overflow units emit nothing; inside: OVERFLOW pieces, then the line's rest
    assert [(S[a:b], d, f) for (a, b, d, f) in recs] == [
        (b"```p\n", 0, oracle.FLAG_OPEN), (b"bbbbbb", oracle.DELIM_NONE, oracle.FLAG_OVERFLOW),
        (b"bbbbbb", oracle.DELIM_NONE, oracle.FLAG_OVERFLOW), (b"b\n", 0, 0), (b"```\n", 0, oracle.FLAG_CLOSE)]
    assert S[tail:] == b"cc"
    # a continuation unit never matches a marker even if its bytes do
    recs2, _ = oracle.fence_records(b"p", 6, b"xxxxxx```p\nq\n")
    assert recs2 == []
    # a marker longer than max_seg can never open a region
    assert oracle.fence_records(b"p", 4, b"```p\nx\n")[0] == []


def test_fence_invariants_random():
    rng = random.Random(11)
    alpha = [b"`", b"p", b"\n", b"a", b"```p\n", b"```\n"]
    for _ in range(3000):
        S = b"".join(rng.choice(alpha) for _ in range(rng.randrange(0, 24)))
        M = rng.choice([3, 5, 8, BIG])
        recs, tail = oracle.fence_records(b"p", M, S)
        ends = [b for (_, b, _, _) in recs]
        assert ends == sorted(ends) and all(b <= tail for b in ends)
        depth = 0
        for (a, b, d, f) in recs:
            assert 0 < b - a <= M
            if f == oracle.FLAG_OPEN:
                assert depth == 0 and S[a:b] == b"```p\n"
                depth = 1
            elif f == oracle.FLAG_CLOSE:
                assert depth == 1 and S[a:b] == b"```\n"
                depth = 0
            else:
                assert depth == 1
                assert (f == 0 and S[b - 1:b] == b"\n") or (f == oracle.FLAG_OVERFLOW and b - a == M)
        assert b"\n" not in S[tail:] and len(S) - tail < M


@pytest.mark.parametrize("L", range(1, 8))
def test_fence_token_index_every_tokenization(L):
    vocab = {}
    rng = random.Random(100 + L)
    strings = [s for s in all_strings([b"`", b"p", b"\n", b"a"], L) if len(s) == L]
    strings = [b"```p\n" + s + b"\n```\n" for s in rng.sample(strings, min(60, len(strings)))]
    for S in strings:
        base, tail = oracle.fence_records(b"p", BIG, S)
        n = len(S)
        for _ in range(40):
            cut = sorted(rng.sample(range(1, n), rng.randrange(0, min(6, n - 1))))
            bounds = [0] + cut + [n]
            pieces = [S[bounds[i]:bounds[i + 1]] for i in range(len(bounds) - 1)]
            ids = [vocab.setdefault(p, len(vocab)) for p in pieces]
            table = {v: k for k, v in vocab.items()}
            recs, stream = round_records(ids, table, FEN, [b"p"], BIG)
            assert stream == S
            assert [(r.byte_offset, r.byte_offset + r.byte_len, r.delim_id, r.flags) for r in recs[:-1]] == base
            for r in recs[:-1]:
                last = r.byte_offset + r.byte_len - 1
                assert r.token_index == max(i for i in range(len(pieces)) if bounds[i] <= last)
            assert recs[-1].byte_offset == tail and recs[-1].flags == oracle.FLAG_FINAL


# ------------------------------------------------------------------ CALL / PLAN grammars (NEXT-2)
CAL, PLN = oracle.PARSER_CALL, oracle.PARSER_PLAN


def search_call_reading(S: bytes, tag: bytes):
    """Independent reading of CALL without overflow, search-based instead of a byte automaton:
    find the next line start whose line begins with the marker, then walk the JSON value with
    an explicit stack to its end, cutting at depth-1 commas; continue after the value."""
    marker = b"@call " + tag + b" "
    recs, pos = [], 0
    while True:
        starts = [0] + [m.end() for m in re.finditer(rb"\n", S)]
        cand = [s for s in starts if s >= pos and S.startswith(marker, s)]
        if not cand:
            break
        a = cand[0]
        recs.append((a, a + len(marker), 0, oracle.FLAG_OPEN))
        c = a + len(marker)
        stack, in_s, esc, i, closed = [], False, False, c, False
        while i < len(S):
            ch = S[i:i + 1]
            if in_s:
                if esc:
                    esc = False
                elif ch == b"\\":
                    esc = True
                elif ch == b'"':
                    in_s = False
            elif not stack:
                if ch in (b"{", b"["):
                    stack.append(ch)
            elif ch == b'"':
                in_s = True
            elif ch in (b"{", b"["):
                stack.append(ch)
            elif ch in (b"}", b"]"):
                stack.pop()
                if not stack:
                    recs.append((c, i + 1, 1, oracle.FLAG_CLOSE))
                    pos, closed = i + 1, True
                    break
            elif ch == b"," and len(stack) == 1:
                recs.append((c, i + 1, 0, 0))
                c = i + 1
            i += 1
        if not closed:
            return recs, c
        # the rest of the closing line is not at a line start: resume at the next line
        nl = S.find(b"\n", pos)
        if nl < 0:
            return recs, _tail_after(S, pos)
        pos = nl + 1
    return recs, _tail_after(S, pos if recs else 0)


def _tail_after(S, pos):
    """FINAL start outside a region: the start of the last line at or after pos."""
    k = S.rfind(b"\n", pos)
    return pos if k < 0 else k + 1


def test_call_random_equals_search_reading():
    rng = random.Random(17)
    toks = [b"@call s ", b"@call s", b"@call t ", b"{", b"}", b"[", b"]", b",", b'"', b"\\", b"a", b"\n", b" "]
    for _ in range(20000):
        S = b"".join(rng.choice(toks) for _ in range(rng.randrange(0, 16)))
        got = oracle.call_records(b"s", BIG, S)
        assert got == search_call_reading(S, b"s"), S


def test_call_search_workload_fields_from_serialisation():
    """Three consecutive calls (the Search workload issues three): OPEN at the
    marker, one piece per member (boundaries from per-member json.dumps), CLOSE at the object end."""
    rng = random.Random(3)
    for _ in range(200):
        objs = [{f"k{j}": rng.choice(["a, b", 7, "x}y", [1, 2], {"z": "}"}]) for j in range(rng.randrange(1, 5))}
                for _ in range(3)]
        parts = [b"Let me look these up.\n"]
        for o in objs:
            parts.append(b"@call search " + json.dumps(o).encode() + b"\n")
        S = b"".join(parts) + b"Answer"
        recs, tail = oracle.call_records(b"search", BIG, S)
        flags = [f for (_, _, _, f) in recs]
        assert flags.count(oracle.FLAG_OPEN) == 3 and flags.count(oracle.FLAG_CLOSE) == 3
        for o in objs:
            items = list(o.items())
            want = [("{" if j == 0 else " ") + json.dumps(k) + ": " + json.dumps(v) + ("," if j + 1 < len(items) else "}")
                    for j, (k, v) in enumerate(items)]
            got = [S[a:b].decode() for (a, b, d, f) in recs[:len(items) + 1][1:]]
            assert got == want
            recs = recs[len(items) + 1:]
        assert S[tail:] == b"Answer"


def test_call_marker_must_start_a_line_and_overflow():
    S = b"x @call s {\"a\": 1}\n@call s {\"a\": 12345678901}\n"
    recs, _ = oracle.call_records(b"s", 12, S)
    assert [(S[a:b], d, f) for (a, b, d, f) in recs] == [
        (b"@call s ", 0, oracle.FLAG_OPEN), (b'{"a": 123456', oracle.DELIM_NONE, oracle.FLAG_OVERFLOW),
        (b"78901}", 1, oracle.FLAG_CLOSE)]


def plan_line_reading(line: bytes) -> bool:
    """Hand-written check of one '\\n'-terminated line: #E<digits> = <Name>[<args>]."""
    if not (line.startswith(b"#E") and line.endswith(b"]\n")):
        return False
    i = 2
    while i < len(line) and line[i:i + 1].isdigit():
        i += 1
    if i == 2 or line[i:i + 3] != b" = ":
        return False
    i += 3
    j = i
    while j < len(line) and (line[j:j + 1].isalnum() or line[j:j + 1] == b"_"):
        j += 1
    if j == i or line[j:j + 1] != b"[":
        return False
    return b"\n" not in line[j + 1:-1]


def test_plan_random_equals_hand_reading():
    rng = random.Random(19)
    toks = [b"#E", b"#", b"E", b"1", b"23", b" = ", b"=", b" ", b"search", b"_", b"[", b"]", b"\n", b"x"]
    for _ in range(20000):
        S = b"".join(rng.choice(toks) for _ in range(rng.randrange(0, 18)))
        recs, tail = oracle.plan_records(BIG, S)
        want = [(m.start(), m.end(), 0, 0) for m in re.finditer(rb"[^\n]*\n", S) if plan_line_reading(m.group(0))]
        assert (recs, tail) == (want, S.rfind(b"\n") + 1), S


def test_plan_four_stages():
    """a 4-stage plan (two searches, a calculator, a formatter)."""
    S = (b"Plan:\n#E1 = search[Microsoft market cap]\n#E2 = search[Apple market cap]\n"
         b"#E3 = calculator[#E1 / #E2]\n#E4 = formatter[ratio: #E3]\nThen answer.")
    recs, tail = oracle.plan_records(4096, S)
    assert len(recs) == 4 and all(S[b - 2:b] == b"]\n" for (_, b, _, _) in recs)
    assert S[tail:] == b"Then answer."


@pytest.mark.parametrize("kind,tag", [(CAL, b"s"), (PLN, b"")])
def test_region_grammars_token_index_random_splits(kind, tag):
    rng = random.Random(23 + kind)
    vocab = {}
    texts = [b'@call s {"a": 1, "b": [2, 3]}\nx\n@call s {"c": "}"}', b"#E1 = s[a]\n#E2 = t[b]\nz"]
    for S in texts * 30:
        n = len(S)
        cut = sorted(rng.sample(range(1, n), rng.randrange(0, 8)))
        bounds = [0] + cut + [n]
        pieces = [S[bounds[i]:bounds[i + 1]] for i in range(len(bounds) - 1)]
        ids = [vocab.setdefault(p, len(vocab)) for p in pieces]
        table = {v: k for k, v in vocab.items()}
        recs, stream = round_records(ids, table, kind, [tag], BIG)
        base, tail = (oracle.call_records(tag, BIG, S) if kind == CAL else oracle.plan_records(BIG, S))
        assert [(r.byte_offset, r.byte_offset + r.byte_len, r.delim_id, r.flags) for r in recs[:-1]] == base
        for r in recs[:-1]:
            last = r.byte_offset + r.byte_len - 1
            assert r.token_index == max(i for i in range(len(pieces)) if bounds[i] <= last)
        assert recs[-1].byte_offset == tail


# ------------------------------------------------------------------ multi-tool region sets (NEXT-2, R24)
def mixed_region_reading(S: bytes, fences: dict, calls: dict):
    """Independent reading of R24 without overflow, search-based: from the current position,
    find the first line start whose line is a fence open marker (b"```" + tag + b"\\n") or
    begins with a call marker (b"@call " + tag + b" "); a fence region is then walked line by
    line (regex) to the b"```\\n" line, a call region through its JSON value with an explicit
    stack (as search_call_reading); scanning resumes at the next line start.
    fences / calls: {tool_id: tag}.  Returns (records with tool ids, FINAL start, FINAL tool)."""
    marks = sorted([(t, b"```" + g + b"\n", "F") for t, g in fences.items()] +
                   [(t, b"@call " + g + b" ", "C") for t, g in calls.items()])
    recs, pos = [], 0
    starts = [0] + [m.end() for m in re.finditer(rb"\n", S)]
    while True:
        found = None
        for s in starts:
            if s < pos:
                continue
            hit = [(t, m, k) for (t, m, k) in marks if S.startswith(m, s)]
            if hit:
                found = (s,) + hit[0]
                break
        if found is None:
            return recs, _tail_after(S, pos), -1
        a, tool, m, kind = found
        recs.append((a, a + len(m), 0, oracle.FLAG_OPEN, tool))
        c = a + len(m)
        if kind == "F":
            closed = False
            for mm in re.finditer(rb"[^\n]*\n", S[c:]):
                x, y = c + mm.start(), c + mm.end()
                if mm.group(0) == b"```\n":
                    recs.append((x, y, 0, oracle.FLAG_CLOSE, tool))
                    pos, closed = y, True
                    break
                recs.append((x, y, 0, 0, tool))
            if not closed:
                last = S.rfind(b"\n", c)
                return recs, (c if last < 0 else last + 1), tool
            continue
        stack, in_s, esc, i, closed = [], False, False, c, False
        while i < len(S):
            ch = S[i:i + 1]
            if in_s:
                if esc:
                    esc = False
                elif ch == b"\\":
                    esc = True
                elif ch == b'"':
                    in_s = False
            elif not stack:
                if ch in (b"{", b"["):
                    stack.append(ch)
            elif ch == b'"':
                in_s = True
            elif ch in (b"{", b"["):
                stack.append(ch)
            elif ch in (b"}", b"]"):
                stack.pop()
                if not stack:
                    recs.append((c, i + 1, 1, oracle.FLAG_CLOSE, tool))
                    pos, closed = i + 1, True
                    break
            elif ch == b"," and len(stack) == 1:
                recs.append((c, i + 1, 0, 0, tool))
                c = i + 1
            i += 1
        if not closed:
            return recs, c, tool
        nl = S.find(b"\n", pos)
        if nl < 0:
            return recs, _tail_after(S, pos), -1
        pos = nl + 1


def test_region_single_tool_is_fence_or_call():
    """A set of one FENCE (CALL) tool is exactly the pinned FENCE (CALL) grammar, overflow included."""
    rng = random.Random(41)
    toks = [b"```p\n", b"```\n", b"@call p ", b"{", b"}", b",", b'"', b"a", b"\n", b" ", b"`"]
    for _ in range(3000):
        S = b"".join(rng.choice(toks) for _ in range(rng.randint(0, 30)))
        M = rng.choice([6, 9, 13, BIG])
        rf, cf, _ = oracle.region_records([(3, FEN, b"p", M)], S)
        assert ([r[:4] for r in rf], cf) == oracle.fence_records(b"p", M, S) and all(r[4] == 3 for r in rf)
        M = rng.choice([8, 11, 17, BIG])
        rc, cc, _ = oracle.region_records([(5, CAL, b"p", M)], S)
        assert ([r[:4] for r in rc], cc) == oracle.call_records(b"p", M, S) and all(r[4] == 5 for r in rc)


def test_region_two_fences_bruteforce():
    """Every string up to length 7 over {`, p, q, \\n, a} with FENCE tools p (id 0) and q (id 1)."""
    n = 0
    for S in all_strings([b"`", b"p", b"q", b"\n", b"a"], 7):
        assert oracle.region_records([(0, FEN, b"p", BIG), (1, FEN, b"q", BIG)], S) == \
            mixed_region_reading(S, {0: b"p", 1: b"q"}, {}), S
        n += 1
    assert n == sum(5 ** k for k in range(8))


def test_region_mixed_fences_and_calls_random():
    """Random streams mixing two fence tags, two call tools, JSON and prose."""
    rng = random.Random(43)
    toks = [b"```py\n", b"```sh\n", b"```\n", b"@call s ", b"@call t ", b"@call u ", b"{", b"}", b"[", b"]",
            b",", b'"', b"\\", b"a", b"\n", b" ", b"`"]
    tools = [(0, FEN, b"py", BIG), (1, FEN, b"sh", BIG), (2, CAL, b"s", BIG), (3, CAL, b"t", BIG)]
    for _ in range(20000):
        S = b"".join(rng.choice(toks) for _ in range(rng.randint(0, 40)))
        assert oracle.region_records(tools, S) == mixed_region_reading(S, {0: b"py", 1: b"sh"}, {2: b"s", 3: b"t"}), S


def test_region_set_outside_cut_is_the_smallest_max_segment():
    """Outside a region the line is cut at the smallest max_segment_bytes of the set; the rest
    of that line is a continuation and cannot open a region (hand-checked)."""
    tools = [(0, FEN, b"p", 6), (1, CAL, b"s", 20)]
    S = b"aaaaaa```p\n```p\nx\n"
    recs, c, t = oracle.region_records(tools, S)
    # "aaaaaa" is cut at 6 bytes, "```p\n" is then a continuation: no OPEN; the next line opens
    assert recs == [(11, 16, 0, oracle.FLAG_OPEN, 0), (16, 18, 0, 0, 0)] and (c, t) == (18, 0)
