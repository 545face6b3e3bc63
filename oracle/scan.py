"""O-2 round driver -- TEST INFRASTRUCTURE (see oracle/__init__.py).

Turns one round of generated token ids into the per-request segment records the
device scan must publish (R5-R13), following SURVEY.md 8(c) O-2 steps 1-6:

  1. bytes: S = T[y_1] || ... || T[y_N] over the round's generated ids (specials
     map to the empty string; prompt/observation inputs are never scanned,
     SPEC.md:102); e_t = sum_{s<=t} |T[y_s]|.
  2./3. cuts from oracle.segment (plain definition).
  4. round end (EOS, max_new_tokens, forced-stream end, cancel): one FINAL record
     for the tail S[c_last, |S|), possibly empty (FENCE: the trailing incomplete line).
  token_index of a cut = min{t : e_t >= c_j} - 1 (0-based index of the generated
  token holding the cut's last byte: "emit completed pieces ... immediately",
  PAPER.md:144).  FINAL carries N-1 (0xFFFFFFFF when the round generated nothing).
"""
from __future__ import annotations

from dataclasses import dataclass

from . import (DELIM_NONE, FLAG_CANCELLED, FLAG_FINAL, PARSER_CALL, PARSER_FENCE, PARSER_PLAN, call_records,
               fence_records, plan_records, region_records, segment)

NO_TOKEN = 0xFFFFFFFF


@dataclass(frozen=True)
class Record:
    round: int
    seq: int
    token_index: int
    byte_offset: int
    byte_len: int
    delim_id: int
    flags: int
    data: bytes
    tool: int = -1


def round_length(tokens, eos: int, max_new: int) -> int:
    """Number of generated tokens in the round: up to and including the first EOS,
    at most max_new (R12)."""
    n = min(len(tokens), max_new)
    for i in range(n):
        if eos >= 0 and tokens[i] == eos:
            return i + 1
    return n


def round_records(tokens, vocab_bytes, kind: int, delims: list[bytes], max_seg: int,
                  round_idx: int = 0, seq_start: int = 0, cancelled: bool = False, tool_id: int = -1,
                  region_tools=None):
    """Records for one round whose generated ids are exactly `tokens` (already cut at
    the round end).  tool_id: the request's tool (each record's `tool`); region_tools: a
    multi-tool set [(tool_id, kind, tag, max_seg)] of FENCE / CALL tools (R24; kind and
    delims are then unused).  Returns (records, stream_bytes)."""
    pieces = [vocab_bytes[t] for t in tokens]
    S = b"".join(pieces)
    ends = []
    acc = 0
    for p in pieces:
        acc += len(p)
        ends.append(acc)
    recs = []
    c_prev = 0
    seq = seq_start
    fin_tool = tool_id
    if region_tools is not None:
        rr, c_prev, fin_tool = region_records(region_tools, S)
        for (a, c, did, fl, t) in rr:
            t1 = next(t_ for t_, e in enumerate(ends) if e >= c)
            recs.append(Record(round_idx, seq, t1, a, c - a, did, fl, S[a:c], t))
            seq += 1
        cuts = []
    elif kind in (PARSER_FENCE, PARSER_CALL, PARSER_PLAN):
        # region grammars: records need not tile S (text outside a region is not tool input);
        # a single FENCE / CALL tool is the set of one (R24), so FINAL carries -1 outside it
        if kind == PARSER_FENCE:
            fr, c_prev = fence_records(delims[0], max_seg, S)
        elif kind == PARSER_CALL:
            fr, c_prev = call_records(delims[0], max_seg, S)
        else:
            fr, c_prev = plan_records(max_seg, S)
        if kind != PARSER_PLAN:
            fin_tool = region_records([(tool_id, kind, delims[0], max_seg)], S)[2] if tool_id >= 0 else -1
        for (a, c, did, fl) in fr:
            t1 = next(t for t, e in enumerate(ends) if e >= c)
            recs.append(Record(round_idx, seq, t1, a, c - a, did, fl, S[a:c], tool_id))
            seq += 1
        cuts = []
    else:
        cuts = segment(kind, delims, max_seg, S)
    for (c, did, fl) in cuts:
        t1 = next(t for t, e in enumerate(ends) if e >= c)  # min{t : e_t >= c} - 1 (0-based)
        recs.append(Record(round_idx, seq, t1, c_prev, c - c_prev, did, fl, S[c_prev:c], tool_id))
        seq += 1
        c_prev = c
    last = len(tokens) - 1 if tokens else NO_TOKEN
    recs.append(Record(round_idx, seq, last, c_prev, len(S) - c_prev, DELIM_NONE,
                       FLAG_FINAL | (FLAG_CANCELLED if cancelled else 0), S[c_prev:], fin_tool))
    return recs, S
