"""CPU oracle for the Conveyor (arXiv 2406.00059) decode hot path -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product library (paper_2406_00059_b200) never
imports it and shares no code with it.

  O-1 (oracle.c)   decoder forward, fp64
  O-2 (oracle.c +  byte-stream segmentation and the
       scan.py)    per-round segment records
  O-3 (latency.py) L_old, Eq. 1/2 bounds, improvement,
                   the partial-vs-sequential DES
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain C, OpenMP over rows/requests)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB_PATH, _SRC, "-lm"])
    return _LIB_PATH


class _Model(ctypes.Structure):
    _fields_ = [("L", ctypes.c_int), ("d", ctypes.c_int), ("H", ctypes.c_int),
                ("Hkv", ctypes.c_int), ("hd", ctypes.c_int), ("dff", ctypes.c_int),
                ("V", ctypes.c_int), ("eps", ctypes.c_double), ("rope_base", ctypes.c_double)]


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        vp, i32, u64, dbl = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_double
        L.orc_weights_create.restype = vp
        L.orc_weights_create.argtypes = [ctypes.POINTER(_Model), u64, i32, i32]
        L.orc_weights_destroy.argtypes = [vp]
        L.orc_req_create.restype = vp
        L.orc_req_create.argtypes = [vp, i32]
        L.orc_req_destroy.argtypes = [vp]
        L.orc_req_synth_prefix.argtypes = [vp, i32, u64]
        L.orc_req_synth_prefix.restype = i32
        L.orc_step.argtypes = [ctypes.POINTER(vp), i32, ctypes.POINTER(ctypes.c_int32),
                               ctypes.POINTER(dbl)]
        L.orc_step.restype = i32
        L.orc_argmax.argtypes = [ctypes.POINTER(dbl), i32]
        L.orc_argmax.restype = i32
        L.orc_hash_value.argtypes = [u64, u64, u64, dbl, i32]
        L.orc_hash_value.restype = dbl
        L.orc_bf16_round.argtypes = [dbl]
        L.orc_bf16_round.restype = dbl
        L.orc_dump_tensor.argtypes = [vp, u64, ctypes.POINTER(dbl)]
        L.orc_dump_tensor.restype = i32
        L.orc_num_threads.restype = i32
        L.orc_segment.argtypes = [i32, i32, ctypes.POINTER(ctypes.c_uint8), ctypes.POINTER(i32), i32,
                                  ctypes.POINTER(ctypes.c_uint8), i32, ctypes.POINTER(i32),
                                  ctypes.POINTER(i32), ctypes.POINTER(i32), i32]
        L.orc_segment.restype = i32
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def num_threads() -> int:
    return lib().orc_num_threads()


def hash_value(seed: int, tid: int, i: int, a: float, bf16: bool) -> float:
    return lib().orc_hash_value(seed, tid, i, a, int(bf16))


def bf16_round(v: float) -> float:
    return lib().orc_bf16_round(v)


# tensor ids
def tid_embed() -> int:
    return 0


def tid_layer(l: int, which: str) -> int:
    return 1 + 8 * l + {"wq": 0, "wk": 1, "wv": 2, "wo": 3, "wg": 4, "wu": 5, "wd": 6}[which]


def tid_lm_head(L: int) -> int:
    return 1 + 8 * L


class Weights:
    """Random-init weights (counter hash), fp32 or bf16 values.  Activations are exact (fp64);
    a bf16 model rounds only its KV cache to bf16 on append."""

    def __init__(self, shape, seed: int, bf16: bool, cache: bool | None = None):
        self.shape = shape
        self.bf16 = bf16
        m = _Model(shape.L, shape.d, shape.H, shape.Hkv, shape.hd, shape.dff, shape.V,
                   shape.eps, shape.rope_base)
        if cache is None:
            cache = shape.n_params_streamed < 200_000_000
        self._h = lib().orc_weights_create(ctypes.byref(m), seed, int(bf16), int(cache))

    def tensor(self, tid: int, rows: int, cols: int) -> np.ndarray:
        out = np.empty((rows, cols), dtype=np.float64)
        lib().orc_dump_tensor(self._h, tid, _dp(out))
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_weights_destroy(self._h)
            self._h = None


class Request:
    """Per-request KV cache (fp64, values rounded to the cache dtype)."""

    def __init__(self, weights: Weights, max_ctx: int):
        self.w = weights
        self._h = lib().orc_req_create(weights._h, max_ctx)

    def synth_prefix(self, prefix_len: int, synth_seed: int):
        if lib().orc_req_synth_prefix(self._h, prefix_len, synth_seed) != 0:
            raise ValueError("prefix longer than max_ctx")

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_req_destroy(self._h)
            self._h = None


def step(reqs: list[Request], tokens) -> np.ndarray:
    """One decode step for independent requests; returns logits [n][V] (fp64)."""
    n = len(reqs)
    V = reqs[0].w.shape.V
    arr = (ctypes.c_void_p * n)(*[r._h for r in reqs])
    tok = np.ascontiguousarray(np.asarray(tokens, dtype=np.int32))
    out = np.empty((n, V), dtype=np.float64)
    rc = lib().orc_step(arr, n, tok.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), _dp(out))
    if rc != 0:
        raise ValueError("orc_step: context full or token out of range")
    return out


def argmax(logits: np.ndarray) -> int:
    x = np.ascontiguousarray(logits, dtype=np.float64)
    return lib().orc_argmax(_dp(x), x.shape[0])


PARSER_LITERAL, PARSER_JSON_MEMBER, PARSER_JSON_OBJECT, PARSER_FENCE, PARSER_CALL, PARSER_PLAN = 0, 1, 2, 3, 4, 5
FLAG_FINAL, FLAG_OVERFLOW, FLAG_CANCELLED, FLAG_OPEN, FLAG_CLOSE = 1, 2, 4, 8, 16
DELIM_NONE = 0xFFFF


def fence_records(tag: bytes, max_seg: int, S: bytes):
    """FENCE region grammar (NEXT-2; reading R21) -- the paper's CodeGen indicators:
    "We use the markdown code block syntax ```python and ``` as the indicators for the start
    and end of the tool"; a complete line of code inside is one partial-
    execution piece ("a complete line of Python code is decoded").

    Plain definition, step by step:
      1. Line units: S is cut after every '\n' byte; a run of max_seg bytes without '\n' is
         cut too (an overflow unit), and the rest of that line is a continuation unit.
      2. A unit is a marker only if it starts a line (is not a continuation): the open marker
         is exactly b"```" + tag + b"\n", the close marker exactly b"```\n".
      3. Walking the units in order with a region flag (initially outside):
           outside: the open marker -> OPEN record, region opens; anything else -> nothing;
           inside:  the close marker -> CLOSE record, region closes;
                    any other '\n'-terminated unit -> piece record (delim_id 0);
                    an overflow unit -> piece record with OVERFLOW (delim_id NONE).
      4. The trailing incomplete unit (no '\n', shorter than max_seg) is left for FINAL.
    Returns (records [(start, end, delim_id, flags)], start of the trailing unit)."""
    open_m, close_m = b"```" + tag + b"\n", b"```\n"
    units = []          # (start, end, ends_with_newline, is_continuation)
    start, cont = 0, False
    for i in range(len(S)):
        if S[i] == 0x0A:
            units.append((start, i + 1, True, cont))
            start, cont = i + 1, False
        elif i + 1 - start == max_seg:
            units.append((start, i + 1, False, cont))
            start, cont = i + 1, True
    recs = []
    inside = False
    for (a, b, nl, c) in units:
        u = S[a:b]
        if not inside:
            if nl and not c and u == open_m:
                recs.append((a, b, 0, FLAG_OPEN))
                inside = True
        else:
            if nl and not c and u == close_m:
                recs.append((a, b, 0, FLAG_CLOSE))
                inside = False
            elif nl:
                recs.append((a, b, 0, 0))
            else:
                recs.append((a, b, DELIM_NONE, FLAG_OVERFLOW))
    return recs, start


def segment(kind: int, delims: list[bytes], max_seg: int, stream: bytes):
    """Cuts of a byte stream (O-2): list of (end_offset, delim_id, flags)."""
    buf = np.zeros(64, dtype=np.uint8)
    lens = np.zeros(8, dtype=np.int32)
    for i, dlm in enumerate(delims):
        buf[8 * i: 8 * i + len(dlm)] = np.frombuffer(dlm, dtype=np.uint8)
        lens[i] = len(dlm)
    S = np.frombuffer(stream, dtype=np.uint8) if len(stream) else np.zeros(1, dtype=np.uint8)
    cap = len(stream) + 1
    ce = np.zeros(cap, dtype=np.int32)
    di = np.zeros(cap, dtype=np.int32)
    fl = np.zeros(cap, dtype=np.int32)
    u8p = ctypes.POINTER(ctypes.c_uint8)
    i32p = ctypes.POINTER(ctypes.c_int32)
    n = lib().orc_segment(kind, len(delims), buf.ctypes.data_as(u8p), lens.ctypes.data_as(i32p),
                          max_seg, S.ctypes.data_as(u8p), len(stream), ce.ctypes.data_as(i32p),
                          di.ctypes.data_as(i32p), fl.ctypes.data_as(i32p), cap)
    if n < 0:
        raise RuntimeError("orc_segment overflow")
    return [(int(ce[j]), int(di[j]), int(fl[j])) for j in range(n)]


def _line_units(S: bytes, max_seg: int):
    """Step 1 shared by the line-based grammars: '\n'-terminated units and max_seg cuts
    (start, end, ends_with_newline, is_continuation)."""
    units = []
    start, cont = 0, False
    for i in range(len(S)):
        if S[i] == 0x0A:
            units.append((start, i + 1, True, cont))
            start, cont = i + 1, False
        elif i + 1 - start == max_seg:
            units.append((start, i + 1, False, cont))
            start, cont = i + 1, True
    return units, start


def call_records(tag: bytes, max_seg: int, S: bytes):
    """CALL region grammar (NEXT-2; reading R22).  SPEC.md:80: "the sentinel
    `@call NAME ` begins a region for tool NAME (ToolStart fires as soon as NAME and the
    trailing space are seen ...); the remainder up to a balanced-brace end is a JSON object ...
    emitting FieldComplete ... region closes at the brace balance returning to zero"; the
    paper's Search/Database trigger is "when Conveyor identifies the function name of the
    tool".  Step by step, byte by byte with a cursor c (start of the
    current piece or line):
      outside a region: a line (bytes since the last '\n' or stream start, not a continuation
        of a max_seg cut) equal to b"@call " + tag + b" " opens the region -> OPEN record
        [c, p), c = p; a '\n' sets c = p; a line reaching max_seg bytes sets c = p and makes
        the rest of the line a continuation (never a marker);
      inside: the JSON automaton of JSON_MEMBER (R10-R11, depth/in_str/esc from 0): ',' at
        depth 1 -> piece record (delim 0), the bracket returning depth to 0 -> CLOSE record
        (delim 1) and the region ends (the rest of that line is not at a line start);
        a piece reaching max_seg bytes -> OVERFLOW record (delim NONE).
    FINAL = S[c, |S|).  Returns (records [(start, end, delim_id, flags)], c)."""
    marker = b"@call " + tag + b" "
    recs = []
    inside = False
    c = 0
    line_ok = True            # the current line started at c and is not a continuation
    depth = in_str = esc = 0
    for i in range(len(S)):
        p = i + 1
        b = S[i]
        if not inside:
            if b == 0x0A:
                c, line_ok = p, True
            elif line_ok and S[c:p] == marker:
                recs.append((c, p, 0, FLAG_OPEN))
                inside, c = True, p
                depth = in_str = esc = 0
            elif p - c == max_seg:
                c, line_ok = p, False
            continue
        hit = -1
        if in_str:
            if esc:
                esc = 0
            elif b == 0x5C:
                esc = 1
            elif b == 0x22:
                in_str = 0
        elif depth == 0:
            if b in (0x7B, 0x5B):
                depth = 1
        else:
            if b == 0x22:
                in_str = 1
            elif b in (0x7B, 0x5B):
                depth = min(depth + 1, 127)
            elif b in (0x7D, 0x5D):
                depth -= 1
                if depth == 0:
                    hit = 1
            elif b == 0x2C and depth == 1:
                hit = 0
        if hit == 1:
            recs.append((c, p, 1, FLAG_CLOSE))
            inside, c, line_ok = False, p, (b == 0x0A)
        elif hit == 0:
            recs.append((c, p, 0, 0))
            c = p
        elif p - c == max_seg:
            recs.append((c, p, DELIM_NONE, FLAG_OVERFLOW))
            c = p
    return recs, c


def region_records(tools, S: bytes):
    """Multi-tool region grammars (NEXT-2; reading R24): one request holds a SET of
    region tools -- FENCE tools ("the markdown code block syntax ```python and ``` as the
    indicators for the start and end of the tool") and CALL tools ("when Conveyor
    identifies the function name of the tool") -- and the open marker that
    appears selects the tool.  tools: [(tool_id, kind, tag, max_seg)] with kind FENCE or CALL.
    Step by step, byte by byte with a cursor c (start of the current line unit or piece):
      outside a region (line_ok: the current line started at c and is neither a continuation of
      a cut nor the rest of a line after a CALL close; M = min max_seg over the set):
        '\n': if line_ok and S[c:p] == b"```" + tag + b"\n" of a FENCE tool -> OPEN record of
              that tool, its region opens; c = p, line_ok = True;
        else if line_ok and S[c:p] == b"@call " + tag + b" " of a CALL tool -> OPEN record of
              that tool, its region opens with the JSON automaton at its start state; c = p;
        else if p - c == M: c = p, line_ok = False;
      inside a FENCE region (its max_seg; cont: the unit continues a cut line):
        '\n': the unit not cont and equal to b"```\n" -> CLOSE record, region closes;
              any other unit -> piece record (delim 0); c = p, cont = False;
        else if p - c == max_seg -> piece record with OVERFLOW (delim NONE); c = p, cont = True;
      inside a CALL region (its max_seg): the JSON automaton of JSON_MEMBER (R10-R11): ',' at
        depth 1 -> piece record (delim 0); the bracket returning depth to 0 -> CLOSE record
        (delim 1), the region closes and the rest of that line is not at a line start; a piece
        reaching max_seg bytes -> OVERFLOW record (delim NONE).
    The lowest tool id wins if two markers match at one byte (impossible for distinct tags).
    With one tool this is fence_records / call_records.  FINAL = S[c, |S|), carrying the tool of
    the region open at the end (-1 outside).
    Returns (records [(start, end, delim_id, flags, tool_id)], c, tool of the FINAL)."""
    tools = sorted(tools)
    M = min(t[3] for t in tools)
    fence_m = {t[0]: b"```" + t[2] + b"\n" for t in tools if t[1] == PARSER_FENCE}
    call_m = {t[0]: b"@call " + t[2] + b" " for t in tools if t[1] == PARSER_CALL}
    kind = {t[0]: t[1] for t in tools}
    mseg = {t[0]: t[3] for t in tools}
    recs = []
    region = None
    c = 0
    line_ok = True
    cont = False
    depth = in_str = esc = 0
    for i in range(len(S)):
        p = i + 1
        b = S[i]
        if region is None:
            if b == 0x0A:
                hit = [t for t, m in fence_m.items() if line_ok and S[c:p] == m]
                if hit:
                    recs.append((c, p, 0, FLAG_OPEN, hit[0]))
                    region, cont = hit[0], False
                c, line_ok = p, True
                continue
            hit = [t for t, m in call_m.items() if line_ok and S[c:p] == m]
            if hit:
                recs.append((c, p, 0, FLAG_OPEN, hit[0]))
                region, c = hit[0], p
                depth = in_str = esc = 0
            elif p - c == M:
                c, line_ok = p, False
            continue
        if kind[region] == PARSER_FENCE:
            if b == 0x0A:
                if not cont and S[c:p] == b"```\n":
                    recs.append((c, p, 0, FLAG_CLOSE, region))
                    region, line_ok = None, True
                else:
                    recs.append((c, p, 0, 0, region))
                c, cont = p, False
            elif p - c == mseg[region]:
                recs.append((c, p, DELIM_NONE, FLAG_OVERFLOW, region))
                c, cont = p, True
            continue
        hit = -1
        if in_str:
            if esc:
                esc = 0
            elif b == 0x5C:
                esc = 1
            elif b == 0x22:
                in_str = 0
        elif depth == 0:
            if b in (0x7B, 0x5B):
                depth = 1
        else:
            if b == 0x22:
                in_str = 1
            elif b in (0x7B, 0x5B):
                depth = min(depth + 1, 127)
            elif b in (0x7D, 0x5D):
                depth -= 1
                if depth == 0:
                    hit = 1
            elif b == 0x2C and depth == 1:
                hit = 0
        if hit == 1:
            recs.append((c, p, 1, FLAG_CLOSE, region))
            region, c, line_ok = None, p, False
        elif hit == 0:
            recs.append((c, p, 0, 0, region))
            c = p
        elif p - c == mseg[region]:
            recs.append((c, p, DELIM_NONE, FLAG_OVERFLOW, region))
            c = p
    return recs, c, (-1 if region is None else region)


def plan_records(max_seg: int, S: bytes):
    r"""PLAN line grammar (NEXT-2; reading R23).  SPEC.md:81: "each newline-
    terminated line matching `#E<digits> = <Name>[<args>]` is one ToolData stage piece
    carrying the full line; non-matching lines are PlainText" (LLMCompiler plans; the paper's
    planning trigger is "a complete stage of the plan is generated").
    Line units as in FENCE (max_seg cuts, continuations never match); a unit is a stage iff
    it is not a continuation, ends with '\n' and its bytes match
    #E[0-9]+ = [A-Za-z0-9_]+\[[^\n]*\]\n  exactly -> piece record (delim 0).
    FINAL = the trailing incomplete unit."""
    import re
    pat = re.compile(rb"#E[0-9]+ = [A-Za-z0-9_]+\[[^\n]*\]\n")
    units, tail = _line_units(S, max_seg)
    recs = [(a, b, 0, 0) for (a, b, nl, c) in units if nl and not c and pat.fullmatch(S[a:b])]
    return recs, tail
