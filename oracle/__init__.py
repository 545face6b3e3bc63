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
        L.orc_weights_create.argtypes = [ctypes.POINTER(_Model), u64, i32, i32, i32]
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
    """Random-init weights (counter hash), fp32 or bf16 values; act_bf16 selects the bf16
    storage-point contract (R4) for activations."""

    def __init__(self, shape, seed: int, bf16: bool, act_bf16: bool, cache: bool | None = None):
        self.shape = shape
        self.bf16 = bf16
        self.act_bf16 = act_bf16
        m = _Model(shape.L, shape.d, shape.H, shape.Hkv, shape.hd, shape.dff, shape.V,
                   shape.eps, shape.rope_base)
        if cache is None:
            cache = shape.n_params_streamed < 200_000_000
        self._h = lib().orc_weights_create(ctypes.byref(m), seed, int(bf16), int(act_bf16), int(cache))

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


PARSER_LITERAL, PARSER_JSON_MEMBER, PARSER_JSON_OBJECT, PARSER_FENCE = 0, 1, 2, 3
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
