"""Thin Python binding over libconveyor's C ABI (include/conveyor.h), same call names.

PyTorch is used only for device memory (weights, KV pool) -- every step of the decode
path (embedding, projections, attention, sampling, trigger scan, compaction, publish) runs
in the library's sm_100a kernels.  No CPU fallback: without the library or a B200 the
calls raise.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import capi
from .capi import check


def model_config(shape, dtype: str = "bf16") -> capi.ModelConfig:
    return capi.ModelConfig(shape.L, shape.d, shape.H, shape.Hkv, shape.hd, shape.dff, shape.V,
                            float(shape.eps), float(shape.rope_base), int(shape.eos),
                            capi.DTYPE_BF16 if dtype == "bf16" else capi.DTYPE_FP32)


def tiled_default(shape, dtype: str) -> bool:
    """Tile-major projection weights (CVY_ENGINE_TILED_WEIGHTS) unless the shape cannot be
    tiled or CVY_TILED_WEIGHTS=0."""
    import os
    if dtype != "bf16" or os.environ.get("CVY_TILED_WEIGHTS", "1") == "0":
        return False
    rows = [(shape.H + 2 * shape.Hkv) * shape.hd, shape.d, 2 * shape.dff]
    cols = [shape.d, shape.H * shape.hd, shape.dff]
    return all(r % 128 == 0 for r in rows) and all(c % 64 == 0 for c in cols)


class DeviceModel:
    """Weights + KV pool as torch CUDA tensors (borrowed by the engine).  `tiled`: pack the
    projection weights tile-major (cvy_pack_weights_tiled); engines over this model get
    CVY_ENGINE_TILED_WEIGHTS automatically."""

    def __init__(self, shape, dtype: str, n_pages: int, seed: int, device: int = 0, tiled: bool | None = None):
        import torch
        self.shape = shape
        self.n_pages = n_pages
        self.dtype = dtype
        self.cfg = model_config(shape, dtype)
        sizes = capi.WeightSizes()
        check(capi.lib().cvy_weight_sizes_for(ctypes.byref(self.cfg), n_pages, ctypes.byref(sizes)))
        dev = torch.device("cuda", device)
        self.tensors = {}
        for name, _ in capi.WeightSizes._fields_:
            nbytes = getattr(sizes, name)
            self.tensors[name] = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=dev)
        self.tensors["kv_pool"].zero_()
        self.w = capi.Weights(*[self.tensors[n].data_ptr() for n, _ in capi.WeightSizes._fields_])
        check(capi.lib().cvy_init_synthetic_weights(ctypes.byref(self.cfg), ctypes.byref(self.w), seed, device))
        self.tiled = tiled_default(shape, dtype) if tiled is None else bool(tiled)
        if self.tiled:
            check(capi.lib().cvy_pack_weights_tiled(ctypes.byref(self.cfg), ctypes.byref(self.w), device))

    def tensor(self, name):
        return self.tensors[name]


@dataclass
class Record:
    req_id: int
    round: int
    seq: int
    step: int
    token_index: int
    byte_offset: int
    byte_len: int
    delim_id: int
    flags: int
    slot: int
    data: bytes
    tool: int = -1


class Engine:
    def __init__(self, model: DeviceModel, vocab: list[bytes], max_slots: int = 64, n_pages: int | None = None,
                 max_pages_per_slot: int = 256, ring_records: int | None = None, round_bytes: int = 1 << 16,
                 round_tokens: int = 4096, input_cap: int = 4096, forced_cap: int = 4096, device: int = 0,
                 flags: int = 0):
        from inputs.vocab import table
        self.model = model
        self.V = model.shape.V
        tb, ln = table(vocab)
        if ring_records is None:
            ring_records = 1
            while ring_records < 64 * max_slots:
                ring_records <<= 1
        if getattr(model, "tiled", False):
            flags |= capi.ENGINE_TILED_WEIGHTS
        self.ecfg = capi.EngineConfig(max_slots, n_pages if n_pages is not None else model.n_pages, max_pages_per_slot,
                                      ring_records, round_bytes, round_tokens, input_cap, forced_cap, device, flags)
        h = ctypes.c_void_p()
        check(capi.lib().cvy_engine_create(ctypes.byref(model.cfg), ctypes.byref(self.ecfg), ctypes.byref(model.w),
                                           tb, ln, ctypes.byref(h)))
        self.h = h
        self._seg_buf = (capi.Segment * 4096)()
        self._byte_buf = ctypes.create_string_buffer(1 << 22)

    def close(self):
        if getattr(self, "h", None):
            capi.lib().cvy_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- the five calls of the paper's problem statement (+ lifecycle helpers)
    def register_tool(self, name: str, parser: int, delims=(), max_segment_bytes: int = 0) -> int:
        n = len(delims)
        bufs = [(ctypes.c_uint8 * len(d)).from_buffer_copy(d) for d in delims]
        arr = (ctypes.POINTER(ctypes.c_uint8) * max(n, 1))(*[ctypes.cast(b, ctypes.POINTER(ctypes.c_uint8)) for b in bufs])
        lens = (ctypes.c_uint32 * max(n, 1))(*[len(d) for d in delims])
        desc = capi.ToolDesc(name.encode(), parser, n, arr if n else None, lens if n else None, max_segment_bytes)
        tid = ctypes.c_int32()
        check(capi.lib().cvy_register_tool(self.h, ctypes.byref(desc), ctypes.byref(tid)))
        return tid.value

    def submit_request(self, prompt, max_new_tokens: int, tool_id: int = -1, mode: int = capi.MODE_PARTIAL,
                       forced=None, synth_prefix_len: int = 0, synth_seed: int = 0, reserve_tokens: int = 0,
                       allow_full: bool = False, tool_set=None):
        p = np.ascontiguousarray(np.asarray(prompt, dtype=np.int32))
        f = np.ascontiguousarray(np.asarray(forced if forced is not None else [], dtype=np.int32))
        ts = np.ascontiguousarray(np.asarray(tool_set if tool_set else [], dtype=np.int32))
        i32p = ctypes.POINTER(ctypes.c_int32)
        desc = capi.RequestDesc(tool_id, mode, p.ctypes.data_as(i32p), len(p), synth_prefix_len, synth_seed,
                                max_new_tokens, f.ctypes.data_as(i32p) if len(f) else None, len(f), reserve_tokens,
                                ts.ctypes.data_as(i32p) if len(ts) else None, len(ts))
        rid = ctypes.c_uint64()
        st = capi.lib().cvy_submit_request(self.h, ctypes.byref(desc), ctypes.byref(rid))
        if allow_full and st == capi.CVY_E_FULL:
            return None
        check(st)
        return rid.value

    def step(self) -> capi.StepInfo:
        info = capi.StepInfo()
        check(capi.lib().cvy_step(self.h, ctypes.byref(info)))
        return info

    def sync(self):
        check(capi.lib().cvy_sync(self.h))

    def poll_segments(self, with_bytes: bool = True) -> list[Record]:
        out = []
        while True:
            n = ctypes.c_uint32()
            used = ctypes.c_size_t()
            st = capi.lib().cvy_poll_segments(self.h, self._seg_buf, len(self._seg_buf), ctypes.byref(n),
                                              self._byte_buf if with_bytes else None,
                                              len(self._byte_buf) if with_bytes else 0, ctypes.byref(used))
            if st == capi.CVY_E_AGAIN:
                return out
            check(st)
            raw = self._byte_buf.raw[:used.value] if with_bytes else b""
            off = 0
            for i in range(n.value):
                s = self._seg_buf[i]
                data = raw[off:off + s.byte_len] if with_bytes else b""
                off += s.byte_len if with_bytes else 0
                out.append(Record(s.req_id, s.round, s.seq, s.step, s.token_index, s.byte_offset, s.byte_len,
                                  s.delim_id, s.flags, s.slot, data, s.tool))
            if n.value < len(self._seg_buf):
                return out

    def inject_observation(self, req_id: int, tokens, max_new_tokens: int, forced=None):
        t = np.ascontiguousarray(np.asarray(tokens, dtype=np.int32))
        f = np.ascontiguousarray(np.asarray(forced if forced is not None else [], dtype=np.int32))
        i32p = ctypes.POINTER(ctypes.c_int32)
        check(capi.lib().cvy_inject_observation(self.h, req_id, t.ctypes.data_as(i32p) if len(t) else None, len(t),
                                                max_new_tokens, f.ctypes.data_as(i32p) if len(f) else None, len(f)))

    def cancel_request(self, req_id: int):
        check(capi.lib().cvy_cancel_request(self.h, req_id))

    def release_request(self, req_id: int):
        check(capi.lib().cvy_release_request(self.h, req_id))

    def request_state(self, req_id: int) -> int:
        return capi.lib().cvy_request_state(self.h, req_id)

    def round_tokens(self, req_id: int, cap: int = 1 << 16) -> list[int]:
        buf = (ctypes.c_int32 * cap)()
        n = ctypes.c_uint32()
        check(capi.lib().cvy_round_tokens(self.h, req_id, buf, cap, ctypes.byref(n)))
        return list(buf[:n.value])

    def debug_logits(self, req_id: int) -> np.ndarray:
        out = np.empty(self.V, dtype=np.float32)
        check(capi.lib().cvy_debug_logits(self.h, req_id, out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), self.V))
        return out

    def debug_buffer(self, which: int) -> bytes:
        n = ctypes.c_size_t()
        check(capi.lib().cvy_debug_buffer(self.h, which, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        check(capi.lib().cvy_debug_buffer(self.h, which, buf, n.value, ctypes.byref(n)))
        return buf.raw

    def perf(self) -> capi.PerfInfo:
        p = capi.PerfInfo()
        check(capi.lib().cvy_perf(self.h, ctypes.byref(p)))
        return p

    def set_kernel_timing(self, on: bool):
        check(capi.lib().cvy_set_kernel_timing(self.h, 1 if on else 0))

    def kernel_times(self):
        buf = (capi.KernelTime * 4096)()
        n = ctypes.c_uint32()
        check(capi.lib().cvy_kernel_times(self.h, buf, len(buf), ctypes.byref(n)))
        return [(buf[i].kind, buf[i].layer, buf[i].ms) for i in range(n.value)]

    def set_kernel_spans(self, on: bool):
        check(capi.lib().cvy_set_kernel_spans(self.h, 1 if on else 0))

    def kernel_spans(self):
        """[(kind, layer, chain, t0_ns, t1_ns)] of the last span-recording step (cvy_kernel_spans)."""
        buf = (capi.KernelSpan * 2048)()
        n = ctypes.c_uint32()
        check(capi.lib().cvy_kernel_spans(self.h, buf, len(buf), ctypes.byref(n)))
        return [(buf[i].kind, buf[i].layer, buf[i].chain, buf[i].t0_ns, buf[i].t1_ns) for i in range(n.value)]

    def stream_ptr(self) -> int:
        return capi.lib().cvy_stream(self.h) or 0


def stats_allgather(engines: list[Engine]) -> np.ndarray:
    arr = (ctypes.c_void_p * len(engines))(*[e.h.value for e in engines])
    out = np.zeros((len(engines), 8), dtype=np.uint64)
    check(capi.lib().cvy_stats_allgather(arr, len(engines), out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))))
    return out


def debug_gemm(W, X, N: int, K: int, B: int, iters: int = 1, device: int = 0, X_lo=None):
    """Y = (X + X_lo) W^T through the decode step's tcgen05 GEMM kernel (test/measurement hook):
    X is the activation's hi plane, X_lo (optional, default zero) its lo plane.
    W, X, X_lo: bf16 CUDA tensors; returns (Y fp32 CUDA tensor [B][N], mean ms per launch)."""
    import os
    import torch
    Y = torch.empty((B, N), dtype=torch.float32, device=W.device)
    ms = ctypes.c_float()
    if X_lo is not None:
        X = torch.cat([X[:B], X_lo[:B]]).contiguous()
        os.environ["CVY_DEBUG_GEMM_LO"] = "1"
    try:
        check(capi.lib().cvy_debug_gemm(W.data_ptr(), X.data_ptr(), Y.data_ptr(), N, K, B, iters, device,
                                        ctypes.byref(ms)))
    finally:
        os.environ.pop("CVY_DEBUG_GEMM_LO", None)
    return Y, ms.value
