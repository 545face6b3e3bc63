"""ctypes mirror of include/conveyor.h (argument marshalling only -- every step of the
decode path runs inside libconveyor.so's CUDA kernels).  Loading fails loudly if the
library is missing: there is no CPU fallback."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CVY_LIB_PATH") or os.path.join(HERE, "libconveyor.so")  # override: A/B builds

CVY_OK, CVY_E_INVAL, CVY_E_NOMEM, CVY_E_FULL, CVY_E_AGAIN = 0, -1, -2, -3, -4
CVY_E_NOTFOUND, CVY_E_STATE, CVY_E_DUP, CVY_E_CUDA, CVY_E_NCCL = -5, -6, -7, -8, -9
STATUS_NAMES = {0: "OK", -1: "E_INVAL", -2: "E_NOMEM", -3: "E_FULL", -4: "E_AGAIN", -5: "E_NOTFOUND",
                -6: "E_STATE", -7: "E_DUP", -8: "E_CUDA", -9: "E_NCCL"}
DTYPE_BF16, DTYPE_FP32 = 0, 1
PARSER_LITERAL, PARSER_JSON_MEMBER, PARSER_JSON_OBJECT, PARSER_FENCE, PARSER_CALL, PARSER_PLAN = 0, 1, 2, 3, 4, 5
MODE_PARTIAL, MODE_SEQUENTIAL = 0, 1
SEG_FINAL, SEG_OVERFLOW, SEG_CANCELLED, SEG_OPEN, SEG_CLOSE = 1, 2, 4, 8, 16
DELIM_NONE = 0xFFFF
NO_TOKEN = 0xFFFFFFFF
ENGINE_NO_GRAPH, ENGINE_DEBUG_LOGITS, ENGINE_SCAN_OFF, ENGINE_NO_PDL = 1, 2, 4, 8
ENGINE_CHUNKED_PREFILL = 32
ENGINE_TILED_WEIGHTS = 64

c_i32, c_u32, c_u64, c_u16, c_f32, c_f64, c_sz, c_vp = (ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint64,
                                                         ctypes.c_uint16, ctypes.c_float, ctypes.c_double,
                                                         ctypes.c_size_t, ctypes.c_void_p)


class ModelConfig(ctypes.Structure):
    _fields_ = [("n_layers", c_i32), ("d_model", c_i32), ("n_heads", c_i32), ("n_kv_heads", c_i32),
                ("head_dim", c_i32), ("d_ff", c_i32), ("vocab", c_i32), ("rms_eps", c_f32),
                ("rope_base", c_f64), ("eos_id", c_i32), ("dtype", c_i32)]


class EngineConfig(ctypes.Structure):
    _fields_ = [("max_slots", c_u32), ("n_pages", c_u32), ("max_pages_per_slot", c_u32),
                ("ring_records", c_u32), ("round_bytes", c_u32), ("round_tokens", c_u32),
                ("input_cap", c_u32), ("forced_cap", c_u32), ("device", c_i32), ("flags", c_u32)]


class Weights(ctypes.Structure):
    _fields_ = [("embed", c_vp), ("lm_head", c_vp), ("final_norm", c_vp), ("attn_norm", c_vp),
                ("mlp_norm", c_vp), ("wqkv", c_vp), ("wo", c_vp), ("wgu", c_vp), ("wd", c_vp),
                ("kv_pool", c_vp)]


class WeightSizes(ctypes.Structure):
    _fields_ = [(n, c_sz) for n in ("embed", "lm_head", "final_norm", "attn_norm", "mlp_norm", "wqkv",
                                    "wo", "wgu", "wd", "kv_pool")]


class ToolDesc(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("parser", c_i32), ("n_delims", c_u32),
                ("delims", ctypes.POINTER(ctypes.POINTER(ctypes.c_uint8))),
                ("delim_lens", ctypes.POINTER(c_u32)), ("max_segment_bytes", c_u32)]


class RequestDesc(ctypes.Structure):
    _fields_ = [("tool_id", c_i32), ("mode", c_i32), ("prompt", ctypes.POINTER(c_i32)), ("prompt_len", c_u32),
                ("synth_prefix_len", c_u32), ("synth_seed", c_u64), ("max_new_tokens", c_u32),
                ("forced", ctypes.POINTER(c_i32)), ("forced_len", c_u32), ("reserve_tokens", c_u32),
                ("tool_set", ctypes.POINTER(c_i32)), ("n_tool_set", c_u32)]


class StepInfo(ctypes.Structure):
    _fields_ = [("step", c_u64), ("n_active", c_u32), ("n_generated", c_u32), ("n_segments", c_u32),
                ("n_finished", c_u32), ("step_ms", c_f32)]


class Segment(ctypes.Structure):
    _fields_ = [("req_id", c_u64), ("round", c_u32), ("seq", c_u32), ("step", c_u32), ("token_index", c_u32),
                ("byte_offset", c_u32), ("byte_len", c_u32), ("delim_id", c_u16), ("flags", c_u16),
                ("slot", c_u16), ("tool", ctypes.c_int16)]


class KernelTime(ctypes.Structure):
    _fields_ = [("kind", c_i32), ("layer", c_i32), ("ms", c_f32)]


class KernelSpan(ctypes.Structure):
    _fields_ = [("kind", c_i32), ("layer", c_i32), ("chain", c_i32), ("t0_ns", c_u64), ("t1_ns", c_u64)]


KERNEL_KINDS = {0: "embed", 1: "gemm_qkv", 2: "attention", 3: "attention_merge", 4: "gemm_o", 5: "gemm_gate_up",
                6: "gemm_down", 7: "gemm_lm_head+sample_scan"}


class PerfInfo(ctypes.Structure):
    _fields_ = [("last_step_ms", c_f32), ("launches_per_step", c_u32), ("slots_bucket", c_u32)]


assert ctypes.sizeof(Segment) == 40

# ------------------------------------------------------------------ native host runtime
class PiecePlan(ctypes.Structure):
    _fields_ = [("skip", c_i32), ("abort", c_i32), ("cost_ms", ctypes.c_double), ("instance", c_i32),
                ("n_deps", c_u32), ("deps", c_i32 * 8)]


PLAN_FN = ctypes.CFUNCTYPE(None, c_vp, c_u32, c_u32, c_u32, ctypes.POINTER(ctypes.c_uint8), c_u32, ctypes.c_uint16,
                           ctypes.POINTER(PiecePlan))


class RuntimeConfig(ctypes.Structure):
    _fields_ = [("mode", c_i32), ("n_workers", c_u32), ("max_inflight", c_u32), ("plan", PLAN_FN),
                ("plan_user", c_vp), ("poll_sleep_us", c_u32)]


class RoundDesc(ctypes.Structure):
    _fields_ = [("forced", ctypes.POINTER(c_i32)), ("forced_len", c_u32), ("tool_id", c_i32),
                ("observation", ctypes.POINTER(c_i32)), ("observation_len", c_u32)]


class RtRequest(ctypes.Structure):
    _fields_ = [("prompt", ctypes.POINTER(c_i32)), ("prompt_len", c_u32), ("synth_prefix_len", c_u32),
                ("synth_seed", c_u64), ("rounds", ctypes.POINTER(RoundDesc)), ("n_rounds", c_u32),
                ("t_arrival", ctypes.c_double)]


class RtRequestLog(ctypes.Structure):
    _fields_ = [("req_id", c_u64), ("t_arrival", ctypes.c_double), ("t_submit", ctypes.c_double),
                ("t_done", ctypes.c_double),
                ("t_abort", ctypes.c_double), ("n_rounds_run", c_u32), ("aborted", c_u32)]


class RtRoundLog(ctypes.Structure):
    _fields_ = [("t_start", ctypes.c_double), ("t_final", ctypes.c_double), ("n_pieces", c_u32)]


class RtPieceLog(ctypes.Structure):
    _fields_ = [("t_avail", ctypes.c_double), ("t_dispatch", ctypes.c_double), ("t_begin", ctypes.c_double),
                ("t_end", ctypes.c_double), ("cost_ms", ctypes.c_double), ("instance", c_i32),
                ("token_index", c_u32), ("n_deps", c_u32), ("deps", c_i32 * 8)]


class RtStats(ctypes.Structure):
    _fields_ = [("steps", c_u64), ("records", c_u64), ("pieces", c_u64), ("injections", c_u64), ("cancels", c_u64),
                ("wall_s", ctypes.c_double), ("poller_cpu_s", ctypes.c_double), ("dispatch_cpu_s", ctypes.c_double),
                ("driver_cpu_s", ctypes.c_double), ("worker_cpu_s", ctypes.c_double)]


# name -> (restype, argtypes): every symbol declared in include/conveyor.h
PROTOTYPES = {
    "cvy_abi_version": (c_i32, []),
    "cvy_last_error": (ctypes.c_char_p, []),
    "cvy_weight_sizes_for": (c_i32, [ctypes.POINTER(ModelConfig), c_u32, ctypes.POINTER(WeightSizes)]),
    "cvy_init_synthetic_weights": (c_i32, [ctypes.POINTER(ModelConfig), ctypes.POINTER(Weights), c_u64, c_i32]),
    "cvy_pack_weights_tiled": (c_i32, [ctypes.POINTER(ModelConfig), ctypes.POINTER(Weights), c_i32]),
    "cvy_engine_create": (c_i32, [ctypes.POINTER(ModelConfig), ctypes.POINTER(EngineConfig), ctypes.POINTER(Weights),
                                  ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(c_vp)]),
    "cvy_engine_destroy": (None, [c_vp]),
    "cvy_register_tool": (c_i32, [c_vp, ctypes.POINTER(ToolDesc), ctypes.POINTER(c_i32)]),
    "cvy_submit_request": (c_i32, [c_vp, ctypes.POINTER(RequestDesc), ctypes.POINTER(c_u64)]),
    "cvy_step": (c_i32, [c_vp, ctypes.POINTER(StepInfo)]),
    "cvy_sync": (c_i32, [c_vp]),
    "cvy_poll_segments": (c_i32, [c_vp, ctypes.POINTER(Segment), c_u32, ctypes.POINTER(c_u32), c_vp, c_sz,
                                  ctypes.POINTER(c_sz)]),
    "cvy_inject_observation": (c_i32, [c_vp, c_u64, ctypes.POINTER(c_i32), c_u32, c_u32, ctypes.POINTER(c_i32),
                                       c_u32]),
    "cvy_cancel_request": (c_i32, [c_vp, c_u64]),
    "cvy_release_request": (c_i32, [c_vp, c_u64]),
    "cvy_round_tokens": (c_i32, [c_vp, c_u64, ctypes.POINTER(c_i32), c_u32, ctypes.POINTER(c_u32)]),
    "cvy_request_state": (c_i32, [c_vp, c_u64]),
    "cvy_debug_logits": (c_i32, [c_vp, c_u64, ctypes.POINTER(c_f32), c_u32]),
    "cvy_perf": (c_i32, [c_vp, ctypes.POINTER(PerfInfo)]),
    "cvy_stream": (c_vp, [c_vp]),
    "cvy_set_kernel_timing": (c_i32, [c_vp, c_i32]),
    "cvy_kernel_times": (c_i32, [c_vp, ctypes.POINTER(KernelTime), c_u32, ctypes.POINTER(c_u32)]),
    "cvy_set_kernel_spans": (c_i32, [c_vp, c_i32]),
    "cvy_kernel_spans": (c_i32, [c_vp, ctypes.POINTER(KernelSpan), c_u32, ctypes.POINTER(c_u32)]),
    "cvy_stats_allgather": (c_i32, [ctypes.POINTER(c_vp), c_i32, ctypes.POINTER(c_u64)]),
    "cvy_debug_buffer": (c_i32, [c_vp, c_i32, c_vp, c_sz, ctypes.POINTER(c_sz)]),
    "cvy_debug_gemm": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_i32, ctypes.POINTER(c_f32)]),
    "cvy_runtime_create": (c_i32, [c_vp, ctypes.POINTER(RuntimeConfig), ctypes.POINTER(c_vp)]),
    "cvy_runtime_run": (c_i32, [c_vp, ctypes.POINTER(RtRequest), c_u32, ctypes.c_double]),
    "cvy_runtime_request_log": (c_i32, [c_vp, c_u32, ctypes.POINTER(RtRequestLog)]),
    "cvy_runtime_round_log": (c_i32, [c_vp, c_u32, c_u32, ctypes.POINTER(RtRoundLog)]),
    "cvy_runtime_piece_log": (c_i32, [c_vp, c_u32, c_u32, c_u32, ctypes.POINTER(RtPieceLog)]),
    "cvy_runtime_stats": (c_i32, [c_vp, ctypes.POINTER(RtStats)]),
    "cvy_runtime_destroy": (None, [c_vp]),
}

_lib = None


class CvyError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libconveyor.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in PROTOTYPES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status: int, allow=()):
    if status != CVY_OK and status not in allow:
        msg = lib().cvy_last_error()
        raise CvyError(status, msg.decode() if msg else "")
    return status
