"""CPU-side checks of the boundary: libconveyor.so builds for sm_100a, loads, exports every
symbol include/conveyor.h declares, and fails loudly (E_CUDA, no CPU fallback) without a GPU."""
import ctypes
import re
import os

import pytest

from conftest import has_gpu
from inputs.configs import MISTRAL_7B, TINY
from paper_2406_00059_b200 import build, capi
from paper_2406_00059_b200.engine import model_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return capi.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "conveyor.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cvy_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported_and_bound(lib):
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
        assert s in capi.PROTOTYPES, s


def test_abi_version(lib):
    assert lib.cvy_abi_version() == 1


def test_weight_sizes_host_only(lib):
    cfg = model_config(MISTRAL_7B, "bf16")
    sz = capi.WeightSizes()
    assert lib.cvy_weight_sizes_for(ctypes.byref(cfg), 1000, ctypes.byref(sz)) == 0
    assert sz.wqkv == 32 * 6144 * 4096 * 2
    assert sz.wgu == 32 * 2 * 14336 * 4096 * 2
    assert sz.kv_pool == 32 * 1000 * 2 * 8 * 16 * 128 * 2
    streamed = sz.wqkv + sz.wo + sz.wgu + sz.wd + sz.lm_head
    assert streamed == 2 * MISTRAL_7B.n_params_streamed  # 14.22 GB of bf16 weights per step


def test_invalid_model_rejected(lib):
    cfg = model_config(TINY, "bf16")
    cfg.head_dim = 48
    sz = capi.WeightSizes()
    assert lib.cvy_weight_sizes_for(ctypes.byref(cfg), 10, ctypes.byref(sz)) == capi.CVY_E_INVAL
    assert b"head_dim" in lib.cvy_last_error()


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_no_gpu_fails_loudly(lib):
    cfg = model_config(TINY, "fp32")
    ecfg = capi.EngineConfig(4, 64, 8, 1024, 4096, 256, 256, 256, 0, 0)
    w = capi.Weights(*([1] * 10))
    h = ctypes.c_void_p()
    tb = bytes(256 * 16)
    ln = bytes([1] * 256)
    st = lib.cvy_engine_create(ctypes.byref(cfg), ctypes.byref(ecfg), ctypes.byref(w), tb, ln, ctypes.byref(h))
    assert st == capi.CVY_E_CUDA and not h.value
    assert lib.cvy_init_synthetic_weights(ctypes.byref(cfg), ctypes.byref(w), 1, 0) == capi.CVY_E_CUDA
    assert lib.cvy_debug_gemm(None, None, None, 128, 64, 4, 1, 0, None) == capi.CVY_E_INVAL


def test_pack_weights_tiled_rejects_before_touching_memory(lib):
    """cvy_pack_weights_tiled validates dtype and shape before any device work (no GPU needed):
    fp32 and projections whose rows are not multiples of 128 are CVY_E_INVAL."""
    from inputs.configs import ModelShape
    w = capi.Weights(*([1] * 10))
    cfg = model_config(TINY, "fp32")
    assert lib.cvy_pack_weights_tiled(ctypes.byref(cfg), ctypes.byref(w), 0) == capi.CVY_E_INVAL
    assert b"bf16" in lib.cvy_last_error()
    odd = ModelShape("odd", L=1, d=128, H=4, Hkv=1, hd=32, dff=384, V=256, eps=1e-5, rope_base=1e4, eos=-1)  # 192 QKV rows
    cfg = model_config(odd, "bf16")
    assert lib.cvy_pack_weights_tiled(ctypes.byref(cfg), ctypes.byref(w), 0) == capi.CVY_E_INVAL
    assert b"% 128" in lib.cvy_last_error()
    assert lib.cvy_pack_weights_tiled(ctypes.byref(cfg), None, 0) == capi.CVY_E_INVAL


def test_null_engine_calls_are_errors(lib):
    assert lib.cvy_step(None, None) == capi.CVY_E_INVAL
    assert lib.cvy_cancel_request(None, 1) == capi.CVY_E_INVAL
    assert lib.cvy_request_state(None, 1) == -1


def test_sass_has_tcgen05_and_tma(lib):
    """The bf16 projection kernel is built from tcgen05.mma + TMA (SASS UTC*MMA / UTMALDG)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "-sass", capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out or "UTCMMA" in out or re.search(r"UTC\w*MMA", out)
    assert "UTMALDG" in out
    assert "LDTM" in out
