"""B200-native decode hot path under Conveyor (arXiv 2406.00059): continuous-batching
decode with a fused device-side tool-trigger scan, behind the C ABI in include/conveyor.h.

    from paper_2406_00059_b200 import build, engine
    build.build()                 # nvcc -> libconveyor.so (sm_100a)
    m = engine.DeviceModel(shape, "bf16", n_pages, seed)
    e = engine.Engine(m, vocab, max_slots=64, n_pages=n_pages)
"""
from . import capi  # noqa: F401
