"""In-step timeline of the 4 GEMMs of one layer (CVY_GEMM_TRACE_LAYER) at the bench config."""
import os, sys
os.environ.setdefault("CVY_GEMM_TRACE_LAYER", "5")
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
import numpy as np
import bench
from inputs.configs import MISTRAL_7B
from paper_2406_00059_b200 import capi
from paper_2406_00059_b200.engine import DeviceModel, Engine
flags = int(os.environ.get("FLAGS", "0"))
B = int(os.environ.get("B", "64"))
vocab, reqs = bench.workload_requests("codegen", range(B), 40)
dm = DeviceModel(MISTRAL_7B, "bf16", B * 40 + 64, seed=1001)
eng = Engine(dm, vocab, max_slots=B, max_pages_per_slot=40, flags=flags)
tool = eng.register_tool("interp", capi.PARSER_LITERAL, [b"\n"])
for r in reqs:
    eng.submit_request([1], 40, tool_id=tool, forced=r["forced"], synth_prefix_len=r["prefix"], synth_seed=r["seed"])
for _ in range(8):
    eng.step()
eng.sync()
names = ["QKV", "O", "GU", "D"]
tr = [np.frombuffer(eng.debug_buffer(10 + k), dtype=np.uint64).reshape(-1, 16).astype(np.float64) for k in range(4)]
t0 = min(t[:, 0][t[:, 0] > 0].min() for t in tr)
prev_end = None
for k in range(4):
    t = tr[k]
    v = t[:, 0] > 0
    st, pd, lm, ep, ex = [(t[v, i] - t0) / 1e3 for i in (0, 1, 3, 4, 5)]
    print(f"{names[k]:3s} CTAs {v.sum():3d}: start {st.min():8.2f}..{st.max():8.2f}  producer done avg {pd.mean():8.2f}  "
          f"last MMA avg {lm.mean():8.2f} max {lm.max():8.2f}  epi done avg {ep.mean():8.2f} max {ep.max():8.2f}  exit max {ex.max():8.2f} us"
          + (f"  gap from prev exit {st.min() - prev_end:6.2f}" if prev_end is not None else ""))
    if (t[v, 6] > 0).all():
        cs, rd = [(t[v, i] - t0) / 1e3 for i in (6, 7)]
        print(f"      split-K: staged+cluster_sync avg {cs.mean():8.2f} max {cs.max():8.2f}  reduce+epi avg {rd.mean():8.2f} "
              f"max {rd.max():8.2f}  (last MMA -> sync {(cs - lm).mean():5.2f}, reduce+epi {(rd - cs).mean():5.2f}, "
              f"final sync {(ep - rd).mean():5.2f})")
        d0, d1 = [(t[v, i] - t0) / 1e3 for i in (8, 9)]
        print(f"      first unit: dsmem loads {(d0 - cs).mean():5.2f}  epilogue_chunk {(d1 - d0).mean():5.2f}  us")
    prev_end = ex.max()
eng.poll_segments()
eng.close()
