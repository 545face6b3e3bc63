"""Phase timeline of one layer inside the persistent all-layers kernel (CVY_GEMM_TRACE_LAYER)
at the bench config: per phase, when the data producers passed the dependency (start) and
when each CTA signalled the phase done (end), min/avg/max over the 148 CTAs, in us from the
earliest start stamp of the traced layer."""
import os, sys
os.environ.setdefault("CVY_GEMM_TRACE_LAYER", "5")
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
os.environ.setdefault("CVY_PERSISTENT", "1")
import numpy as np
import bench
from inputs.configs import MISTRAL_7B
from paper_2406_00059_b200 import capi
from paper_2406_00059_b200.engine import DeviceModel, Engine
B = int(os.environ.get("B", "64"))
vocab, reqs = bench.codegen_workload(B, 40)
dm = DeviceModel(MISTRAL_7B, "bf16", B * 40 + 64, seed=1001)
eng = Engine(dm, vocab, max_slots=B, max_pages_per_slot=40)
tool = eng.register_tool("interp", capi.PARSER_LITERAL, [b"\n"])
for r in reqs:
    eng.submit_request([1], 40, tool_id=tool, forced=r["forced"], synth_prefix_len=r["prefix"], synth_seed=r["seed"])
for _ in range(8):
    eng.step()
eng.sync()
raw = np.concatenate([np.frombuffer(eng.debug_buffer(10 + k), dtype=np.uint64) for k in range(2)])
t = raw.reshape(-1, 32).astype(np.float64)
t0 = t[:, 0][t[:, 0] > 0].min()
names = ["QKV", "attn", "O", "GU", "down"]
def col(i):
    v = (t[:, i] - t0) / 1e3
    return f"{v.min():7.2f} {v.mean():7.2f} {v.max():7.2f}"
print("phase  start(min avg max)        last-acc/attn-end          last-MMA                  done")
for p in range(5):
    print(f"{names[p]:5s} {col(p)} | {col(16 + p)} | {col(24 + p) if p != 1 else ' ' * 23} | {col(8 + p)}")
tp = int(os.environ.get("CVY_PK_TRACE_PHASE", "1"))
print(f"epilogue detail of GEMM {tp}: ")
def colz(i):
    v = t[:, i]
    v = v[v > 0]
    v = (v - t0) / 1e3
    return f"n={len(v)} {v.min():7.2f} {v.mean():7.2f} {v.max():7.2f}" if len(v) else "none"
red = t[:, 5] > 0
print("  reducers n=%d: acc received -> tags ok %.2f | chunk0 copies %.2f | chunk0 epi %.2f | chunk1 copies %.2f | chunk1 epi %.2f us (avg deltas)" % (
    red.sum(), *(np.mean((t[red, b_] - t[red, a_]) / 1e3) for a_, b_ in ((15, 5), (5, 6), (6, 7), (7, 13), (13, 14)))))
print("  reducers: acc received at %.2f avg, done at %.2f avg / %.2f max" % (((t[red, 15] - t0) / 1e3).mean(), ((t[red, 14] - t0) / 1e3).mean(), ((t[red, 14] - t0) / 1e3).max()))
print("attention per CTA (us, avg/max): wait xfull %.2f/%.2f  page compute(warp0) %.2f/%.2f  q load %.2f/%.2f  finish %.2f/%.2f  runs %.1f units %.1f" % (
    t[:, 21].mean() / 1e3, t[:, 21].max() / 1e3, t[:, 22].mean() / 1e3, t[:, 22].max() / 1e3, t[:, 23].mean() / 1e3,
    t[:, 23].max() / 1e3, t[:, 29].mean() / 1e3, t[:, 29].max() / 1e3, t[:, 30].mean(), t[:, 31].mean()))
eng.poll_segments()
eng.close()
