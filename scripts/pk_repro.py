"""Persistent-kernel bring-up: one engine at the bench's batch on an L-layer 7B slice, a few
steps, logits vs the one-kernel-per-op path (CVY_ENGINE_NO_PERSISTENT) of the same weights."""
import os, sys, time
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
os.environ.setdefault("CVY_PERSISTENT", "1")
import numpy as np
import bench
from inputs.configs import MISTRAL_7B, slice_of
from paper_2406_00059_b200 import capi
from paper_2406_00059_b200.engine import DeviceModel, Engine

L = int(os.environ.get("L", "2"))
B = int(os.environ.get("B", "64"))
steps = int(os.environ.get("STEPS", "3"))
shape = slice_of(MISTRAL_7B, L=L, name=f"7b-L{L}") if L < 32 else MISTRAL_7B
vocab, reqs = bench.codegen_workload(B, 40)
dm = DeviceModel(shape, "bf16", B * 40 + 64, seed=1001)
out = {}
for flags in (capi.ENGINE_DEBUG_LOGITS, capi.ENGINE_DEBUG_LOGITS | capi.ENGINE_NO_PERSISTENT):
    eng = Engine(dm, vocab, max_slots=B, max_pages_per_slot=40, flags=flags)
    tool = eng.register_tool("interp", capi.PARSER_LITERAL, [b"\n"])
    rids = [eng.submit_request([1], 40, tool_id=tool, forced=r["forced"], synth_prefix_len=r["prefix"],
                               synth_seed=r["seed"]) for r in reqs]
    logs = []
    for s in range(steps):
        t0 = time.time()
        eng.step()
        eng.sync()
        logs.append(np.stack([eng.debug_logits(r) for r in rids]))
        print(f"flags {flags} step {s} ok {1e3*(time.time()-t0):.1f} ms", flush=True)
    eng.poll_segments()
    eng.close()
    out[flags] = logs
a, b = out[capi.ENGINE_DEBUG_LOGITS], out[capi.ENGINE_DEBUG_LOGITS | capi.ENGINE_NO_PERSISTENT]
for s in range(steps):
    d = np.abs(a[s] - b[s])
    print(f"step {s}: max |persistent - per-op| = {d.max():.3e}  (row of max {np.unravel_index(d.argmax(), d.shape)})")
