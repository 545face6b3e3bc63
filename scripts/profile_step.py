"""One decode step at a bench config bracketed by cudaProfilerStart/Stop, for ncu with
--profile-from-start off (launch list of a whole step, or --set full of chosen kernels).

  WORKLOAD=validation|codegen  (default codegen: B=64 C1; validation: B=512, 2K contexts, C4)
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv python scripts/profile_step.py
"""
import os
import sys

R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
import torch  # noqa: E402

import bench  # noqa: E402
from inputs.configs import MISTRAL_7B  # noqa: E402
from paper_2406_00059_b200 import capi  # noqa: E402
from paper_2406_00059_b200.engine import DeviceModel, Engine  # noqa: E402

name = os.environ.get("WORKLOAD", "codegen")
B = int(os.environ.get("B", str(bench.WORKLOADS[name]["batch"])))
WARM = int(os.environ.get("WARM", "6"))
gen = 64
prefix = bench.default_prefix(name, gen)
vocab, reqs = bench.workload_requests(name, range(B), gen, prefix)
pps = (max(r["prefix"] for r in reqs) + gen + 64 + 15) // 16 + 1
dm = DeviceModel(MISTRAL_7B, "bf16", B * pps + 64, seed=1001)
eng = Engine(dm, vocab, max_slots=B, max_pages_per_slot=pps)
if name == "validation":
    tool = eng.register_tool("validator", capi.PARSER_JSON_MEMBER)
else:
    tool = eng.register_tool("interp", capi.PARSER_LITERAL, [b"\n"])
for r in reqs:
    eng.submit_request([1], gen, tool_id=tool, forced=r["forced"], synth_prefix_len=r["prefix"], synth_seed=r["seed"])
for _ in range(WARM):
    eng.step()
    eng.poll_segments()
eng.sync()
torch.cuda.synchronize()
torch.cuda.profiler.start()
eng.step()
eng.sync()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("workload", name, "B", B, "ctx_mean", sum(r["prefix"] for r in reqs) / B + WARM + 1)
eng.poll_segments()
eng.close()
