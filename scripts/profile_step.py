"""One decode step at the bench config bracketed by cudaProfilerStart/Stop, for ncu with
--profile-from-start off (launch list of a whole step, or --set full of chosen kernels).

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

B = int(os.environ.get("B", "64"))
WARM = int(os.environ.get("WARM", "6"))
vocab, reqs = bench.codegen_workload(B, 64)
dm = DeviceModel(MISTRAL_7B, "bf16", B * 40 + 64, seed=1001)
eng = Engine(dm, vocab, max_slots=B, max_pages_per_slot=40)
tool = eng.register_tool("interp", capi.PARSER_LITERAL, [b"\n"])
for r in reqs:
    eng.submit_request([1], 64, tool_id=tool, forced=r["forced"], synth_prefix_len=r["prefix"], synth_seed=r["seed"])
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
print("ctx_mean", sum(r["prefix"] for r in reqs) / B + WARM + 1)
eng.poll_segments()
eng.close()
