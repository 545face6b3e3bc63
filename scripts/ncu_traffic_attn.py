"""From an `ncu --set full` report of one attention launch at C4 (scripts/prof_c4.sh:
WORKLOAD=validation, B = 512, synthetic prefix 1792, profiled after 6 warm-up steps, so every slot
attends over 1799 keys), write profiles/attention_traffic.json: measured DRAM bytes per launch
next to the algorithmic bytes bench.py's roofline uses (runs here, no GPU).

  python scripts/ncu_traffic_attn.py gpurun_out/c4_attn.ncu-rep [B] [nkeys]
"""
import csv
import io
import json
import os
import subprocess
import sys

R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
import bench  # noqa: E402
from inputs.configs import MISTRAL_7B  # noqa: E402

rep = sys.argv[1]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 512
nkeys = int(sys.argv[3]) if len(sys.argv) > 3 else 1799
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def val(d, k):
    return float(d[k].replace(",", "")) * scale.get(units[hdr.index(k)], 1.0)


d = [dict(zip(hdr, r)) for r in rows[2:] if "attention" in dict(zip(hdr, r)).get("Kernel Name", "")][0]
dram = val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum")
alg = bench.attention_launch_bytes(MISTRAL_7B, [nkeys - 1] * B)
t = val(d, "gpu__time_duration.sum")
res = {"per_launch_bytes": dram, "alg_per_launch_bytes": alg, "ratio": dram / alg, "ncu_us": t * 1e6,
       "ncu_GBps_dram": dram / t / 1e9, "batch": B, "nkeys": nkeys,
       "source": f"ncu --set full --clock-control none, one attention launch at C4 ({os.path.basename(rep)})"}
with open(os.path.join(R, "profiles", "attention_traffic.json"), "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res, indent=1))
