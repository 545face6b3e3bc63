"""From an `ncu --set full` report of layer 0's four projection GEMMs (QKV, O, gate/up, down,
in launch order) at the bench config, write profiles/gemm_traffic.json: measured DRAM bytes
per launch next to the algorithmic bytes bench.py's roofline uses (runs here, no GPU).

  python scripts/ncu_traffic.py gpurun_out/prof_gemm.ncu-rep [B]
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
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def val(d, k):
    u = units[hdr.index(k)]
    return float(d[k].replace(",", "")) * scale.get(u, 1.0)


gemms = [dict(zip(hdr, r)) for r in rows[2:] if "gemm_tc_kernel" in dict(zip(hdr, r)).get("Kernel Name", "")]
names, kinds = ["gemm_qkv", "gemm_o", "gemm_gate_up", "gemm_down"], [1, 4, 5, 6]
by = {}
for d, name, kind in zip(gemms, names, kinds):
    dram = val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum")
    alg = bench.gemm_launch_bytes(MISTRAL_7B, kind, B)
    t = val(d, "gpu__time_duration.sum")
    by[name] = {"dram_bytes": dram, "alg_bytes": alg, "ratio": dram / alg, "ncu_us": t * 1e6,
                "ncu_GBps_alg": alg / t / 1e9}
n = len(by)
res = {"per_launch_bytes": sum(v["dram_bytes"] for v in by.values()) / n,
       "alg_per_launch_bytes": sum(v["alg_bytes"] for v in by.values()) / n,
       "by_gemm": by, "batch": B,
       "source": f"ncu --set full --clock-control none of layer 0's projection GEMMs ({os.path.basename(rep)})"}
res["ratio"] = res["per_launch_bytes"] / res["alg_per_launch_bytes"]
with open(os.path.join(R, "profiles", "gemm_traffic.json"), "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps(res, indent=1))
