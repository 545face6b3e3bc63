"""Summarise an ncu launch list of one decode step by kernel: launches, total time, share of the
step, DRAM bytes (read + write) and L2 bytes when captured.  ncu times are cold-cache and
serialised (no PDL overlap), so the SHARE is what compares with bench.py's in-graph kernel times.

  python scripts/launch_summary.py gpurun_out/validation_launches.csv"""
import csv
import sys

scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, iid, im, iv, iu = (h.index(k) for k in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
per = {}
for r in rows[1:]:
    name = r[ik]
    name = name[:name.index("(CUtensorMap")] if "(CUtensorMap" in name else name.split("(")[0]
    d = per.setdefault(r[iid], {"name": name})
    d[r[im]] = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
agg, tot = {}, 0.0
for d in per.values():
    a = agg.setdefault(d["name"], [0, 0.0, 0.0, 0.0])
    t = d.get("gpu__time_duration.sum", 0.0)
    a[0] += 1
    a[1] += t
    a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    a[3] += d.get("lts__t_bytes.sum", 0.0)
    tot += t
print(f"{'launches':>8s} {'total_us':>10s} {'share':>6s} {'DRAM_GB':>8s} {'GB/s':>7s} {'L2_GB':>7s}  kernel")
for name, (n, t, dram, l2) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:8d} {t:10.1f} {t / tot:6.3f} {dram / 1e9:8.3f} {dram / (t * 1e-6) / 1e9 if t else 0:7.0f} {l2 / 1e9:7.3f}  {name[:90]}")
print(f"{'':8s} {tot:10.1f}  total (serialised, cold)")
