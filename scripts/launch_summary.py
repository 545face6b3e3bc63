"""Summarise an ncu launch list (gpu__time_duration.sum per launch, one decode step) by kernel:
launches, total us, share of the step.  ncu times are cold-cache and serialised (no PDL
overlap), so the SHARE is what compares with bench.py's in-graph kernel times."""
import csv
import sys

scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg, tot = {}, 0.0
for r in rows[1:]:
    name = r[ik]
    name = name[:name.index("(CUtensorMap")] if "(CUtensorMap" in name else name.split("(")[0]
    v = float(r[iv].replace(",", "")) * scale[r[iu]]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
    tot += v
print(f"{'launches':>8s} {'total_us':>10s} {'avg_us':>8s} {'share':>6s}  kernel")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c:8d} {v:10.1f} {v / c:8.2f} {100 * v / tot:5.1f}%  {k}")
print(f"{len(rows) - 1:8d} {tot:10.1f}           total (one decode step, B=64, 7B bf16)")
