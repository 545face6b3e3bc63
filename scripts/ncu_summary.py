"""Summarise an ncu report: key metrics + top stall source lines (run here, no GPU)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr = raw[0]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tc.sum", "sm__inst_executed_pipe_tmem.sum", "launch__registers_per_thread",
        "smsp__cycles_active.avg", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
for row in raw[2:]:
    d = dict(zip(hdr, row))
    print(d.get("Kernel Name", "")[:80])
    for k in keys:
        if k in d:
            print(f"  {k} = {d[k]} {raw[1][hdr.index(k)]}")
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv"))))
h = src[1]
i_src, i_s = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
seen, data = set(), []
for r in src[2:]:
    if len(r) <= i_s or r[0] in seen:
        continue
    seen.add(r[0])
    data.append((int(r[i_s]) if r[i_s].isdigit() else 0, r[0][-5:], r[i_src].strip()[:100]))
tot = sum(d[0] for d in data) or 1
print("top stall sites (of", tot, "samples):")
for s, a, t in sorted(data, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"  {s:6d} {100*s/tot:5.1f}%  {a}  {t}")
