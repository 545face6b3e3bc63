"""Map ncu per-instruction stall samples to CUDA source lines via nvdisasm -g line info.
usage: ncu_lines.py report.ncu-rep cubin mangled_function_name [topN]"""
import csv, io, re, subprocess, sys, collections
rep, cubin, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
i_s = h.index("Warp Stall Sampling (All Samples)")
samples = {}
for r in rows[2:]:
    if len(r) > i_s and r[i_s].isdigit():
        samples[int(r[0], 16)] = samples.get(int(r[0], 16), 0) + int(r[i_s])
base = min(samples)
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
sec = dis.split(".text." + fn + ":")[1].split("//--------------------- .text.")[0]
line_of = {}
cur = "?"
for ln in sec.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m:
        line_of[int(m.group(1), 16)] = cur
agg = collections.Counter()
for a, s in samples.items():
    agg[line_of.get(a - base, "?")] += s
tot = sum(agg.values())
for k, v in agg.most_common(top):
    print(f"{v:6d} {100 * v / tot:5.1f}%  {k}")
