"""Key metrics of every kernel in an ncu --page raw --csv export (run here, no GPU):
grid, block, registers, duration, DRAM bytes and throughput, L2 throughput, tensor-pipe activity,
issue activity, SM clock.   python scripts/ncu_keys.py gpurun_out/validation_gemm_raw.csv"""
import csv
import sys

KEYS = ["launch__grid_size", "launch__block_size", "launch__cluster_dim_x", "launch__registers_per_thread",
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second"]
rows = list(csv.reader(open(sys.argv[1])))
h, units = rows[0], rows[1]
for r in rows[2:]:
    d = dict(zip(h, r))
    print(d.get("Kernel Name", "")[:90])
    for k in KEYS:
        if k in d and d[k] != "":
            print(f"   {k:<72} {d[k]} {units[h.index(k)]}")
