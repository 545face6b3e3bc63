# Round-2 end evidence: the default bench line (C4, 200 steps, latency A/B, cpu_baseline), the C1
# line, then the ncu launch lists and --set full summaries of both (scripts/prof_r02.sh).
timeout 1500 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench_c4 rc $?
timeout 900 python bench.py --workload codegen --no-cpu-baseline --no-latency > gpurun_out/bench_c1_final.json 2> gpurun_out/bench_c1_final.err; echo bench_c1 rc $?
bash scripts/prof_r02.sh
