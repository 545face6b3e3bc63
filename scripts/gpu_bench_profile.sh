#!/bin/bash
# One gpurun call: bench (ours + reference), ncu launch list of one step, ncu --set full of
# the first layer's 4 projection GEMMs + the attention kernel.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
nproc > gpurun_out/host_cores.txt; lscpu | grep "Model name" >> gpurun_out/host_cores.txt
python bench.py --steps ${STEPS:-50} --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
tail -c 3000 gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps ${REF_STEPS:-3} --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
tail -c 600 gpurun_out/bench_ref.json
if [ "${NCU:-1}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm_tc|attention|embed" -s 486 -c 170 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo ncu_list_rc=$?
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 387 -c 5 -o gpurun_out/prof_gemm -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu_full_rc=$?
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention_kernel -s 96 -c 2 -o gpurun_out/prof_attn -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_attn.log 2>&1; echo ncu_attn_rc=$?
fi
