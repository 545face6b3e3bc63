#!/bin/bash
# One gpurun call: bench (ours + reference), the ncu launch list of one decode step, and
# ncu --set full of layer 0's 4 projection GEMMs + its attention kernel.  Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
nproc > gpurun_out/host_cores.txt; lscpu | grep "Model name" >> gpurun_out/host_cores.txt
if [ "${BENCH:-1}" = "1" ]; then
python bench.py --steps ${STEPS:-50} --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
tail -c 3000 gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps ${REF_STEPS:-3} --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
tail -c 600 gpurun_out/bench_ref.json
fi
if [ "${NCU:-1}" = "1" ]; then
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python scripts/profile_step.py > gpurun_out/ncu_list.log 2>&1; echo ncu_list_rc=$?
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -c 4 \
    -o gpurun_out/prof_gemm -f python scripts/profile_step.py > gpurun_out/ncu_full.log 2>&1; echo ncu_full_rc=$?
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attention -c 1 \
    -o gpurun_out/prof_attn -f python scripts/profile_step.py > gpurun_out/ncu_attn.log 2>&1; echo ncu_attn_rc=$?
fi
