# Round-2 profiles of the final code: per workload (C4 validation, C1 codegen) the ncu launch list
# of one decode step (DRAM bytes, L2 bytes) and ncu --set full of layer 0's four projection GEMMs
# and one attention launch.  Outputs in gpurun_out/.
for wl in validation codegen; do
  export WORKLOAD=$wl
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv --log-file gpurun_out/${wl}_launches.csv python scripts/profile_step.py > gpurun_out/${wl}_list.log 2>&1; echo ${wl} list_rc=$?
  timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -c 4 -o gpurun_out/${wl}_gemm -f python scripts/profile_step.py > gpurun_out/${wl}_full.log 2>&1; echo ${wl} full_rc=$?
  timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attention -c 1 -o gpurun_out/${wl}_attn -f python scripts/profile_step.py > gpurun_out/${wl}_attn.log 2>&1; echo ${wl} attn_rc=$?
done
# summarise on the box (reports with source exceed gpurun's copy-back limit)
for f in gpurun_out/*_gemm.ncu-rep gpurun_out/*_attn.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > ${b}_raw.csv 2>/dev/null
  python scripts/ncu_summary.py $f 25 > ${b}_summary.txt 2>&1
done
python scripts/ncu_traffic_attn.py gpurun_out/validation_attn.ncu-rep 512 1799 > gpurun_out/attn_traffic.log 2>&1
python scripts/ncu_traffic.py gpurun_out/codegen_gemm.ncu-rep 64 > gpurun_out/gemm_traffic.log 2>&1
cp profiles/attention_traffic.json profiles/gemm_traffic.json gpurun_out/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
