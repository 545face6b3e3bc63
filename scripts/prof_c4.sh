export WORKLOAD=validation
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python scripts/profile_step.py > gpurun_out/c4_list.log 2>&1; echo list_rc=$?
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -c 4 -o gpurun_out/c4_gemm -f python scripts/profile_step.py > gpurun_out/c4_full.log 2>&1; echo full_rc=$?
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attention -c 1 -o gpurun_out/c4_attn -f python scripts/profile_step.py > gpurun_out/c4_attn.log 2>&1; echo attn_rc=$?
