for shp in "6144 4096" "4096 4096" "28672 4096" "4096 14336"; do
  echo "== $shp"; CVY_GEMM_TRACE=1 python scripts/gemm_b512.py child $shp 512 2>&1 | tail -7
done
CVY_PARITY_LOG=gpurun_out/parity.jsonl timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "full_32 or two_layer_slice_bf16 or large_batch or slice_b40 or tiny_bf16" 2>&1 | tail -3
cat gpurun_out/parity.jsonl
