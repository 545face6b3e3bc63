for env in "" "CVY_GEMM_BQ=256" "CVY_GEMM_BQ=256 CVY_GEMM_NSUB=2" "CVY_GEMM_BQ=256 CVY_GEMM_NSUB=2 CVY_GEMM_BK=32"; do
  for shp in "6144 4096" "4096 4096" "28672 4096" "4096 14336"; do
    echo "== $env $shp"; env $env CVY_GEMM_TRACE=1 python scripts/gemm_b512.py child $shp 512 2>&1 | tail -7
  done
done
