#!/bin/bash
# cross-kernel L2 weight prefetch: KB per next-kernel CTA vs step time
for kb in ${PF_LIST:-0 128 256 512}; do
  r=$(CVY_GEMM_PF_KB=$kb python bench.py --steps 50 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), d['roofline']['kernels_ms_per_step'])")
  echo "pf_kb=$kb: tok/s ms/step kernels = $r"
done
