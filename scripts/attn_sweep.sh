#!/bin/bash
# attention pipeline depth x split count sweep at the bench config (kernel ms per step)
for st in 2 3 4; do for sp in 1 2 3; do
  r=$(CVY_ATTN_STAGES=$st CVY_ATTN_SPLITS=$sp python bench.py --steps 30 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernels_ms_per_step']; print(round(d['ms_per_step'],3), k.get('attention'), k.get('attention_merge'))")
  echo "stages=$st splits=$sp: step_ms attn_ms merge_ms = $r"
done; done
