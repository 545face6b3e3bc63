for p in "" "--prefix 328" "--prefix 528" "--prefix 128"; do
timeout 300 python bench.py --workload codegen --steps 30 --warmup 5 --no-cpu-baseline --no-latency $p 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$p', round(d['ms_per_step'],3), d['config']['ctx_mean'], round(d['step_roofline']['frac'],3), {k: v['ms_per_step'] for k, v in d['kernels'].items() if k=='attention'}, round(d['kernels']['attention']['hbm_frac'],3))"
done
