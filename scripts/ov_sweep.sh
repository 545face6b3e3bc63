# batch-split overlap sweep at C4 (B=512, 2K contexts): step time per knob setting
run() { env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-latency 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$*', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], {k: v['ms_per_step'] for k, v in d['kernels'].items()}, flush=True)"; }
for cfg in "$@"; do run $cfg; done
