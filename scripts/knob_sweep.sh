# step time per knob setting: bash scripts/knob_sweep.sh WORKLOAD "K1=V1 K2=V2" ...
wl=$1; shift
run() { env "$@" timeout 300 python bench.py --workload $wl --steps 30 --warmup 5 --no-cpu-baseline --no-latency 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$wl', '$*', round(d['ms_per_step'],3), round(d['ms_per_step_median'],3), round(d['step_roofline']['frac'],3), d['clocks']['sm_mhz'], {k: v['ms_per_step'] for k, v in d['kernels'].items()}, flush=True)"; }
for cfg in "$@"; do run $cfg; done
