# Same-box A/B of two builds: the working tree (new) against the .oldtree worktree (old),
# interleaved, 30 timed steps each: bash scripts/ab_trees.sh WORKLOAD [rounds]
wl=$1; n=${2:-2}
one() { (cd $1 && timeout 400 python bench.py --workload $wl --steps 30 --warmup 5 --no-cpu-baseline --no-latency 2>/dev/null) | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$wl', '$2', round(d['ms_per_step'],3), round(d['ms_per_step_median'],3), d['clocks']['sm_mhz'], {k: v['ms_per_step'] for k, v in d['kernels'].items()}, flush=True)"; }
for i in $(seq $n); do one . new; one .oldtree old; done
