# GPU parity suite (margins logged) + smoke + a short bench at C4 and C1
rm -f gpurun_out/parity.jsonl
CVY_PARITY_LOG=gpurun_out/parity.jsonl timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest.log
tail -15 gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-latency > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench rc $?
timeout 600 python bench.py --workload codegen --steps 30 --warmup 5 --no-cpu-baseline --no-latency > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench rc $?
for f in gpurun_out/bench_c4.json gpurun_out/bench_c1.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', round(d['value']), round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), d['clocks']['sm_mhz'], {k: v['ms_per_step'] for k, v in d['kernels'].items()})"; done
