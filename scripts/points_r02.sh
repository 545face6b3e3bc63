# round-2 measurement points: trigger-scan overhead at C4 and C1 (3 interleaved pairs each), and
# small-batch decode points (B = 1, 8, 32) to show the tcgen05 GEMM streams weights at HBM speed
run() { wl=$1; shift; timeout 300 python bench.py --workload $wl --steps 30 --warmup 5 --no-cpu-baseline --no-latency "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
k=d['kernels']; g=sum(v['ms_per_step'] for n,v in k.items() if n.startswith('gemm')); gb=sum(v['alg_bytes'] for n,v in k.items() if n.startswith('gemm'))
print(json.dumps({'workload':'$wl','args':'$*','B':d['config']['batch_per_gpu'],'ms':round(d['ms_per_step'],4),'ms_med':round(d['ms_per_step_median'],4),'tok_s':round(d['value']),'step_frac':round(d['step_roofline']['frac'],3),'gemm_ms':round(g,4),'gemm_TBps':round(gb/g/1e9,3),'attn_ms':k['attention']['ms_per_step'],'sm_mhz':d['clocks']['sm_mhz']}), flush=True)"; }
for i in 1 2 3; do run validation; run validation --scan-off; done
for i in 1 2 3; do run codegen; run codegen --scan-off; done
for b in 1 8 32; do run codegen --batch $b; done
