# batch-split overlap sweep at C4 (B=512, 2K contexts): step time per knob setting
set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "large_batch" 2>&1 | tail -3
run() { env "$@" timeout 300 python bench.py --batch 512 --prefix-min 1792 --prefix-spread 0 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$*', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
run CVY_OVERLAP=0
run CVY_OVERLAP=1
run CVY_OV_GEMM_SMS=64
run CVY_OV_GEMM_SMS=96
run CVY_OV_GEMM_SMS=120
run CVY_OV_PRIO=0
run CVY_OV_PRIO=2
run CVY_OV_SERIAL_ATTN=0
