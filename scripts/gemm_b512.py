"""B=512 projection GEMM variants through cvy_debug_gemm (timing only).
python scripts/gemm_b512.py  -> one JSON line per (config, shape): us, TF/s (hi/lo pair counted)."""
import json, os, subprocess, sys
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    from paper_2406_00059_b200.engine import debug_gemm
    N, K, B = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    W = torch.randn((N, K), device="cuda").to(torch.bfloat16)
    X = torch.randn((B, K), device="cuda").to(torch.bfloat16)
    _, ms = debug_gemm(W, X, N, K, B, iters=30)
    print(json.dumps({"N": N, "K": K, "B": B, "us": round(ms * 1e3, 2), "TFs": round(4.0 * N * K * B / ms / 1e9, 1)}))
    sys.exit(0)
shapes = [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)]
B = int(os.environ.get("B", "512"))
envs = json.loads(os.environ.get("ENVS", "null")) or [
    {}, {"CVY_GEMM_NSUB": "2"}, {"CVY_GEMM_BQ": "256"}, {"CVY_GEMM_BQ": "256", "CVY_GEMM_BK": "32"},
    {"CVY_GEMM_BQ": "256", "CVY_GEMM_NSUB": "2"}, {"CVY_GEMM_BQ": "256", "CVY_GEMM_NSUB": "2", "CVY_GEMM_BK": "32"}]
for env in envs:
    tot = 0.0
    for (N, K) in shapes:
        e = dict(os.environ); e.update(env)
        out = subprocess.run([sys.executable, __file__, "child", str(N), str(K), str(B)], env=e, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
        print(json.dumps(env), line, flush=True)
        try:
            tot += json.loads(line)["us"]
        except Exception:
            pass
    print(json.dumps(env), "layer_sum_us", round(tot, 1), flush=True)
