"""GEMM microbenchmark through the cvy_debug_gemm hook (timing only)."""
import os, sys, subprocess, json
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    from paper_2406_00059_b200.engine import debug_gemm
    N, K, B = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    W = torch.randn((N, K), device="cuda").to(torch.bfloat16)
    X = torch.randn((B, K), device="cuda").to(torch.bfloat16)
    _, ms = debug_gemm(W, X, N, K, B, iters=50)
    print(json.dumps({"N": N, "K": K, "B": B, "us": ms * 1e3, "GBps": N * K * 2 / ms / 1e6}))
    sys.exit(0)
cases = [(4096, 4096, 64), (6144, 4096, 64), (28672, 4096, 64), (4096, 14336, 64), (32000, 4096, 64)]
envs = [{}, {"CVY_GEMM_DEBUG": "1"}]
for env in envs:
    for (N, K, B) in cases:
        e = dict(os.environ); e.update(env)
        out = subprocess.run([sys.executable, __file__, "child", str(N), str(K), str(B)], env=e, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
        print(env, line, flush=True)
