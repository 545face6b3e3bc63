"""A/B of the GEMM batch-tile width (CVY_GEMM_BQ) through cvy_debug_gemm (timing only)."""
import os, sys, subprocess
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
cases = [(28672, 4096, 128), (4096, 14336, 128), (6144, 4096, 128), (4096, 4096, 128), (28672, 4096, 64), (6144, 4096, 64)]
for bq in ("128", "64", "32"):
    for (N, K, B) in cases:
        e = dict(os.environ)
        e["CVY_GEMM_BQ"] = bq
        out = subprocess.run([sys.executable, R + "/scripts/gemm_micro.py", "child", str(N), str(K), str(B)], env=e,
                             capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-200:]
        print("BQ", bq, line, flush=True)
