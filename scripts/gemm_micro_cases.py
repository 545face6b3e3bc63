import os, sys, subprocess
R = "/root/repo"
cases = [(28672, 4096, 32), (28672, 4096, 64), (28672, 4096, 128), (28672, 4096, 256), (4096, 14336, 64), (4096, 14336, 128), (6144, 4096, 64), (6144, 4096, 128)]
for env in [{}, {"CVY_GEMM_NSUB": "1"}]:
    for (N, K, B) in cases:
        e = dict(os.environ); e.update(env)
        out = subprocess.run([sys.executable, R + "/scripts/gemm_micro.py", "child", str(N), str(K), str(B)], env=e, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-200:]
        print(env, line, flush=True)
