"""Run one debug GEMM (for ncu captures): python scripts/one_gemm.py N K B"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_00059_b200.engine import debug_gemm
N, K, B = map(int, sys.argv[1:4])
W = torch.randn((N, K), device="cuda").to(torch.bfloat16)
X = torch.randn((B, K), device="cuda").to(torch.bfloat16)
_, ms = debug_gemm(W, X, N, K, B, iters=2)
print(N, K, B, ms * 1e3, "us")
