"""Diagnostic: tiny-width model, one request, one step: GPU intermediates vs a numpy mirror of the
oracle's bf16 storage points (prints only)."""
import sys, os
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import numpy as np, torch
import oracle
from gpu_harness import make_engine, free_running_parity
from inputs.configs import TINY, slice_of, MISTRAL_7B
from inputs.vocab import byte_level_vocab
from paper_2406_00059_b200 import capi

V = byte_level_vocab()
for L in (0, 1, 2):
    shape = slice_of(TINY, L=L, name=f"tiny-L{L}")
    for dt, tol in (("fp32", 1), ("bf16", 1)):
        try:
            d, _ = free_running_parity(shape, dt, V, [list(b"# task 0\n"), list(b"hi\n")], 6, seed=1000, tol=tol)
            print(f"tiny L={L} {dt}: max |gpu-oracle| = {d:.3e}", flush=True)
        except Exception as ex:
            print(f"tiny L={L} {dt}: EXC {ex}", flush=True)

def bf(a):
    return torch.tensor(a, dtype=torch.float32).to(torch.bfloat16).double().numpy()

# one step, L=1, bf16, compare intermediates
shape = slice_of(TINY, L=1, name="tiny-L1")
dm, eng = make_engine(shape, "bf16", V, 1, 1000, flags=capi.ENGINE_DEBUG_LOGITS | capi.ENGINE_NO_GRAPH)
tok = 35
rid = eng.submit_request([tok], 1)
eng.step(); eng.sync()
act_ld = max(shape.d, shape.H * shape.hd, shape.dff)
def get(which, dtype, n):
    raw = eng.debug_buffer(which)
    if dtype == "bf16":
        a = np.frombuffer(raw, dtype=np.uint16).astype(np.uint32) << 16
        return a.view(np.float32).astype(np.float64)[:n]
    return np.frombuffer(raw, dtype=np.float32).astype(np.float64)[:n]
x_g = get(0, "f32", shape.d)
q_g = get(2, "f32", shape.H * shape.hd)
o_g = get(3, "bf16", shape.H * shape.hd)
h_g = get(4, "bf16", shape.dff)
act_g = get(1, "bf16", shape.d)
lg_g = eng.debug_logits(rid)
w = oracle.Weights(shape, 1000, bf16=True, act_bf16=True)
T = lambda tid, r, c: w.tensor(tid, r, c)
d, H, Hkv, hd, dff = shape.d, shape.H, shape.Hkv, shape.hd, shape.dff
E = T(0, shape.V, d); Wq = T(1, H*hd, d); Wk = T(2, Hkv*hd, d); Wv = T(3, Hkv*hd, d); Wo = T(4, d, H*hd)
Wg = T(5, dff, d); Wu = T(6, dff, d); Wd = T(7, d, dff); Wl = T(9, shape.V, d)
x = E[tok].copy()
s = 1/np.sqrt(np.mean(x*x) + shape.eps); u = bf(x)
q = s * (Wq @ u); k = s * (Wk @ u); v = s * (Wv @ u)
# pos 0: rope identity; one key: o = v per group
G = H // Hkv
o = np.concatenate([bf(v)[ (j//G)*hd:(j//G+1)*hd] for j in range(H)]); o = bf(o)
print("q max diff", np.abs(q - q_g).max(), "q max", np.abs(q).max())
print("o max diff", np.abs(o - o_g).max(), "o max", np.abs(o).max())
x = x + Wo @ o
s2 = 1/np.sqrt(np.mean(x*x) + shape.eps); u2 = bf(x)
g = s2 * (Wg @ u2); up = s2 * (Wu @ u2); hh = bf(g/(1+np.exp(-g)) * up)
print("h max diff", np.abs(hh - h_g).max(), "h max", np.abs(hh).max())
x = x + Wd @ hh
print("x max diff", np.abs(x - x_g).max(), "x max", np.abs(x).max())
sf = 1/np.sqrt(np.mean(x*x) + shape.eps); uf = bf(x)
print("act max diff", np.abs(uf - act_g).max())
lg = sf * (Wl @ uf)
print("logits max diff", np.abs(lg - lg_g).max(), "logit max", np.abs(lg).max())
r = oracle.Request(w, 8); ol = oracle.step([r], [tok])[0]
print("oracle vs numpy mirror", np.abs(ol - lg).max())

from paper_2406_00059_b200.engine import debug_gemm
for (N, K, B) in [(256, 128, 4), (4096, 4096, 64), (4096, 4096, 512), (32000, 4096, 32)]:
    g = torch.Generator(device="cuda").manual_seed(1)
    W = (torch.rand((N, K), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    X = (torch.rand((B, K), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    Y, ms = debug_gemm(W, X, N, K, B, iters=20)
    ref = X.double() @ W.double().T
    err = (Y.double() - ref).abs().max().item()
    print(f"gemm N={N} K={K} B={B}: max err {err:.3e}, ref std {ref.std().item():.2f}, {ms*1e3:.1f} us, "
          f"{N*K*2/ms/1e6:.0f} GB/s weights", flush=True)
