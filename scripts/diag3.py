import sys, os
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import numpy as np, torch
import oracle
from gpu_harness import make_engine
from inputs.configs import TINY, slice_of, MISTRAL_7B
from inputs.vocab import synthetic_vocab
from paper_2406_00059_b200 import capi

def bf(a):
    return torch.tensor(a, dtype=torch.float32).to(torch.bfloat16).double().numpy()
V32 = synthetic_vocab(32000)
shape = slice_of(MISTRAL_7B, L=1, name="7b1")
dm, eng = make_engine(shape, "bf16", V32, 1, 1000, flags=capi.ENGINE_DEBUG_LOGITS | capi.ENGINE_NO_GRAPH, max_pages_per_slot=4)
tok = 500
rid = eng.submit_request([tok], 1)
eng.step(); eng.sync()
def get(which, dtype, n):
    raw = eng.debug_buffer(which)
    if dtype == "bf16":
        a = np.frombuffer(raw, dtype=np.uint16).astype(np.uint32) << 16
        return a.view(np.float32).astype(np.float64)[:n]
    return np.frombuffer(raw, dtype=np.float32).astype(np.float64)[:n]
d, H, Hkv, hd, dff = shape.d, shape.H, shape.Hkv, shape.hd, shape.dff
x_g = get(0, "f32", d); q_g = get(2, "f32", H * hd); o_g = get(3, "bf16", H * hd); h_g = get(4, "bf16", dff); act_g = get(1, "bf16", d)
lg_g = eng.debug_logits(rid)
# GPU weights back from the device for a direct comparison
wq_gpu = dm.tensors["wqkv"].view(torch.bfloat16)[: (H+2*Hkv)*hd*d].view((H+2*Hkv)*hd, d).double().cpu().numpy()
wgu_gpu = dm.tensors["wgu"].view(torch.bfloat16)[: 2*dff*d].view(2*dff, d).double().cpu().numpy()
w = oracle.Weights(shape, 1000, bf16=True, act_bf16=True, cache=False)
T = lambda tid, r, c: w.tensor(tid, r, c)
Wq = T(1, H*hd, d); Wk = T(2, Hkv*hd, d); Wv = T(3, Hkv*hd, d)
print("wq gpu vs oracle", np.abs(wq_gpu[:H*hd] - Wq).max(), np.abs(wq_gpu[H*hd:(H+Hkv)*hd] - Wk).max(), np.abs(wq_gpu[(H+Hkv)*hd:] - Wv).max(), flush=True)
Wg = T(5, dff, d); Wu = T(6, dff, d)
gi = np.concatenate([np.arange(128*j, 128*j+64) for j in range(dff//64)]); ui = gi + 64
print("wg gpu vs oracle", np.abs(wgu_gpu[gi] - Wg).max(), "wu", np.abs(wgu_gpu[ui] - Wu).max(), flush=True)
del wq_gpu, wgu_gpu
E = T(0, shape.V, d); Wo = T(4, d, H*hd); Wd = T(7, d, dff); Wl = T(9, shape.V, d)
x = E[tok].copy()
s = 1/np.sqrt(np.mean(x*x) + shape.eps); u = bf(x)
q = s * (Wq @ u); k = s * (Wk @ u); v = s * (Wv @ u)
G = H // Hkv
o = bf(np.concatenate([bf(v)[(j//G)*hd:(j//G+1)*hd] for j in range(H)]))
print("q max diff", np.abs(q - q_g).max(), "q max", np.abs(q).max())
print("o max diff", np.abs(o - o_g).max(), "o max", np.abs(o).max(), "n diff", int((o != o_g).sum()))
x = x + Wo @ o
s2 = 1/np.sqrt(np.mean(x*x) + shape.eps); u2 = bf(x)
g = s2 * (Wg @ u2); up = s2 * (Wu @ u2); hh = bf(g/(1+np.exp(-g)) * up)
print("h max diff", np.abs(hh - h_g).max(), "h max", np.abs(hh).max(), "n diff", int((hh != h_g).sum()))
x = x + Wd @ hh
print("x max diff", np.abs(x - x_g).max(), "x max", np.abs(x).max())
sf = 1/np.sqrt(np.mean(x*x) + shape.eps); uf = bf(x)
print("act max diff", np.abs(uf - act_g).max(), "n diff", int((uf != act_g).sum()))
lg = sf * (Wl @ uf)
print("logits max diff", np.abs(lg - lg_g).max(), "logit max", np.abs(lg).max())
r = oracle.Request(w, 8); ol = oracle.step([r], [tok])[0]
print("oracle vs numpy mirror", np.abs(ol - lg).max())
