"""Diagnostic: GPU vs oracle logit error statistics on 7B-width slices (prints, no asserts)."""
import sys, os, random
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle
from gpu_harness import make_engine
from inputs.configs import MISTRAL_7B, TINY, slice_of
from inputs.vocab import synthetic_vocab

def run(L, B, sample, prefix_base=20):
    shape = slice_of(MISTRAL_7B, L=L, name=f"7b-L{L}")
    vocab = synthetic_vocab(32000)
    seed = 1005
    dm, eng = make_engine(shape, "bf16", vocab, B, seed, max_pages_per_slot=8)
    rng = random.Random(3)
    prompts = [[1, rng.randrange(3, 32000)] for _ in range(B)]
    rids = [eng.submit_request(p, 2, synth_prefix_len=prefix_base + (i % 50), synth_seed=i) for i, p in enumerate(prompts)]
    wb = oracle.Weights(shape, seed, bf16=True, act_bf16=False)
    wx = oracle.Weights(shape, seed, bf16=False, act_bf16=False)
    we = oracle.Weights(shape, seed, bf16=True, act_bf16=False)
    ob, oe = [], []
    for i in sample:
        for w, lst in ((wb, ob), (we, oe)):
            r = oracle.Request(w, 100); r.synth_prefix(prefix_base + (i % 50), i); lst.append(r)
    eng.step(); eng.sync()
    lb = oracle.step(ob, [prompts[i][0] for i in sample])
    le = oracle.step(oe, [prompts[i][0] for i in sample])
    for j, i in enumerate(sample):
        g = eng.debug_logits(rids[i]).astype(np.float64)
        d = np.abs(g - lb[j]); de = np.abs(lb[j] - le[j]); dge = np.abs(g - le[j])
        print(f"L={L} B={B} req {i}: |gpu-orc_bf16| max {d.max():.4f} p99.9 {np.quantile(d,0.999):.4f} mean {d.mean():.5f}"
              f" | |orc_bf16-orc_exact| max {de.max():.4f} | |gpu-exact| max {dge.max():.4f} | logit std {lb[j].std():.3f}"
              f" argmax gpu {int(np.argmax(g))} orc {int(np.argmax(lb[j]))}", flush=True)
    eng.close()

run(1, 32, [0, 1, 5, 17, 31])
run(1, 512, [0, 255, 256, 300, 511])
