import sys, os
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import numpy as np
import oracle
from gpu_harness import make_engine
from inputs.configs import TINY, slice_of, MISTRAL_7B
from inputs.vocab import byte_level_vocab, synthetic_vocab
from paper_2406_00059_b200 import capi

def per_step(shape, dt, vocab, prompt, steps, prefix=0, sseed=0, nreq=1, label=""):
    dm, eng = make_engine(shape, dt, vocab, nreq, 1000, max_pages_per_slot=16)
    bf = dt == "bf16"
    w = oracle.Weights(shape, 1000, bf16=bf, act_bf16=bf)
    r = oracle.Request(w, prefix + len(prompt) + steps + 2)
    if prefix: r.synth_prefix(prefix, sseed)
    rid = eng.submit_request(prompt, steps, synth_prefix_len=prefix, synth_seed=sseed)
    seq = list(prompt); errs = []
    for t in range(len(prompt) - 1 + steps):
        eng.step(); eng.sync()
        g = eng.debug_logits(rid).astype(np.float64)
        o = oracle.step([r], [seq[t]])[0]
        errs.append(np.abs(g - o).max())
        if t >= len(prompt) - 1:
            seq.append(eng.round_tokens(rid)[-1])
        eng.poll_segments()
    eng.close()
    print(label, " ".join(f"{e:.1e}" for e in errs), flush=True)

V = byte_level_vocab()
per_step(TINY, "bf16", V, list(b"# task\n"), 60, label="tiny bf16 L2:")
per_step(TINY, "fp32", V, list(b"# task\n"), 60, label="tiny fp32 L2:")
s1 = slice_of(TINY, L=1, name="t1")
per_step(s1, "bf16", V, [35], 40, label="tiny bf16 L1 from pos0:")
per_step(s1, "bf16", V, [35], 5, prefix=20, sseed=3, label="tiny bf16 L1 prefix20:")
per_step(s1, "fp32", V, [35], 5, prefix=20, sseed=3, label="tiny fp32 L1 prefix20:")
V32 = synthetic_vocab(32000)
s7 = slice_of(MISTRAL_7B, L=1, name="7b1")
per_step(s7, "bf16", V32, [1, 500], 12, label="7b-L1 bf16 from pos0:")
per_step(s7, "bf16", V32, [1, 500], 2, prefix=20, sseed=3, label="7b-L1 bf16 prefix20:")
