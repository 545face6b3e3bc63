"""Which kernel of a chunked-prefill pass is nondeterministic: a 1-layer 7B-width model, the
prefill pass of tests/test_gpu_parity.py::test_chunked_prefill...[7b-L2] repeated REPS times;
per buffer of the pass (q, attention output o, SwiGLU h, final residual x, next act) the rows
that differ from the first repetition.  GPU only (diagnostic)."""
import ctypes, os, random, sys
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
sys.path.insert(0, os.path.join(R, "tests"))
import numpy as np
from paper_2406_00059_b200 import capi
from inputs.configs import MISTRAL_7B, slice_of
from inputs.vocab import synthetic_vocab
from gpu_harness import make_engine

L = int(os.environ.get("LAYERS", "1"))
shape, vocab = slice_of(MISTRAL_7B, L=L, name="7b-L"), synthetic_vocab(32000)
V = shape.V
xflags = int(os.environ.get("XFLAGS", "0"))
names = {9: "q", 20: "o", 21: "h", 8: "x", 22: "act"}
ref = None
for rep in range(int(os.environ.get("REPS", "8"))):
    rng = random.Random(31)
    flags = capi.ENGINE_DEBUG_LOGITS | capi.ENGINE_CHUNKED_PREFILL | xflags
    dm, eng = make_engine(shape, "bf16", vocab, 5, 1010, flags=flags, max_pages_per_slot=16)
    prompts = [[rng.randrange(3, V) for _ in range(n)] for n in (1, 2, 17, 40, 65)]
    prefix = [0, 9, 0, 21, 3]
    rids = [eng.submit_request(p, 3, synth_prefix_len=prefix[i], synth_seed=40 + i) for i, p in enumerate(prompts)]
    eng.step()
    eng.sync()
    bufs = {}
    for w in names:
        nb = ctypes.c_size_t()
        capi.lib().cvy_debug_buffer(eng.h, w, None, 0, ctypes.byref(nb))
        b = np.zeros(nb.value, dtype=np.uint8)
        capi.lib().cvy_debug_buffer(eng.h, w, b.ctypes.data_as(ctypes.c_void_p), nb.value, ctypes.byref(nb))
        if w in (8, 9):
            bufs[w] = b.view(np.float32).reshape(512, -1)[:120]
        else:  # [2 planes][512][act_ld] bf16 -> hi plane rows as uint16
            bufs[w] = b.view(np.uint16).reshape(2, 512, -1)[:, :120]
    eng.close()
    if ref is None:
        ref = bufs
        continue
    out = []
    for w, nm in names.items():
        d = bufs[w] != ref[w]
        rows = sorted(set(int(r) for r in np.argwhere(d.reshape(d.shape[0], -1) if w in (8, 9) else d.any(axis=0))[:, 0]))
        if rows:
            out.append(f"{nm}: rows {rows[:12]}")
    print("rep", rep, "; ".join(out) if out else "identical", flush=True)
