"""Run-to-run determinism of the first decode step after a chunked-prefill pass (the shape of
tests/test_gpu_parity.py::test_chunked_prefill...[7b-L2]); prints the max |logit diff| of each
repetition against the first, per engine-flag variant.  GPU only (diagnostic)."""
import random, sys, os
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R)
sys.path.insert(0, os.path.join(R, 'tests'))
import numpy as np
from paper_2406_00059_b200 import capi
from inputs.configs import MISTRAL_7B, slice_of
from inputs.vocab import synthetic_vocab
from gpu_harness import make_engine

shape, vocab = slice_of(MISTRAL_7B, L=2, name="7b-L2"), synthetic_vocab(32000)
V = shape.V
variants = {os.environ.get("TAG", "default"): int(os.environ.get("XFLAGS", "0"))}
reps = int(os.environ.get("REPS", "6"))
for name, extra in variants.items():
    ref = None
    diffs = []
    hashes = []
    for rep in range(reps):
        rng = random.Random(31)
        flags = capi.ENGINE_DEBUG_LOGITS | capi.ENGINE_CHUNKED_PREFILL | extra
        dm, eng = make_engine(shape, "bf16", vocab, 5, 1010, flags=flags, max_pages_per_slot=16)
        prompts = [[rng.randrange(3, V) for _ in range(n)] for n in (1, 2, 17, 40, 65)]
        prefix = [0, 9, 0, 21, 3]
        rids = [eng.submit_request(p, 3, synth_prefix_len=prefix[i], synth_seed=40 + i) for i, p in enumerate(prompts)]
        if rep == 0 and name == "default":
            pt = eng.debug_page_table(rids[4]) if hasattr(eng, "debug_page_table") else None
            print("slot 4 pages", pt, flush=True)
        eng.step()
        eng.sync()
        if rep == 0:
            import ctypes
            for which in (6, 7):
                nb = ctypes.c_size_t()
                capi.lib().cvy_debug_buffer(eng.h, which, None, 0, ctypes.byref(nb))
                buf = np.zeros(nb.value // 4, dtype=np.int32)
                capi.lib().cvy_debug_buffer(eng.h, which, buf.ctypes.data_as(ctypes.c_void_p), nb.value, ctypes.byref(nb))
                if which == 6:
                    ptab = buf.reshape(-1, 16)[:5]
                    print("page table", ptab.tolist(), flush=True)
                else:
                    t = buf.reshape(3, -1)
                    rows = [(int(t[0, i]), int(t[1, i])) for i in range(t.shape[1]) if t[1, i] >= 0]
                    dup = len(rows) - len(set(rows))
                    print("prefill rows", len(rows), "duplicates", dup, "per slot", {s_: [p_ for s2, p_ in rows if s2 == s_][:3] + ['..'] for s_ in set(r[0] for r in rows)}, flush=True)
        import torch
        kvraw = dm.tensors["kv_pool"].view(torch.bfloat16)
        kv = kvraw.float().cpu().numpy()
        if rep == 0:
            print("kv_pool elements", kv.size, "=", kv.size / (2 * 2 * 8 * 16 * 128), "pages x layers", flush=True)
        kv = kv.reshape(2, -1, 8, 2, 16, 128)  # [L][pages][Hkv][K/V][16][hd]
        if rep == 0:
            nz = sorted(set((int(a), int(b)) for a, b in np.argwhere(np.abs(kv).sum(axis=(2, 3, 4, 5)) > 0)))
            print("nonzero (layer, page):", nz, flush=True)
        lg = np.stack([eng.debug_logits(r).astype(np.float64) for r in rids])
        eng.close()
        import hashlib
        hashes.append(hashlib.md5(kv.tobytes()).hexdigest()[:8])
        if ref is None:
            ref, kref = lg, kv
        else:
            diffs.append([float(np.max(np.abs(lg[i] - ref[i]))) for i in range(5)])
            bad = np.argwhere(np.abs(kv - kref) > 0)
            if len(bad):
                pages = sorted(set(int(b[1]) for b in bad))
                owner = {}
                for sl in range(5):
                    for j, pg in enumerate(ptab[sl]):
                        if pg or (sl == 0 and j == 0):
                            owner.setdefault(int(pg), (sl, j))
                agg = {}
                for b in bad:
                    l, pg, g, c, tk = (int(x) for x in b[:5])
                    sl, j = owner.get(pg, (-1, -1))
                    key = (l, sl, j * 16 + tk if sl >= 0 else (pg, tk), "KV"[c])
                    agg.setdefault(key, set()).add(g)
                vals = [(float(kv[tuple(b)]), float(kref[tuple(b)])) for b in bad[:4]]
                print(name, rep, "KV differs:", len(bad), "elements; (layer, slot, pos, K/V): heads",
                      {k: sorted(v) for k, v in sorted(agg.items(), key=str)}, "values", vals, flush=True)
    print(name, "KV hashes", hashes, flush=True)
