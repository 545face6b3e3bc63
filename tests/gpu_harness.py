"""Shared helpers for the -m gpu parity tests: drive libconveyor through its C ABI and the
oracle side by side on the same seeded inputs (inputs/)."""
from __future__ import annotations

import json
import os

import numpy as np

import oracle
from oracle.scan import round_records
from paper_2406_00059_b200 import build, capi
from paper_2406_00059_b200.engine import DeviceModel, Engine

_built = False


def ensure_built():
    global _built
    if not _built:
        build.build()
        _built = True


def make_engine(shape, dtype, vocab, max_slots, seed, n_pages=None, flags=capi.ENGINE_DEBUG_LOGITS,
                max_pages_per_slot=64, **kw):
    ensure_built()
    if n_pages is None:
        n_pages = max_slots * max_pages_per_slot
    dm = DeviceModel(shape, dtype, n_pages, seed)
    eng = Engine(dm, vocab, max_slots=max_slots, max_pages_per_slot=max_pages_per_slot, flags=flags, **kw)
    return dm, eng


def free_running_parity(shape, dtype, vocab, prompts, max_new, seed, tol, prefix=0, synth_seeds=None,
                        max_pages_per_slot=64, graph=True, extra_flags=0):
    """Submit every prompt, step until all rounds end, and compare every step's GPU logits
    (cvy_debug_logits) with the oracle fed the same input tokens.  Returns (max_abs_diff,
    generated token lists)."""
    flags = capi.ENGINE_DEBUG_LOGITS | (0 if graph else capi.ENGINE_NO_GRAPH) | extra_flags
    dm, eng = make_engine(shape, dtype, vocab, len(prompts), seed, flags=flags,
                          max_pages_per_slot=max_pages_per_slot)
    bf16 = dtype == "bf16"
    w = oracle.Weights(shape, seed, bf16=bf16)
    max_ctx = prefix + max(len(p) for p in prompts) + max_new + 2
    oreqs = []
    rids = []
    for i, p in enumerate(prompts):
        r = oracle.Request(w, max_ctx)
        ss = synth_seeds[i] if synth_seeds else 0
        if prefix:
            r.synth_prefix(prefix, ss)
        oreqs.append(r)
        rids.append(eng.submit_request(p, max_new, synth_prefix_len=prefix, synth_seed=ss))
    seqs = [list(p) for p in prompts]
    gens = [[] for _ in prompts]
    done = [False] * len(prompts)
    maxdiff = 0.0
    t = 0
    while not all(done):
        eng.step()
        eng.sync()
        live = [i for i in range(len(prompts)) if not done[i]]
        gpu = {i: eng.debug_logits(rids[i]) for i in live}
        ora = oracle.step([oreqs[i] for i in live], [seqs[i][t] for i in live])
        for j, i in enumerate(live):
            d = float(np.max(np.abs(gpu[i].astype(np.float64) - ora[j])))
            maxdiff = max(maxdiff, d)
            assert d < tol, f"request {i} step {t}: max |gpu - oracle| = {d}"
            if t >= len(prompts[i]) - 1:
                toks = eng.round_tokens(rids[i])
                assert len(toks) == len(gens[i]) + 1
                g = toks[-1]
                # the GPU's greedy choice is a valid argmax of the oracle's logits
                assert ora[j][g] >= ora[j].max() - 2 * tol, (i, t, g, int(np.argmax(ora[j])))
                gens[i].append(g)
                seqs[i].append(g)
                if len(gens[i]) >= max_new or (shape.eos >= 0 and g == shape.eos):
                    done[i] = True
        eng.poll_segments()
        t += 1
    eng.close()
    log = os.environ.get("CVY_PARITY_LOG")
    if log:  # measured margins (e.g. gpurun_out/parity.jsonl), for DESIGN.md §4
        with open(log, "a") as f:
            f.write(json.dumps({"test": os.environ.get("PYTEST_CURRENT_TEST", ""), "shape": shape.name,
                                "dtype": dtype, "B": len(prompts), "max_abs_diff": maxdiff, "tol": tol}) + "\n")
    return maxdiff, gens


def group_records(recs):
    out = {}
    for r in recs:
        out.setdefault(r.req_id, []).append(r)
    return out


def expected_records(tokens, vocab, kind, delims, max_seg=4096, round_idx=0, seq_start=0, cancelled=False):
    recs, _ = round_records(tokens, vocab, kind, delims, max_seg, round_idx, seq_start, cancelled)
    return [(r.round, r.seq, r.token_index, r.byte_offset, r.byte_len, r.delim_id, r.flags, r.data) for r in recs]


def as_tuples(recs):
    return [(r.round, r.seq, r.token_index, r.byte_offset, r.byte_len, r.delim_id, r.flags, r.data) for r in recs]
