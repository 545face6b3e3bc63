"""GPU parity (B200, via gpurun): libconveyor's CUDA path vs the CPU oracle, through the C ABI.

Tolerances (BASELINE.json north_star): logits max-abs 1e-4 on the fp32 path and 2e-2 on the
bf16 path; trigger positions and segment records bit-exact under teacher forcing.
"""
import json
import random

import numpy as np
import pytest

import oracle
from oracle.scan import round_records
from gpu_harness import (as_tuples, ensure_built, expected_records, free_running_parity, group_records,
                         make_engine)
from inputs.configs import MISTRAL_7B, TINY, slice_of
from inputs.vocab import Tokenizer, byte_level_vocab, synthetic_vocab
from inputs.workloads import SINE_SCRIPT_13, codegen_script, plan_stages, validation_call
from paper_2406_00059_b200 import capi

pytestmark = pytest.mark.gpu

BYTE_VOCAB = byte_level_vocab()


def tiny_prompts(n):
    return [list(f"# task {i}\n".encode()) for i in range(n)]


# ------------------------------------------------------------------ the GEMM kernel alone
@pytest.mark.parametrize("N,K,B", [(256, 128, 4), (384, 192, 16), (6144, 4096, 64), (4096, 4096, 64),
                                   (28672, 4096, 64), (4096, 14336, 64), (32000, 4096, 64),
                                   (4096, 4096, 128), (4096, 4096, 200), (4096, 4096, 512), (1000, 640, 33)])
def test_tc_gemm_matches_fp64(N, K, B):
    import torch
    from paper_2406_00059_b200.engine import debug_gemm
    ensure_built()
    g = torch.Generator(device="cuda").manual_seed(N * 7 + K * 3 + B)
    W = (torch.rand((N, K), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    X = (torch.rand((B, K), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    Y, _ = debug_gemm(W, X, N, K, B)
    ref = X.double() @ W.double().T
    err = (Y.double() - ref).abs().max().item()
    assert err < 1e-6 * K + 1e-5, err  # fp32 accumulation of exact bf16 products


@pytest.mark.parametrize("N,K,B", [(4096, 4096, 512), (28672, 4096, 512), (6144, 4096, 512),
                                   (4096, 14336, 512), (4096, 4096, 256), (512, 256, 160),
                                   (6144, 4096, 64), (4096, 14336, 64), (1024, 256, 32),
                                   (28672, 4096, 256), (6144, 4096, 384), (28672, 4096, 384), (14336, 4096, 200)])
def test_tc_gemm_cta_pair_matches_fp64(N, K, B, monkeypatch):
    """CTA-pair (cta_group::2) GEMMs on batch tiles: whole 256-row pair tiles and stream-K over
    pairs, with a non-zero lo plane (the peer CTA's half of the B operand)."""
    import torch
    from paper_2406_00059_b200.engine import debug_gemm
    ensure_built()
    monkeypatch.setenv("CVY_GEMM_PAIR", str(1 << 4))  # EPI_STORE
    if B <= 128:
        monkeypatch.setenv("CVY_GEMM_PAIR_SMALL", "1")
    g = torch.Generator(device="cuda").manual_seed(N * 5 + K + B)
    W = (torch.rand((N, K), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    X = (torch.rand((B, K), generator=g, device="cuda") * 2 - 1).to(torch.bfloat16)
    Xlo = ((torch.rand((B, K), generator=g, device="cuda") * 2 - 1) * 2.0 ** -9).to(torch.bfloat16)
    Y, _ = debug_gemm(W, X, N, K, B, X_lo=Xlo)
    ref = (X.double() + Xlo.double()) @ W.double().T
    err = (Y.double() - ref).abs().max().item()
    assert err < 1e-6 * K + 1e-5, err


# ------------------------------------------------------------------ tiny config, free running
def test_tiny_fp32_free_running_logits_1e4():
    d, gens = free_running_parity(TINY, "fp32", BYTE_VOCAB, tiny_prompts(4), max_new=64, seed=1000, tol=1e-4)
    assert d < 1e-4 and all(len(g) == 64 for g in gens)


def test_tiny_bf16_free_running_logits_2e2():
    d, gens = free_running_parity(TINY, "bf16", BYTE_VOCAB, tiny_prompts(4), max_new=64, seed=1000, tol=2e-2)
    assert d < 2e-2


def test_tiny_bf16_no_graph_matches_graph():
    a, ga = free_running_parity(TINY, "bf16", BYTE_VOCAB, tiny_prompts(3), 16, seed=1001, tol=2e-2, graph=False)
    b, gb = free_running_parity(TINY, "bf16", BYTE_VOCAB, tiny_prompts(3), 16, seed=1001, tol=2e-2, graph=True)
    assert ga == gb


def test_tiny_fp32_with_synthetic_prefix():
    d, _ = free_running_parity(TINY, "fp32", BYTE_VOCAB, tiny_prompts(3), max_new=8, seed=1002, tol=1e-4,
                               prefix=37, synth_seeds=[1, 2, 3])
    assert d < 1e-4


# ------------------------------------------------------------------ 7B shape
def test_7b_two_layer_slice_bf16():
    """2-layer 7B slice, three requests of different prompt lengths over a 40-token prefix."""
    shape = slice_of(MISTRAL_7B, L=2, name="7b-L2")
    vocab = synthetic_vocab(32000)
    prompts = [[1, 300, 5000], [1, 77], [1, 31999, 2000, 12]]
    d, _ = free_running_parity(shape, "bf16", vocab, prompts, max_new=3, seed=1003, tol=2e-2, prefix=40,
                               synth_seeds=[11, 12, 13])
    assert d < 2e-2


def test_pack_weights_tiled_is_the_tile_permutation():
    """cvy_pack_weights_tiled moves element (r, k) of every [L*R][K] projection matrix to
    ((r/128)*(K/64) + k/64)*8192 + (r%128)*64 + k%64 (conveyor.h): bit-exact against the
    row-major weights viewed as [L*R/128][128][K/64][64] and transposed on the middle axes."""
    import torch
    from paper_2406_00059_b200.engine import DeviceModel
    ensure_built()
    sh = slice_of(MISTRAL_7B, L=2, name="7b-L2")
    row = DeviceModel(sh, "bf16", 16, seed=7, tiled=False)
    til = DeviceModel(sh, "bf16", 16, seed=7, tiled=True)
    mats = {"wqkv": ((sh.H + 2 * sh.Hkv) * sh.hd, sh.d, sh.L), "wo": (sh.d, sh.H * sh.hd, sh.L),
            "wgu": (2 * sh.dff, sh.d, sh.L), "wd": (sh.d, sh.dff, sh.L), "lm_head": (sh.V, sh.d, 1)}  # V % 128 == 0
    for name, (R, K, L) in mats.items():
        n = L * R * K * 2
        a = row.tensor(name)[:n].view(torch.int16).view(L * R // 128, 128, K // 64, 64)
        b = til.tensor(name)[:n].view(torch.int16).view(L * R // 128, K // 64, 128, 64)
        assert torch.equal(a.permute(0, 2, 1, 3).contiguous(), b), name
    for name in ("embed", "final_norm", "attn_norm", "mlp_norm"):
        assert torch.equal(row.tensor(name), til.tensor(name)), name


@pytest.mark.parametrize("tiled", ["1", "0"])
def test_7b_two_layer_slice_weight_layouts(tiled, monkeypatch):
    """The projection GEMMs over tile-major (CVY_ENGINE_TILED_WEIGHTS) and row-major weights."""
    monkeypatch.setenv("CVY_TILED_WEIGHTS", tiled)
    shape = slice_of(MISTRAL_7B, L=2, name="7b-L2")
    vocab = synthetic_vocab(32000)
    prompts = [[1, 300, 5000], [1, 77], [1, 31999, 2000, 12]]
    d, _ = free_running_parity(shape, "bf16", vocab, prompts, max_new=3, seed=1003, tol=2e-2, prefix=40,
                               synth_seeds=[11, 12, 13])
    assert d < 2e-2


@pytest.mark.parametrize("H,Hkv,hd,prefix", [(8, 2, 64, 90), (4, 2, 128, 230), (4, 4, 128, 17), (8, 8, 64, 300),
                                             (8, 2, 128, 500)])
def test_tensor_core_attention_shapes(H, Hkv, hd, prefix):
    """The TMA + mma.sync attention kernels across head_dim 64/128 and GQA groups 1, 2, 4,
    contexts spanning several 4-page pipeline stages and split-KV partitions."""
    from inputs.configs import ModelShape
    shape = ModelShape(f"att-{H}-{Hkv}-{hd}", L=2, d=512, H=H, Hkv=Hkv, hd=hd, dff=1024, V=512, eps=1e-5,
                       rope_base=1e4, eos=-1)
    vocab = [bytes([i % 256]) * (1 + i // 256) for i in range(512)]
    prompts = [[5, 300], [7], [100, 200, 300]]
    d, _ = free_running_parity(shape, "bf16", vocab, prompts, max_new=4, seed=1013, tol=2e-2, prefix=prefix,
                               synth_seeds=[21, 22, 23])
    assert d < 2e-3


def test_7b_slice_b40_long_contexts_sampled():
    """40 requests with 100..600-token synthetic contexts on a 2-layer 7B slice: multi-chunk
    attention runs, batch-padded GEMMs.  Sampled requests vs the oracle, two steps."""
    shape = slice_of(MISTRAL_7B, L=2, name="7b-L2")
    vocab = synthetic_vocab(32000)
    B, seed = 40, 1006
    dm, eng = make_engine(shape, "bf16", vocab, B, seed, max_pages_per_slot=40)
    rng = random.Random(5)
    prompts = [[1, rng.randrange(3, 32000), rng.randrange(3, 32000)] for _ in range(B)]
    prefix = [100 + (i * 37) % 500 for i in range(B)]
    rids = [eng.submit_request(p, 2, synth_prefix_len=prefix[i], synth_seed=100 + i) for i, p in enumerate(prompts)]
    sample = [0, 7, 19, 33, 39]
    w = oracle.Weights(shape, seed, bf16=True)
    oreqs = []
    for i in sample:
        r = oracle.Request(w, prefix[i] + 8)
        r.synth_prefix(prefix[i], 100 + i)
        oreqs.append(r)
    for t in range(2):
        eng.step()
        eng.sync()
        ora = oracle.step(oreqs, [prompts[i][t] for i in sample])
        for j, i in enumerate(sample):
            d = float(np.max(np.abs(eng.debug_logits(rids[i]) - ora[j])))
            assert d < 2e-2, (i, t, d)
    eng.poll_segments()
    eng.close()


@pytest.mark.slow
def test_7b_full_32_layers_bf16_b2():
    vocab = synthetic_vocab(32000)
    d, _ = free_running_parity(MISTRAL_7B, "bf16", vocab, [[1, 523], [1, 9000]], max_new=2, seed=1004, tol=2e-2,
                               prefix=16, synth_seeds=[5, 6])
    assert d < 2e-2


@pytest.mark.parametrize("B", [512, 200])
def test_7b_width_large_batch_sampled(B):
    """B=512 (validation-config batch) and B=200 (Bp=256) on a 1-layer 7B-width slice: every GEMM
    runs on 128-column batch tiles (CTA pairs for QKV / gate-up, and O / down at 4 batch tiles);
    sampled requests are checked against the oracle one by one."""
    shape = slice_of(MISTRAL_7B, L=1, name="7b-L1")
    vocab = synthetic_vocab(32000)
    seed = 1005
    dm, eng = make_engine(shape, "bf16", vocab, B, seed, max_pages_per_slot=8)
    rng = random.Random(3)
    prompts = [[1, rng.randrange(3, 32000)] for _ in range(B)]
    rids = [eng.submit_request(p, 2, synth_prefix_len=20 + (i % 50), synth_seed=i) for i, p in enumerate(prompts)]
    sample = sorted({i for i in (0, 1, 137, 255, 256, 300, 511) if i < B} | {B - 1})
    w = oracle.Weights(shape, seed, bf16=True)
    oreqs = {}
    for i in sample:
        r = oracle.Request(w, 100)
        r.synth_prefix(20 + (i % 50), i)
        oreqs[i] = r
    eng.step()
    eng.sync()
    ora = oracle.step([oreqs[i] for i in sample], [prompts[i][0] for i in sample])
    for j, i in enumerate(sample):
        gl = eng.debug_logits(rids[i])
        assert np.max(np.abs(gl - ora[j])) < 2e-2, i
    eng.poll_segments()
    eng.close()


# ------------------------------------------------------------------ trigger scan: bit-exact
def run_forced(eng, reqs, steps_cap=10000):
    """reqs: list of (prompt, forced, tool_id, max_new).  Steps until every FINAL is polled."""
    rids = [eng.submit_request(p, mx, tool_id=t, forced=f) for (p, f, t, mx) in reqs]
    got = []
    finals = set()
    for _ in range(steps_cap):
        eng.step()
        for r in eng.poll_segments():
            got.append(r)
            if r.flags & capi.SEG_FINAL:
                finals.add(r.req_id)
        if len(finals) == len(rids):
            break
    eng.sync()
    for r in eng.poll_segments():
        got.append(r)
    return rids, group_records(got)


def test_tiny_teacher_forced_newline_segments_bitexact():
    dm, eng = make_engine(TINY, "bf16", BYTE_VOCAB, 4, 1006)
    tool = eng.register_tool("python", capi.PARSER_LITERAL, [b"\n"])
    rng = random.Random(5)
    forced = [list(codegen_script(rng, n_lines=8).encode())[:64] for _ in range(4)]
    reqs = [(list(b"# task\n"), f, tool, 64) for f in forced]
    rids, got = run_forced(eng, reqs)
    for rid, f in zip(rids, forced):
        assert as_tuples(got[rid]) == expected_records(f, BYTE_VOCAB, oracle.PARSER_LITERAL, [b"\n"])
    eng.close()


def test_vocab32k_all_parsers_bitexact_b64():
    """Synthetic 32k vocab (delimiters inside multi-byte tokens), three tools, 64 requests:
    code lines with '\\n' and ';' (+ a short max_segment for OVERFLOW), 4-stage JSON plans
    (object completion), validation calls (member completion)."""
    shape = slice_of(TINY, L=2, V=32000, name="tiny-v32k")
    vocab = synthetic_vocab(32000)
    tok = Tokenizer(vocab)
    dm, eng = make_engine(shape, "bf16", vocab, 64, 1007, max_pages_per_slot=48)
    t_code = eng.register_tool("interp", capi.PARSER_LITERAL, [b"\n", b";", b"):\n"])
    t_short = eng.register_tool("interp-short", capi.PARSER_LITERAL, [b"\n"], max_segment_bytes=24)
    t_plan = eng.register_tool("planner", capi.PARSER_JSON_OBJECT)
    t_val = eng.register_tool("validator", capi.PARSER_JSON_MEMBER)
    rng = random.Random(9)
    reqs, meta = [], []
    for i in range(64):
        k = i % 4
        if k == 0:
            text, tool, kind, dl, ms = codegen_script(rng, 30), t_code, oracle.PARSER_LITERAL, [b"\n", b";", b"):\n"], 4096
        elif k == 1:
            text, tool, kind, dl, ms = codegen_script(rng, 20), t_short, oracle.PARSER_LITERAL, [b"\n"], 24
        elif k == 2:
            text, tool, kind, dl, ms = plan_stages(rng), t_plan, oracle.PARSER_JSON_OBJECT, [], 4096
        else:
            text, tool, kind, dl, ms = validation_call(rng, rng.random() < 0.5), t_val, oracle.PARSER_JSON_MEMBER, [], 4096
        f = tok.encode(text)[:500]
        reqs.append(([1, rng.randrange(3, 32000)], f, tool, 600))
        meta.append((f, kind, dl, ms))
    rids, got = run_forced(eng, reqs)
    for rid, (f, kind, dl, ms) in zip(rids, meta):
        assert as_tuples(got[rid]) == expected_records(f, vocab, kind, dl, ms), rid
    eng.close()


def fenced_text(rng, tag="python"):
    """Prose, a bash block (not the tool's tag), the tool's fenced block with code lines and
    one very long line, trailing prose (an unterminated last line is the FINAL tail)."""
    code = codegen_script(rng, rng.randrange(4, 12))
    long_line = "x = [" + ", ".join(str(rng.randrange(1000)) for _ in range(40)) + "]\n"
    return ("Sure, here is the plan.\n```bash\npip install torch\n```\n```" + tag + "\n" + code + long_line +
            "```\nThe figure is saved" + (" as sine.png" if rng.random() < 0.5 else ".\n"))


def test_fence_region_grammar_bitexact():
    """NEXT-2 FENCE parser on the device: byte-level vocab (tiny) and the synthetic 32k vocab
    (markers split across and inside multi-byte tokens), OPEN / piece / CLOSE records, an
    OVERFLOW cut inside the region (max_segment_bytes 64), bit-exact vs oracle.fence_records."""
    for shape, vocab, B in ((TINY, BYTE_VOCAB, 6), (slice_of(TINY, L=2, V=32000, name="tiny-v32k"), synthetic_vocab(32000), 24)):
        dm, eng = make_engine(shape, "bf16", vocab, B, 1008, max_pages_per_slot=64)
        t_py = eng.register_tool("py", capi.PARSER_FENCE, [b"python"], max_segment_bytes=64)
        t_sh = eng.register_tool("sh", capi.PARSER_FENCE, [b"bash"])
        rng = random.Random(13)
        reqs, meta = [], []
        for i in range(B):
            tag, tool, ms = ("python", t_py, 64) if i % 3 else ("bash", t_sh, 4096)
            text = fenced_text(rng, "python")
            if len(vocab) == 256:
                f = list(text.encode())[:900]
            else:
                f = Tokenizer(vocab).encode(text)[:500]
            reqs.append(([1, 7], f, tool, 1000))
            meta.append((f, tag.encode(), ms))
        rids, got = run_forced(eng, reqs)
        n_open = 0
        for rid, (f, tag, ms) in zip(rids, meta):
            exp = expected_records(f, vocab, oracle.PARSER_FENCE, [tag], ms)
            assert as_tuples(got[rid]) == exp, rid
            n_open += sum(1 for r in exp if r[6] & oracle.FLAG_OPEN)
        assert n_open >= B  # every request opened its region
        eng.close()


def call_text(rng):
    """Prose, three @call search lines with JSON arguments (commas and braces inside strings,
    a nested list), an @call for another tool (prose), a long argument (OVERFLOW), trailing prose."""
    lines = ["I need to look up three things."]
    for _ in range(3):
        args = {"q": rng.choice(["hello, world", "a}b{c", "how to \"quote\""]), "n": rng.randrange(10),
                "opts": [1, 2, {"k": "v"}]}
        lines.append("@call search " + json.dumps(args))
    lines.append("@call calculator " + json.dumps({"x": 2}))
    lines.append("@call search " + json.dumps({"long": "y" * rng.randrange(40, 90)}))
    return "\n".join(lines) + "\nThat is all" + ("\n" if rng.random() < 0.5 else "")


def plan_text(rng):
    stages = ["#E1 = search[Microsoft market cap]", "#E2 = search[Apple market cap]",
              "#E3 = calculator[#E1 / #E2]", "#E4 = formatter[ratio=#E3]"]
    noise = ["Thought: compare the two.", "#E5 = bad name[x]", "#E = search[x]", "#E6 = ok[unterminated"]
    lines = ["Plan:"] + [x for st in stages for x in (st, rng.choice(noise))]
    return "\n".join(lines) + "\n#E7 = last[" + "z" * rng.randrange(1, 80) + "]"


@pytest.mark.parametrize("grammar", ["call", "plan"])
def test_call_and_plan_grammars_bitexact(grammar):
    """NEXT-2 CALL (R22) and PLAN (R23) parsers on the device, byte-level and 32k vocabularies,
    with a 64-byte max segment (OVERFLOW inside a call), bit-exact vs the oracle."""
    for shape, vocab, B in ((TINY, BYTE_VOCAB, 6), (slice_of(TINY, L=2, V=32000, name="tiny-v32k"), synthetic_vocab(32000), 24)):
        dm, eng = make_engine(shape, "bf16", vocab, B, 1009, max_pages_per_slot=64)
        if grammar == "call":
            tool = eng.register_tool("search", capi.PARSER_CALL, [b"search"], max_segment_bytes=64)
            kind, dl, ms, gen = oracle.PARSER_CALL, [b"search"], 64, call_text
        else:
            tool = eng.register_tool("planner", capi.PARSER_PLAN, [], max_segment_bytes=64)
            kind, dl, ms, gen = oracle.PARSER_PLAN, [b""], 64, plan_text
        rng = random.Random(29)
        reqs, meta = [], []
        for i in range(B):
            text = gen(rng)
            f = list(text.encode())[:900] if len(vocab) == 256 else Tokenizer(vocab).encode(text)[:500]
            reqs.append(([1, 7], f, tool, 1000))
            meta.append(f)
        rids, got = run_forced(eng, reqs)
        n_rec = 0
        for rid, f in zip(rids, meta):
            exp = expected_records(f, vocab, kind, dl, ms)
            assert as_tuples(got[rid]) == exp, rid
            n_rec += len(exp) - 1
        assert n_rec >= 4 * B
        eng.close()


def test_eos_ends_round_and_multi_round_inject():
    """EOS (id 2, no bytes) ends round 0; the observation is injected and round 1 generates;
    records and seq continue across rounds."""
    import dataclasses
    shape = dataclasses.replace(slice_of(TINY, L=2, V=32000, name="tiny-v32k-eos"), eos=2)
    vocab = synthetic_vocab(32000)
    tok = Tokenizer(vocab)
    dm, eng = make_engine(shape, "fp32", vocab, 2, 1008, max_pages_per_slot=32)
    tool = eng.register_tool("search", capi.PARSER_LITERAL, [b"\n"])
    f0 = tok.encode('search("hello world in Go")\nsearch("x")\n') + [2, 77, 78]
    obs = tok.encode("\n[OBSERVATION search]\nresult text\n")
    f1 = tok.encode("answer: done\n") + [2]
    rid = eng.submit_request([1, 500], 100, tool_id=tool, forced=f0, reserve_tokens=64)
    recs = []
    for _ in range(200):
        eng.step()
        recs += eng.poll_segments()
        if any(r.flags & capi.SEG_FINAL for r in recs):
            break
    n0 = f0.index(2) + 1
    exp0 = expected_records(f0[:n0], vocab, oracle.PARSER_LITERAL, [b"\n"])
    assert as_tuples(recs) == exp0
    assert eng.request_state(rid) == 1
    eng.inject_observation(rid, obs, 50, forced=f1)
    recs1 = []
    for _ in range(200):
        eng.step()
        recs1 += eng.poll_segments()
        if any(r.flags & capi.SEG_FINAL for r in recs1):
            break
    exp1 = expected_records(f1, vocab, oracle.PARSER_LITERAL, [b"\n"], round_idx=1, seq_start=len(exp0))
    assert as_tuples(recs1) == exp1
    assert eng.round_tokens(rid) == f1
    eng.release_request(rid)
    eng.close()


def test_cancel_emits_final_cancelled_with_tail():
    dm, eng = make_engine(TINY, "bf16", BYTE_VOCAB, 2, 1009)
    tool = eng.register_tool("validator", capi.PARSER_JSON_MEMBER)
    rng = random.Random(2)
    f = list(validation_call(rng, True).encode())
    rid = eng.submit_request(list(b"{"), 1000, tool_id=tool, forced=f)
    recs = []
    for _ in range(40):
        eng.step()
        recs += eng.poll_segments()
    eng.cancel_request(rid)
    eng.cancel_request(rid)  # idempotent
    for _ in range(5):
        eng.step()
    eng.sync()
    recs += eng.poll_segments()
    fin = [r for r in recs if r.flags & capi.SEG_FINAL]
    assert len(fin) == 1 and fin[0].flags == capi.SEG_FINAL | capi.SEG_CANCELLED
    n = fin[0].token_index + 1
    assert as_tuples(recs) == expected_records(f[:n], BYTE_VOCAB, oracle.PARSER_JSON_MEMBER, [], cancelled=True)
    assert eng.request_state(rid) == 2
    eng.release_request(rid)
    eng.close()


def test_paper_13_line_script_13_segments_on_gpu():
    dm, eng = make_engine(TINY, "bf16", BYTE_VOCAB, 1, 1010, max_pages_per_slot=32)
    tool = eng.register_tool("python", capi.PARSER_LITERAL, [b"\n"])
    f = list(SINE_SCRIPT_13.encode())
    rids, got = run_forced(eng, [(list(b"```python\n"), f, tool, 1000)])
    recs = got[rids[0]]
    assert len(recs) == 14 and recs[-1].flags == capi.SEG_FINAL and recs[-1].byte_len == 0
    assert b"".join(r.data for r in recs) == SINE_SCRIPT_13.encode()
    eng.close()


def test_submit_errors_and_full():
    dm, eng = make_engine(TINY, "bf16", BYTE_VOCAB, 2, 1011, n_pages=8, max_pages_per_slot=4)
    with pytest.raises(capi.CvyError) as ei:
        eng.submit_request([], 4)
    assert ei.value.status == capi.CVY_E_INVAL
    with pytest.raises(capi.CvyError) as ei:
        eng.submit_request([1], 4, tool_id=5)
    assert ei.value.status == capi.CVY_E_NOTFOUND
    a = eng.submit_request([1], 4)
    b = eng.submit_request([1], 4)
    assert eng.submit_request([1], 4, allow_full=True) is None
    with pytest.raises(capi.CvyError) as ei:
        eng.register_tool("late", capi.PARSER_JSON_OBJECT)
    assert ei.value.status == capi.CVY_E_STATE
    with pytest.raises(capi.CvyError) as ei:
        eng.release_request(a)
    assert ei.value.status == capi.CVY_E_STATE
    eng.close()


def test_degenerate_cases_bitexact():
    """Degenerate inputs: a step with no request in flight is a no-op (no records, no error);
    one-token rounds (LITERAL and JSON tools) give exactly one FINAL holding that token's bytes;
    a stream made only of zero-byte special tokens gives one empty FINAL; a stream without any
    delimiter gives one FINAL with all bytes; max_new_tokens = 1 free-running generates exactly
    one token.  Records bit-exact against the oracle's round_records."""
    vocab = synthetic_vocab(32000)
    shape = slice_of(TINY, L=2, V=32000, name="tiny-v32k")
    dm, eng = make_engine(shape, "bf16", vocab, 8, 1014, max_pages_per_slot=8)
    lit = eng.register_tool("interp", capi.PARSER_LITERAL, [b"\n"])
    js = eng.register_tool("validator", capi.PARSER_JSON_MEMBER)
    for _ in range(3):  # nothing in flight
        eng.step()
    eng.sync()
    assert eng.poll_segments() == []
    tok = Tokenizer(vocab)
    nl = tok.encode("print(1)\n")[-1]
    cases = [(lit, capi.PARSER_LITERAL, [b"\n"], [nl]),                     # one token holding the delimiter
             (js, capi.PARSER_JSON_MEMBER, [], tok.encode("{")[:1]),          # one token, no cut
             (lit, capi.PARSER_LITERAL, [b"\n"], [0, 1, 0]),                  # zero-byte specials only
             (lit, capi.PARSER_LITERAL, [b"\n"], tok.encode("x = 1 + 2 no newline"))]
    rids = [eng.submit_request([1], len(f), tool_id=t, forced=f) for t, _, _, f in cases]
    free = eng.submit_request([1, 5], 1)
    for _ in range(24):
        eng.step()
    eng.sync()
    got = group_records(eng.poll_segments())
    okind = {capi.PARSER_LITERAL: oracle.PARSER_LITERAL, capi.PARSER_JSON_MEMBER: oracle.PARSER_JSON_MEMBER}
    for rid, (_, kind, delims, forced) in zip(rids, cases):
        assert as_tuples(got[rid]) == expected_records(forced, vocab, okind[kind], delims), forced
    assert len(eng.round_tokens(free)) == 1 and eng.request_state(free) == 1
    assert [r.flags & capi.SEG_FINAL for r in got.get(free, [])] in ([], [capi.SEG_FINAL])
    eng.close()


def test_tool_registration_errors():
    dm, eng = make_engine(TINY, "bf16", BYTE_VOCAB, 1, 1012)
    eng.register_tool("a", capi.PARSER_LITERAL, [b"\n"])
    for args, status in [(("a", capi.PARSER_JSON_OBJECT, []), capi.CVY_E_DUP),
                         (("b", capi.PARSER_LITERAL, []), capi.CVY_E_INVAL),
                         (("c", capi.PARSER_LITERAL, [b"123456789"]), capi.CVY_E_INVAL),
                         (("d", capi.PARSER_LITERAL, [b";", b";"]), capi.CVY_E_INVAL),
                         (("e", capi.PARSER_JSON_MEMBER, [b","]), capi.CVY_E_INVAL),
                         (("f", capi.PARSER_FENCE, []), capi.CVY_E_INVAL),
                         (("g", capi.PARSER_FENCE, [b"py", b"sh"]), capi.CVY_E_INVAL),
                         (("h", capi.PARSER_FENCE, [b"py\n"]), capi.CVY_E_INVAL),
                         (("i", capi.PARSER_FENCE, [b"pythonpy3"]), capi.CVY_E_INVAL),
                         (("j", capi.PARSER_FENCE, [b"python"], 8), capi.CVY_E_INVAL),
                         (("k", capi.PARSER_CALL, []), capi.CVY_E_INVAL),
                         (("l", capi.PARSER_CALL, [b"search"], 12), capi.CVY_E_INVAL),
                         (("m", capi.PARSER_PLAN, [b"#"]), capi.CVY_E_INVAL)]:
        with pytest.raises(capi.CvyError) as ei:
            eng.register_tool(*args)
        assert ei.value.status == status
    eng.close()


# ------------------------------------------------------------------ NEXT-1: chunked prefill
@pytest.mark.parametrize("which", ["tiny", "7b-L2", "7b-L2-wide"])
def test_chunked_prefill_prompts_and_observations_match_oracle(which):
    """CVY_ENGINE_CHUNKED_PREFILL: all prompt tokens but the last (and, after a FINAL, the last
    generated token + all observation tokens but the last) run as one batched prefill pass;
    the next decode step starts at the last input.  The oracle is fed the same tokens one by one
    (forced decode, the plain definition); logits of every generating step within tolerance."""
    if which == "tiny":
        shape, vocab = TINY, BYTE_VOCAB
    else:
        shape, vocab = slice_of(MISTRAL_7B, L=2, name="7b-L2"), synthetic_vocab(32000)
    V = shape.V
    rng = random.Random(31)
    B, seed, max_new = 5, 1010, 3
    flags = capi.ENGINE_DEBUG_LOGITS | capi.ENGINE_CHUNKED_PREFILL
    dm, eng = make_engine(shape, "bf16", vocab, B, seed, flags=flags, max_pages_per_slot=16)
    w = oracle.Weights(shape, seed, bf16=True)
    # 1 + 16 + 39 + 150 (+ the 65-token prompt's 64) rows: a 256-row pass (unmerged stream-K GEMMs)
    # 7b-L2-wide: 205 prefill rows -> a 256-row pass on two batch tiles (CTA-pair stream-K QKV and
    # gate/up, cluster split-K O / down)
    last = {"tiny": 151, "7b-L2": 65, "7b-L2-wide": 150}[which]
    prompts = [[rng.randrange(3, V) for _ in range(n)] for n in (1, 2, 17, 40, last)]
    prefix = [0, 9, 0, 21, 3]
    obs = [[rng.randrange(3, V) for _ in range(n)] for n in (1, 5, 30, 2, 0)]
    oreqs, rids = [], []
    for i, p in enumerate(prompts):
        r = oracle.Request(w, 256)
        if prefix[i]:
            r.synth_prefix(prefix[i], 40 + i)
        for t in p[:-1]:
            oracle.step([r], [t])
        oreqs.append(r)
        rids.append(eng.submit_request(p, max_new, synth_prefix_len=prefix[i], synth_seed=40 + i))
    nxt = [p[-1] for p in prompts]
    worst = 0.0
    for rnd in range(2):
        gens = [[] for _ in range(B)]
        for t in range(max_new):
            eng.step()
            eng.sync()
            ora = oracle.step(oreqs, nxt)
            for i in range(B):
                gl = eng.debug_logits(rids[i])
                d = float(np.max(np.abs(gl.astype(np.float64) - ora[i])))
                worst = max(worst, d)
                assert d < 2e-2, (which, rnd, t, i, d)
                g = eng.round_tokens(rids[i])[-1]
                assert ora[i][g] >= ora[i].max() - 4e-2
                gens[i].append(g)
                nxt[i] = g
        for _ in range(3):
            eng.step()
            eng.poll_segments()
        eng.sync()
        eng.poll_segments()
        if rnd == 0:
            for i in range(B):
                # next round: last generated token, then the observation (R19)
                seq = [gens[i][-1]] + obs[i]
                for t in seq[:-1]:
                    oracle.step([oreqs[i]], [t])
                nxt[i] = seq[-1]
                eng.inject_observation(rids[i], obs[i], max_new)
    assert worst < 2e-2
    eng.close()


# ------------------------------------------------------------------ round-2 parity gaps
def test_json_overflow_bitexact_short_segments():
    """JSON_MEMBER / JSON_OBJECT with max_segment_bytes 16..64 (R13: an OVERFLOW cut every M bytes
    without a natural cut; the automaton state carries on), 32k vocab, bit-exact vs the oracle."""
    shape = slice_of(TINY, L=2, V=32000, name="tiny-v32k")
    vocab = synthetic_vocab(32000)
    tok = Tokenizer(vocab)
    dm, eng = make_engine(shape, "bf16", vocab, 32, 1021, max_pages_per_slot=48)
    cfgs = [(capi.PARSER_JSON_MEMBER, 16), (capi.PARSER_JSON_MEMBER, 24), (capi.PARSER_JSON_MEMBER, 40),
            (capi.PARSER_JSON_MEMBER, 64), (capi.PARSER_JSON_OBJECT, 20), (capi.PARSER_JSON_OBJECT, 48)]
    tools = [eng.register_tool(f"json{i}", kind, max_segment_bytes=ms) for i, (kind, ms) in enumerate(cfgs)]
    rng = random.Random(21)
    reqs, meta = [], []
    for i in range(32):
        k = i % len(cfgs)
        kind, ms = cfgs[k]
        text = validation_call(rng, rng.random() < 0.5) if kind == capi.PARSER_JSON_MEMBER else plan_stages(rng)
        f = tok.encode(text)[:500]
        reqs.append(([1, rng.randrange(3, 32000)], f, tools[k], 600))
        meta.append((f, kind, ms))
    rids, got = run_forced(eng, reqs)
    n_over = 0
    for rid, (f, kind, ms) in zip(rids, meta):
        exp = expected_records(f, vocab, kind, [], ms)
        assert as_tuples(got[rid]) == exp, rid
        n_over += sum(1 for r in exp if r[6] & oracle.FLAG_OVERFLOW)
    assert n_over > 50  # the OVERFLOW branch is exercised, not just reachable
    eng.close()


def test_ring_wrap_and_backpressure_bitexact():
    """The smallest ring the ABI accepts (32 x slots records, power of two) carries > 10x its
    capacity while a slow poller thread drains it: cvy_step blocks on back-pressure instead of
    overwriting, and every request's record sequence stays bit-exact."""
    import threading
    import time
    B = 16
    ring = 512  # pow2 >= 32 * 16
    dm, eng = make_engine(TINY, "bf16", BYTE_VOCAB, B, 1022, ring_records=ring, max_pages_per_slot=40)
    delims = [b"a", b";", b"\n"]
    tool = eng.register_tool("dense", capi.PARSER_LITERAL, delims)
    rng = random.Random(22)
    forced = [[rng.choice(b"ab;\n") for _ in range(450)] for _ in range(B)]
    rids = [eng.submit_request(list(b"# t\n"), 1000, tool_id=tool, forced=f) for f in forced]
    got, stop = [], threading.Event()

    def poller():
        while not stop.is_set():
            got.extend(eng.poll_segments())
            time.sleep(0.004)

    th = threading.Thread(target=poller, daemon=True)
    th.start()
    blocked_steps = 0
    for _ in range(470):
        t0 = time.perf_counter()
        eng.step()
        blocked_steps += (time.perf_counter() - t0) > 0.003
    eng.sync()
    time.sleep(0.05)
    stop.set()
    th.join()
    got.extend(eng.poll_segments())
    by = group_records(got)
    total = sum(len(v) for v in by.values())
    assert total > 10 * ring
    assert blocked_steps > 0  # back-pressure actually engaged
    for rid, f in zip(rids, forced):
        assert as_tuples(by[rid]) == expected_records(f, BYTE_VOCAB, oracle.PARSER_LITERAL, delims), rid
    eng.close()


def test_abort_and_refill_matches_oracle():
    """NEXT-3 on the real engine: 32 validation requests through 8 slots.  A request whose
    `location` member (seq 2) lacks ', ST' is cancelled when that record is polled (the
    validator's abort); finished / aborted requests are released at once and the
    next queued request is admitted into the freed slot.  Every request's records are bit-exact
    against the oracle (aborted ones: the stream up to the GPU's cut, FINAL|CANCELLED), and every
    step's logits of every request -- refilled slots included -- are within 2e-2 of the oracle."""
    shape = slice_of(TINY, L=2, V=32000, name="tiny-v32k")
    vocab = synthetic_vocab(32000)
    tok = Tokenizer(vocab)
    S, N = 8, 32
    seed = 1023
    dm, eng = make_engine(shape, "bf16", vocab, S, seed, max_pages_per_slot=40)
    tool = eng.register_tool("validator", capi.PARSER_JSON_MEMBER)
    rng = random.Random(23)
    bad = [rng.random() < 0.5 for _ in range(N)]
    forced = [tok.encode(validation_call(rng, b))[:300] for b in bad]
    prompts = [[1, rng.randrange(3, 32000)] for _ in range(N)]
    w = oracle.Weights(shape, seed, bf16=True)
    queue = list(range(N))
    live = {}      # rid -> [request index, oracle request, inputs fed, refilled slot?, cancel issued?]
    recs, finished, rid_of = {}, {}, {}
    maxdiff, refilled_checked, admitted = 0.0, 0, 0

    def admit():
        nonlocal admitted
        while queue and len(live) < S:
            i = queue.pop(0)
            rid = eng.submit_request(prompts[i], 1000, tool_id=tool, forced=forced[i])
            live[rid] = [i, oracle.Request(w, len(prompts[i]) + len(forced[i]) + 4), 0, admitted >= S, False]
            rid_of[i] = rid
            recs[rid] = []
            admitted += 1

    admit()
    for _ in range(4000):
        if not live:
            break
        eng.step()
        eng.sync()
        # every live request ran this step (submitted before it, round not over): compare its
        # logits with the oracle fed the same input -- until a cancel makes the step count uncertain
        ins, ors, gls = [], [], []
        for rid, st in live.items():
            i, orq, j, refill, cancelled = st
            n_in = len(prompts[i]) + len(forced[i]) - 1
            if cancelled or j >= n_in:
                continue
            ins.append(prompts[i][j] if j < len(prompts[i]) else forced[i][j - len(prompts[i])])
            ors.append(orq)
            gls.append((eng.debug_logits(rid), refill))
            st[2] = j + 1
        if ors:
            for (gl, refill), o in zip(gls, oracle.step(ors, ins)):
                d = float(np.max(np.abs(gl.astype(np.float64) - o)))
                maxdiff = max(maxdiff, d)
                assert d < 2e-2, d
                refilled_checked += refill
        for r in eng.poll_segments():
            recs[r.req_id].append(r)
            st = live.get(r.req_id)
            if st and bad[st[0]] and r.seq == 2 and not (r.flags & capi.SEG_FINAL) and not st[4]:
                eng.cancel_request(r.req_id)  # the validator's abort
                st[4] = True
            if r.flags & capi.SEG_FINAL:
                finished[r.req_id] = r
        for rid in [x for x in live if x in finished]:
            eng.release_request(rid)  # frees the slot and its pages at once ...
            del live[rid]
        admit()                       # ... and the next queued request takes it
    assert not live and not queue and len(finished) == N
    n_cancelled = 0
    for i in range(N):
        rid = rid_of[i]
        fin = finished[rid]
        cancelled = bool(fin.flags & capi.SEG_CANCELLED)
        n_cancelled += cancelled
        n = fin.token_index + 1 if cancelled else len(forced[i])
        exp = expected_records(forced[i][:n], vocab, oracle.PARSER_JSON_MEMBER, [], cancelled=cancelled)
        assert as_tuples(recs[rid]) == exp, i
        if cancelled:
            assert bad[i] and n < len(forced[i])
    assert n_cancelled >= 8 and refilled_checked > 100
    eng.close()


def multi_tool_text(rng):
    """Prose, a ```python block, an @call search, a ```bash block, an @call calc, a fence of a
    tag outside the set (prose), in a seeded order."""
    parts = ["Plan: run the script, then query.\n",
             "```python\n" + codegen_script(rng, rng.randint(4, 8)) + "```\n",
             "@call search " + json.dumps({"q": "sine wave " + str(rng.randint(0, 99)), "n": 3}) + "\n",
             "```bash\nls -la /tmp\necho done; cat out.txt\n```\n",
             "@call calc " + json.dumps({"expr": f"{rng.randint(1, 99)} * {rng.randint(1, 99)}"}) + " ok\n",
             "```js\nconsole.log(1)\n```\n",
             "Finally: " + "".join(rng.choice("abc ,\n") for _ in range(30))]
    rng.shuffle(parts)
    return "".join(parts)


@pytest.mark.parametrize("vocab_kind", ["byte", "32k"])
def test_multi_tool_sets_bitexact(vocab_kind):
    """NEXT-2 multi-tool routing (R24): each request holds a SET of region tools -- python and
    bash FENCE tools and search and calc CALL tools -- and the marker that appears selects the
    tool; records carry the tool id.  Bit-exact (tool field included) against oracle
    region_records, with OVERFLOW inside regions (a short max_segment_bytes on one tool)."""
    if vocab_kind == "byte":
        shape, vocab = TINY, BYTE_VOCAB
        enc = lambda t: list(t.encode())
    else:
        shape, vocab = slice_of(TINY, L=2, V=32000, name="tiny-v32k"), synthetic_vocab(32000)
        tok = Tokenizer(vocab)
        enc = tok.encode
    dm, eng = make_engine(shape, "bf16", vocab, 16, 1024, max_pages_per_slot=64)
    specs = [("py", capi.PARSER_FENCE, b"python", 4096), ("sh", capi.PARSER_FENCE, b"bash", 24),
             ("search", capi.PARSER_CALL, b"search", 4096), ("calc", capi.PARSER_CALL, b"calc", 4096)]
    ids = {n: eng.register_tool(n, k, [tag], max_segment_bytes=ms) for (n, k, tag, ms) in specs}
    region_tools = [(ids[n], k, tag, ms) for (n, k, tag, ms) in specs]
    rng = random.Random(24)
    reqs, forced = [], []
    for i in range(16):
        f = enc(multi_tool_text(rng))[:900]
        forced.append(f)
        reqs.append(f)
    rids = [eng.submit_request([1, 10], 1000, forced=f, tool_set=list(ids.values())) for f in reqs]
    got = []
    finals = set()
    for _ in range(2000):
        eng.step()
        for r in eng.poll_segments():
            got.append(r)
            if r.flags & capi.SEG_FINAL:
                finals.add(r.req_id)
        if len(finals) == len(rids):
            break
    eng.sync()
    got += eng.poll_segments()
    by = group_records(got)
    n_tools_seen = set()
    for rid, f in zip(rids, forced):
        exp, _ = round_records(f, vocab, 0, [], 4096, region_tools=region_tools)
        want = [(r.round, r.seq, r.token_index, r.byte_offset, r.byte_len, r.delim_id, r.flags, r.data, r.tool)
                for r in exp]
        have = [(r.round, r.seq, r.token_index, r.byte_offset, r.byte_len, r.delim_id, r.flags, r.data, r.tool)
                for r in by[rid]]
        assert have == want, rid
        n_tools_seen |= {r[8] for r in want if r[8] >= 0}
    assert n_tools_seen == set(ids.values())
    eng.close()


def test_prefill_attention_is_deterministic_with_odd_page_counts():
    """Regression: with 2 pages per stage, the warp of a pair that has no page in the last stage
    (odd page count) used to arrive on the slot's empty barrier without waiting for the stage --
    its arrival could complete the PREVIOUS phase while its partner was still reading, and the
    producer overwrote that page (rows with 5 pages of keys came out wrong ~1 run in 4).  The
    attention output of a chunked-prefill pass with such rows must be identical run to run."""
    import ctypes
    shape, vocab = slice_of(MISTRAL_7B, L=1, name="7b-L1"), synthetic_vocab(32000)
    ref = None
    for rep in range(6):
        rng = random.Random(31)
        flags = capi.ENGINE_DEBUG_LOGITS | capi.ENGINE_CHUNKED_PREFILL
        dm, eng = make_engine(shape, "bf16", vocab, 5, 1010, flags=flags, max_pages_per_slot=16)
        prompts = [[rng.randrange(3, shape.V) for _ in range(n)] for n in (1, 2, 17, 40, 65)]
        for i, p in enumerate(prompts):
            eng.submit_request(p, 3, synth_prefix_len=[0, 9, 0, 21, 3][i], synth_seed=40 + i)
        eng.step()
        eng.sync()
        nb = ctypes.c_size_t()
        assert capi.lib().cvy_debug_buffer(eng.h, 20, None, 0, ctypes.byref(nb)) == 0
        o = np.zeros(nb.value, dtype=np.uint8)
        assert capi.lib().cvy_debug_buffer(eng.h, 20, o.ctypes.data_as(ctypes.c_void_p), nb.value,
                                           ctypes.byref(nb)) == 0
        eng.close()
        if ref is None:
            ref = o
        else:
            assert np.array_equal(o, ref), f"attention output differs in repetition {rep}"
