"""Pins for oracle O-1 (decoder forward) against things other than itself.

 * HF MistralForCausalLM (transformers, fp64, CPU) with the same weights: the paper only
   names Mistral-7B-Instruct-v0.2, so the architecture reading (R1-R3) is
   pinned to the library definition of that family -- tiny config and a 1-layer slice at
   the full 7B width (d=4096, GQA 32/8, hd=128, RoPE base 1e6).
 * HF with an injected post-RoPE KV prefix (DynamicCache) pins the synthetic-prefix path.
 * splitmix64 textbook value, bf16 rounding vs torch, argmax tie / NaN rules (R6),
   batch independence (continuous batching), KV-cache decode == full causal
   forward.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from inputs.configs import MISTRAL_7B, TINY, slice_of


def hf_model(shape, w: "oracle.Weights"):
    from transformers import MistralConfig, MistralForCausalLM
    cfg = MistralConfig(vocab_size=shape.V, hidden_size=shape.d, intermediate_size=shape.dff,
                        num_hidden_layers=shape.L, num_attention_heads=shape.H,
                        num_key_value_heads=shape.Hkv, head_dim=shape.hd, rms_norm_eps=shape.eps,
                        sliding_window=None, tie_word_embeddings=False,
                        max_position_embeddings=8192, rope_theta=shape.rope_base)
    torch.manual_seed(0)
    m = MistralForCausalLM(cfg).double().eval()
    sd = m.state_dict()
    H, Hkv, hd, d, dff, V = shape.H, shape.Hkv, shape.hd, shape.d, shape.dff, shape.V
    def put(name, tid, r, c):
        sd[name].copy_(torch.from_numpy(w.tensor(tid, r, c)))
    put("model.embed_tokens.weight", oracle.tid_embed(), V, d)
    put("lm_head.weight", oracle.tid_lm_head(shape.L), V, d)
    for l in range(shape.L):
        p = f"model.layers.{l}."
        put(p + "self_attn.q_proj.weight", oracle.tid_layer(l, "wq"), H * hd, d)
        put(p + "self_attn.k_proj.weight", oracle.tid_layer(l, "wk"), Hkv * hd, d)
        put(p + "self_attn.v_proj.weight", oracle.tid_layer(l, "wv"), Hkv * hd, d)
        put(p + "self_attn.o_proj.weight", oracle.tid_layer(l, "wo"), d, H * hd)
        put(p + "mlp.gate_proj.weight", oracle.tid_layer(l, "wg"), dff, d)
        put(p + "mlp.up_proj.weight", oracle.tid_layer(l, "wu"), dff, d)
        put(p + "mlp.down_proj.weight", oracle.tid_layer(l, "wd"), d, dff)
        sd[p + "input_layernorm.weight"].fill_(1.0)
        sd[p + "post_attention_layernorm.weight"].fill_(1.0)
    sd["model.norm.weight"].fill_(1.0)
    m.load_state_dict(sd)
    return m


def oracle_incremental(w, tokens, prefix=0, synth_seed=0):
    r = oracle.Request(w, max_ctx=prefix + len(tokens) + 1)
    if prefix:
        r.synth_prefix(prefix, synth_seed)
    return np.stack([oracle.step([r], [t])[0] for t in tokens])


def test_splitmix64_textbook_value():
    # SplitMix64 from state 0: first output 0xE220A8397B1DCDAF (Vigna's reference sequence)
    h = 0xE220A8397B1DCDAF
    u = (h >> 11) * 2.0 ** -53
    a = 0.02 * math.sqrt(3.0)
    exp = float(np.float32(a * (2 * u - 1)))
    assert oracle.hash_value(0, 0, 0, a, False) == exp


def test_bf16_round_matches_torch():
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.standard_normal(2000), rng.standard_normal(200) * 1e-3, [0.0, -1.0, 3.0]])
    for x in xs:
        ref = torch.tensor(float(np.float32(x)), dtype=torch.float32).to(torch.bfloat16).double().item()
        assert oracle.bf16_round(float(x)) == ref


def test_weights_distribution():
    w = oracle.Weights(TINY, seed=1000, bf16=False)
    e = w.tensor(oracle.tid_layer(0, "wd"), TINY.d, TINY.dff)
    assert abs(e.std() - 0.02) < 0.002 and abs(e.mean()) < 0.002
    assert np.all(np.abs(e) <= 0.02 * math.sqrt(3) + 1e-9)


@pytest.mark.parametrize("bf16w", [False, True])
def test_tiny_matches_hf_mistral(bf16w):
    w = oracle.Weights(TINY, seed=1000, bf16=bf16w)
    toks = [35, 9, 200, 17, 17, 101, 10, 255, 0, 64, 65, 66]
    mine = oracle_incremental(w, toks)
    m = hf_model(TINY, w)
    with torch.no_grad():
        ref = m(torch.tensor([toks])).logits[0].numpy()
    # KV cache stored as fp32 (bf16 for bf16 models) is the only rounding in exact mode
    tol = 1e-5 if not bf16w else 2e-3
    assert np.max(np.abs(mine - ref)) < tol
    assert np.max(np.abs(ref)) > 0.1


def test_tiny_prefix_matches_hf_with_injected_cache():
    from transformers import DynamicCache
    w = oracle.Weights(TINY, seed=1001, bf16=False)
    P, seed = 9, 5
    toks = [3, 77, 10, 10, 42]
    mine = oracle_incremental(w, toks, prefix=P, synth_seed=seed)
    m = hf_model(TINY, w)
    sh = TINY
    cache = DynamicCache()
    for l in range(sh.L):
        tid = (1 << 62) ^ (seed * sh.L + l)
        K = np.zeros((1, sh.Hkv, P, sh.hd))
        Vv = np.zeros((1, sh.Hkv, P, sh.hd))
        for pos in range(P):
            for c in range(2):
                for g in range(sh.Hkv):
                    for e in range(sh.hd):
                        i = ((pos * 2 + c) * sh.Hkv + g) * sh.hd + e
                        val = oracle.hash_value(0, tid, i, math.sqrt(3.0), False)
                        (K if c == 0 else Vv)[0, g, pos, e] = val
        cache.update(torch.from_numpy(K), torch.from_numpy(Vv), l)
    with torch.no_grad():
        out = m(torch.tensor([toks]), past_key_values=cache,
                position_ids=torch.arange(P, P + len(toks))[None], use_cache=True)
    ref = out.logits[0].numpy()
    assert np.max(np.abs(mine - ref)) < 1e-5


@pytest.mark.slow
def test_7b_width_slice_matches_hf():
    shape = slice_of(MISTRAL_7B, L=1, V=512, name="7b-width-L1")
    w = oracle.Weights(shape, seed=1003, bf16=False, cache=True)
    toks = [5, 300, 2, 77]
    mine = oracle_incremental(w, toks)
    m = hf_model(shape, w)
    with torch.no_grad():
        ref = m(torch.tensor([toks])).logits[0].numpy()
    assert np.max(np.abs(mine - ref)) < 1e-5  # fp32 KV cache rounding only
    del m


def test_batch_independence_and_slot_order():
    w = oracle.Weights(TINY, seed=1002, bf16=True)
    seqs = [[1, 2, 3, 4], [200, 100, 50, 25], [9, 9, 9, 9]]
    alone = [oracle_incremental(w, s) for s in seqs]
    reqs = [oracle.Request(w, 8) for _ in seqs]
    order = [2, 0, 1]
    for t in range(4):
        lg = oracle.step([reqs[i] for i in order], [seqs[i][t] for i in order])
        for j, i in enumerate(order):
            assert np.array_equal(lg[j], alone[i][t])


def test_argmax_rules():
    assert oracle.argmax(np.array([1.0, 3.0, 3.0, 2.0])) == 1
    assert oracle.argmax(np.array([np.nan, -5.0, np.nan])) == 1
    assert oracle.argmax(np.array([-np.inf, -np.inf])) == 0
    x = np.zeros(100)
    x[37] = 1e-12
    assert oracle.argmax(x) == 37


def test_zero_layer_closed_form():
    """L=0 special case (no attention, no MLP): logits = RMSNorm(E[x]) W_lm^T."""
    shape = slice_of(TINY, L=0, name="tiny-L0")
    w = oracle.Weights(shape, seed=1005, bf16=False)
    E = w.tensor(oracle.tid_embed(), shape.V, shape.d)
    W = w.tensor(oracle.tid_lm_head(0), shape.V, shape.d)
    for tok in [0, 17, 255]:
        lg = oracle_incremental(w, [tok])[0]
        x = E[tok]
        u = x / np.sqrt(np.mean(x * x) + shape.eps)
        assert np.allclose(lg, W @ u, atol=1e-12, rtol=1e-10)
