// epilogue.cuh -- fused GEMM epilogues (RMSNorm scale, RoPE + paged-KV append, residual
// add + next-norm input, SwiGLU, LM-head tile argmax) and the sampling / trigger-scan /
// compaction epilogue (K6) that runs in the CTA finishing the last LM-head tile.
//
// Every epilogue runs on 128 threads ("et" = 0..127 = the tile row owned by the thread)
// over column chunks of 32 batch entries; values arrive in registers from TMEM (tcgen05
// path), from the stream-K accumulator (multi-CTA tiles) or from the SIMT fp32 GEMM.
#pragma once
#include "common.cuh"
#include "step_params.h"

namespace cvy {

constexpr int kEpiThreads = 128;
constexpr int kEsmLd = 33;  // padded row of the [128][33] exchange buffer
constexpr uint32_t kEpiBar = 1;

// 128-thread barrier of this thread's epilogue group: threads 0..127 (barrier 1), or the second
// group of the gate/up GEMM, threads 192..319 (barrier 3); see gemm_sm100.cuh
CVY_DEV void epi_sync() { named_bar_sync(threadIdx.x >= 192 ? 3u : kEpiBar, kEpiThreads); }

// Per-column (= per slot) metadata the epilogues need, gathered once per CTA into shared
// memory so the per-element epilogue never chases global pointers:
//   scale[b]  = 1/sqrt(mean(x_b^2) + eps) from the per-128-block partial sums (fixed order)
//   pos[b]    = position of the slot's current token (RoPE angle)
//   kvoff[b]  = element offset, inside one layer of the KV pool, of (page(pos), K, kv-head 0,
//               row pos%16); -1 if the slot is idle or out of reserved positions.
struct EpiMeta {
    float* scale;
    int* pos;
    long long* kvoff;
};
CVY_DEV void epilogue_prepare(const StepParams& P, const EpiArgs& E, EpiMeta& m, int et) {
    const int nblk = P.d / 128;
    if (E.kind == EPI_QKV || E.kind == EPI_SWIGLU || E.kind == EPI_LMHEAD) {
        for (int b = et; b < P.Bp; b += kEpiThreads) {
            float acc = 0.f;
            for (int t = 0; t < nblk; ++t) acc += P.ssq[(size_t)t * P.Bmax + b];
            m.scale[b] = rsqrtf(acc / (float)P.d + P.eps);
        }
    }
    if (E.kind == EPI_QKV) {
        const size_t page_elems = (size_t)2 * P.Hkv * kPageTokens * P.hd;
        for (int b = et; b < P.Bp; b += kEpiThreads) {
            int pos, sb;
            bool ok;
            if (P.row_slot) {  // prefill row (NEXT-1): the host reserved its pages
                pos = P.row_pos[b];
                sb = P.row_slot[b];
                ok = pos >= 0;
            } else {
                const SlotDev& s = P.slots[b];
                pos = s.pos;
                sb = b;
                ok = s.active && pos < s.max_pos;
            }
            long long off = -1;
            if (ok) {
                const int page = P.page_table[(size_t)sb * P.max_pages + pos / kPageTokens];
                off = (long long)((size_t)page * page_elems + (size_t)(pos % kPageTokens) * P.hd);
            }
            m.pos[b] = min(max(pos, 0), P.max_rope_pos - 1);
            m.kvoff[b] = off;
        }
    }
}

// 16-byte vector stores of a run of consecutive rows of one column (16-B aligned targets)
template <typename T> CVY_DEV void store_row32(T* dst, const float* w);
template <> CVY_DEV void store_row32<float>(float* dst, const float* w) {
    float4* d = reinterpret_cast<float4*>(dst);
#pragma unroll
    for (int q = 0; q < 8; ++q) d[q] = make_float4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
}
template <> CVY_DEV void store_row32<__nv_bfloat16>(__nv_bfloat16* dst, const float* w) {
    uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        __nv_bfloat162 p0 = __floats2bfloat162_rn(w[8 * q], w[8 * q + 1]);
        __nv_bfloat162 p1 = __floats2bfloat162_rn(w[8 * q + 2], w[8 * q + 3]);
        __nv_bfloat162 p2 = __floats2bfloat162_rn(w[8 * q + 4], w[8 * q + 5]);
        __nv_bfloat162 p3 = __floats2bfloat162_rn(w[8 * q + 6], w[8 * q + 7]);
        d[q] = make_uint4(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1),
                          *reinterpret_cast<uint32_t*>(&p2), *reinterpret_cast<uint32_t*>(&p3));
    }
}
// NR (16 or 32) consecutive rows of one column, 16-byte vectors
template <typename T, int NR> CVY_DEV void store_rows(T* dst, const float* w);
template <> CVY_DEV void store_rows<float, 32>(float* dst, const float* w) { store_row32<float>(dst, w); }
template <> CVY_DEV void store_rows<__nv_bfloat16, 32>(__nv_bfloat16* dst, const float* w) { store_row32<__nv_bfloat16>(dst, w); }
template <> CVY_DEV void store_rows<float, 16>(float* dst, const float* w) {
    float4* d = reinterpret_cast<float4*>(dst);
#pragma unroll
    for (int q = 0; q < 4; ++q) d[q] = make_float4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
}
template <> CVY_DEV void store_rows<__nv_bfloat16, 16>(__nv_bfloat16* dst, const float* w) {
    uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        __nv_bfloat162 p0 = __floats2bfloat162_rn(w[8 * q], w[8 * q + 1]);
        __nv_bfloat162 p1 = __floats2bfloat162_rn(w[8 * q + 2], w[8 * q + 3]);
        __nv_bfloat162 p2 = __floats2bfloat162_rn(w[8 * q + 4], w[8 * q + 5]);
        __nv_bfloat162 p3 = __floats2bfloat162_rn(w[8 * q + 6], w[8 * q + 7]);
        d[q] = make_uint4(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1),
                          *reinterpret_cast<uint32_t*>(&p2), *reinterpret_cast<uint32_t*>(&p3));
    }
}
// (hi, lo) activation planes of a run of N consecutive rows (N = 16 or 32)
template <typename T, int NR> CVY_DEV void store_act_rows(T* dst, size_t plane, const float* w);
template <> CVY_DEV void store_act_rows<float, 32>(float* dst, size_t, const float* w) { store_row32<float>(dst, w); }
template <> CVY_DEV void store_act_rows<float, 16>(float* dst, size_t, const float* w) {
    float4* d = reinterpret_cast<float4*>(dst);
#pragma unroll
    for (int q = 0; q < 4; ++q) d[q] = make_float4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
}
template <int NR> CVY_DEV void store_act_rows_bf16(__nv_bfloat16* dst, size_t plane, const float* w) {
    uint32_t hi[NR / 2], lo[NR / 2];
#pragma unroll
    for (int r = 0; r < NR; r += 2) {
        const __nv_bfloat16 h0 = __float2bfloat16_rn(w[r]), h1 = __float2bfloat16_rn(w[r + 1]);
        const __nv_bfloat16 l0 = __float2bfloat16_rn(w[r] - __bfloat162float(h0));
        const __nv_bfloat16 l1 = __float2bfloat16_rn(w[r + 1] - __bfloat162float(h1));
        __nv_bfloat162 ph, pl;
        ph.x = h0; ph.y = h1;
        pl.x = l0; pl.y = l1;
        hi[r / 2] = *reinterpret_cast<uint32_t*>(&ph);
        lo[r / 2] = *reinterpret_cast<uint32_t*>(&pl);
    }
    uint4* dh = reinterpret_cast<uint4*>(dst);
    uint4* dl = reinterpret_cast<uint4*>(dst + plane);
#pragma unroll
    for (int q = 0; q < NR / 8; ++q) {
        dh[q] = make_uint4(hi[4 * q], hi[4 * q + 1], hi[4 * q + 2], hi[4 * q + 3]);
        dl[q] = make_uint4(lo[4 * q], lo[4 * q + 1], lo[4 * q + 2], lo[4 * q + 3]);
    }
}
template <> CVY_DEV void store_act_rows<__nv_bfloat16, 32>(__nv_bfloat16* dst, size_t plane, const float* w) {
    store_act_rows_bf16<32>(dst, plane, w);
}
template <> CVY_DEV void store_act_rows<__nv_bfloat16, 16>(__nv_bfloat16* dst, size_t plane, const float* w) {
    store_act_rows_bf16<16>(dst, plane, w);
}
template <typename T> CVY_DEV void store_act_row32(T* dst, size_t plane, const float* w) { store_act_rows<T, 32>(dst, plane, w); }
template <typename T> CVY_DEV void store_act_row16(T* dst, size_t plane, const float* w) { store_act_rows<T, 16>(dst, plane, w); }

// One 32-column chunk of one 128-row sub-tile.  n0 = first global row of the sub-tile.
// W = columns in v (32, or 16 for the split-K reduce-scatter units): the per-row loops run W
// iterations (instruction latency is what bounds an epilogue).
template <typename T, int KIND = -1, int W = 32>
CVY_DEV void epilogue_chunk(const StepParams& P, const EpiArgs& E, int n0, int cb, float* v, float* esm,
                            const EpiMeta& M, int et) {
    static_assert(W == 16 || W == 32, "chunk width");
    const float* s_scale = M.scale;
    const int n = n0 + et;
    const int ncols = min(W, P.Bp - cb);
    switch (KIND >= 0 ? KIND : E.kind) {
        case EPI_QKV: {
            const int hd = P.hd, half = hd >> 1;
            const int qk_rows = (P.H + P.Hkv) * hd;
            const int dim = n % hd;
            const int j = dim & (half - 1);
            const bool rot = n < qk_rows;
            // all global inputs first (RoPE cos/sin of every column), then compute, then store
            float2 cs[32];
#pragma unroll
            for (int i = 0; i < W; ++i)
                cs[i] = (rot && i < ncols) ? __ldg(&P.rope[(size_t)M.pos[cb + i] * half + j]) : make_float2(1.f, 0.f);
#pragma unroll
            for (int i = 0; i < W; ++i) v[i] *= s_scale[cb + i];
#pragma unroll
            for (int i = 0; i < W; ++i) esm[et * kEsmLd + i] = v[i];
            epi_sync();
            const int partner = et ^ half;
            float out[32];
#pragma unroll
            for (int i = 0; i < W; ++i) {
                const float pv = esm[partner * kEsmLd + i];
                out[i] = dim < half ? (v[i] * cs[i].x - pv * cs[i].y) : (v[i] * cs[i].x + pv * cs[i].y);
            }
            epi_sync();
#pragma unroll
            for (int i = 0; i < W; ++i) esm[et * kEsmLd + i] = out[i];
            epi_sync();
            // transposed stores: thread -> (column b, RP = W consecutive rows), 16-byte vectors;
            // 128 / RP threads per column, so every epilogue thread works at W = 16 too
            {
                constexpr int RP = W, NPART = 128 / W;
                const int col = et / NPART, part = et % NPART;
                const int r0 = n0 + part * RP;
                if (col < ncols && r0 < E.N) {
                    const int b = cb + col;
                    float w[RP];
#pragma unroll
                    for (int r = 0; r < RP; ++r) w[r] = esm[(part * RP + r) * kEsmLd + col];
                    if (r0 < P.H * hd) {
                        float4* dq = reinterpret_cast<float4*>(P.q + (size_t)b * (P.H * hd) + r0);
#pragma unroll
                        for (int q = 0; q < RP / 4; ++q) dq[q] = make_float4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
                    } else if (M.kvoff[b] >= 0) {
                        const int c = r0 >= qk_rows ? 1 : 0;
                        const int rel = r0 - P.H * hd - c * P.Hkv * hd;
                        const int g = rel / hd, e = rel % hd;
                        T* kv = reinterpret_cast<T*>(P.kv_pool) +
                                (size_t)E.layer * P.n_pages * (size_t)(2 * P.Hkv * kPageTokens * hd) + M.kvoff[b] +
                                (size_t)(g * 2 + c) * (kPageTokens * hd) + e;
                        store_rows<T, RP>(kv, w);
                    }
                }
            }
            epi_sync();
            break;
        }
        case EPI_RESID: {
            // v: this thread's row (n0 + et) for 32 columns -> esm; then thread -> (column b,
            // 32 consecutive rows): x += v, act = x * w_norm (hi, lo), sum of squares
            // transposed: thread -> (column b, RP = W consecutive rows), 128 / RP threads per column
            constexpr int RP = W, NPART = 128 / W;
            const int col = et / NPART, part = et % NPART;
            const int r0 = n0 + part * RP;
            const bool ok = col < ncols && r0 < E.N;
            const int b = cb + col;
            // the residual and norm-weight loads do not depend on the exchange: issue them first
            // so their latency hides behind the exchange stores and barrier
            float xv[RP], wn[RP];
            if (ok) {
                const float4* xs = reinterpret_cast<const float4*>(P.x + (size_t)b * P.d + r0);
                const float4* ws = reinterpret_cast<const float4*>(E.norm_w + r0);
#pragma unroll
                for (int q = 0; q < RP / 4; ++q) {
                    const float4 a = xs[q], w4 = __ldg(ws + q);
                    xv[4 * q] = a.x; xv[4 * q + 1] = a.y; xv[4 * q + 2] = a.z; xv[4 * q + 3] = a.w;
                    wn[4 * q] = w4.x; wn[4 * q + 1] = w4.y; wn[4 * q + 2] = w4.z; wn[4 * q + 3] = w4.w;
                }
            }
#pragma unroll
            for (int i = 0; i < W; ++i) esm[et * kEsmLd + i] = v[i];
            epi_sync();
            {
                float ss = 0.f;
                if (ok) {
#pragma unroll
                    for (int r = 0; r < RP; ++r) {
                        xv[r] += esm[(part * RP + r) * kEsmLd + col];
                        ss += xv[r] * xv[r];
                    }
                    float4* xd = reinterpret_cast<float4*>(P.x + (size_t)b * P.d + r0);
#pragma unroll
                    for (int q = 0; q < RP / 4; ++q) xd[q] = make_float4(xv[4 * q], xv[4 * q + 1], xv[4 * q + 2], xv[4 * q + 3]);
#pragma unroll
                    for (int r = 0; r < RP; ++r) wn[r] *= xv[r];
                    store_act_rows<T, RP>(reinterpret_cast<T*>(P.act) + (size_t)b * P.act_ld + r0, (size_t)P.act_plane, wn);
                }
                // the NPART threads of a column are consecutive lanes of one warp; the partial
                // sums over the 128-row block combine in a fixed order
#pragma unroll
                for (int o = 1; o < NPART; o <<= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
                if (ok && part == 0) P.ssq[(size_t)(n0 / 128) * P.Bmax + b] = ss;
            }
            epi_sync();
            break;
        }
        case EPI_SWIGLU: {
            // sub-tile rows 0..63: gate rows j0..j0+63; rows 64..127: up rows j0..j0+63
#pragma unroll
            for (int i = 0; i < W; ++i) esm[et * kEsmLd + i] = v[i] * s_scale[cb + i];
            epi_sync();
            {
                const int col = et >> 2, part = et & 3;   // part -> 16 consecutive j
                const int j0 = (n0 / 128) * 64 + part * 16;
                if (col < ncols && j0 < P.dff) {
                    float a[16];
#pragma unroll
                    for (int r = 0; r < 16; ++r) {
                        const float g = esm[(part * 16 + r) * kEsmLd + col];
                        const float u = esm[(64 + part * 16 + r) * kEsmLd + col];
                        a[r] = __fdividef(g, 1.f + __expf(-g)) * u;  // silu(g) u; 1 + e^-g >= 1
                    }
                    store_act_row16<T>(reinterpret_cast<T*>(P.h) + (size_t)(cb + col) * P.act_ld + j0,
                                       (size_t)P.act_plane, a);
                }
            }
            epi_sync();
            break;
        }
        case EPI_STORE: {
#pragma unroll
            for (int i = 0; i < 32; ++i)
                if (n < E.N && i < ncols) E.store_out[(size_t)(cb + i) * E.N + n] = v[i];
            break;
        }
        case EPI_LMHEAD: {
            const bool valid = n < P.V;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                float lg = v[i] * s_scale[cb + i];
                if (P.dbg_logits && valid && i < ncols) P.dbg_logits[(size_t)(cb + i) * P.V + n] = lg;
                esm[et * kEsmLd + i] = valid ? lg : -INFINITY;
            }
            epi_sync();
            // warp-level tile argmax: warp w takes columns w, w+4, ...; each lane folds 4 of
            // the tile's 128 rows (conflict-free: row stride 33 words), then a 5-step shuffle
            // max over the 64-bit (value, ~index) keys; lane 0 folds the tile's best into the
            // column's global key (atomicMax keeps the largest value, lowest index on ties)
            {
                const int w = et >> 5, ln = et & 31;
                for (int c = w; c < ncols; c += kEpiThreads / 32) {
                    unsigned long long best = 0;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int r = ln + 32 * i;
                        const unsigned long long k = argmax_key(esm[r * kEsmLd + c], (uint32_t)(n0 + r));
                        best = k > best ? k : best;
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
                        best = t > best ? t : best;
                    }
                    if (ln == 0) atomicMax(&P.am_keys[cb + c], best);
                }
            }
            epi_sync();
            break;
        }
    }
}

// ------------------------------------------------------------------ K6: sample + scan + publish
struct ScanOut {
    uint32_t off[kMaxRecPerSlot], len[kMaxRecPerSlot], tok[kMaxRecPerSlot];
    uint16_t did[kMaxRecPerSlot], flags[kMaxRecPerSlot];
    int16_t tool[kMaxRecPerSlot];
    int n;
};

CVY_DEV void scan_emit(ScanOut& so, uint32_t off, uint32_t len, uint32_t tok, uint16_t did, uint16_t fl, int tool) {
    if (so.n < kMaxRecPerSlot) {
        so.off[so.n] = off;
        so.len[so.n] = len;
        so.tok[so.n] = tok;
        so.did[so.n] = did;
        so.flags[so.n] = fl;
        so.tool[so.n] = (int16_t)tool;
        so.n++;
    }
}

// One byte through the JSON automaton (R10-R11): returns 0 for a ',' at depth 1 (member
// parsers only), 1 for the bracket returning depth to 0, -1 otherwise.
CVY_DEV int json_step(SlotDev& s, uint8_t b, bool member) {
    int hit = -1;
    if (s.in_str) {
        if (s.esc) s.esc = 0;
        else if (b == '\\') s.esc = 1;
        else if (b == '"') s.in_str = 0;
    } else if (s.depth == 0) {
        if (b == '{' || b == '[') s.depth = 1;
    } else {
        if (b == '"') s.in_str = 1;
        else if (b == '{' || b == '[') { if (s.depth < 127) s.depth += 1; }
        else if (b == '}' || b == ']') { s.depth -= 1; if (s.depth == 0) hit = 1; }
        else if (b == ',' && s.depth == 1 && member) hit = 0;
    }
    return hit;
}

// Region tool sets (NEXT-2, R24; a single FENCE or CALL tool is the set of one).
// Outside a region (region < 0): seg_start = start of the current line unit, win = the tools
// whose open marker ("```" TAG "\n" / "@call " TAG " ", packed in dpack / dlen[0]) this line no
// longer matches (all ones: a continuation of a cut line or the rest of a line after a CALL
// close -- never a marker); the marker that completes opens its tool's region (OPEN record).
// Inside a FENCE region: line units, esc = 2 not the close marker "```\n", 4 continuation;
// inside a CALL region: the JSON_MEMBER automaton, its closing bracket ends the region.
CVY_DEV void scan_byte_set(SlotDev& s, const ToolDev* tools, uint8_t b, uint32_t tok_idx, ScanOut& so) {
    s.stream_len += 1;
    const uint32_t p = s.stream_len;
    const uint32_t since = p - s.seg_start;
    if (s.region < 0) {
        const uint32_t k = since - 1;  // index of this byte in the line
        int opened = -1;
        uint64_t cand = s.tool_set & ~s.win;
        while (cand) {
            const int i = __ffsll((long long)cand) - 1;
            cand &= cand - 1;
            const ToolDev& t = tools[i];
            const uint32_t mlen = (uint32_t)t.dlen[0];
            if (k >= mlen || b != (uint8_t)(t.dpack[k >> 3] >> (8 * (k & 7)))) {
                s.win |= 1ull << i;
                continue;
            }
            if (since == mlen && opened < 0) opened = i;  // lowest tool id first
        }
        if (opened >= 0) {
            scan_emit(so, s.seg_start, since, tok_idx, 0, CVY_SEG_OPEN, opened);
            s.seg_start = p;
            s.region = opened;
            s.win = 0;
            s.depth = s.in_str = s.esc = 0;
        } else if (b == '\n') {
            s.seg_start = p;
            s.win = 0;
        } else if ((int)since == s.set_max_seg) {
            s.seg_start = p;
            s.win = ~0ull;
        }
        return;
    }
    const ToolDev& t = tools[s.region];
    if (t.kind == CVY_PARSER_FENCE) {
        const uint32_t k = since - 1;
        if (k >= 4 || b != (k < 3 ? (uint8_t)'`' : (uint8_t)'\n')) s.esc |= 2;
        if (b == '\n') {
            if (!(s.esc & 6) && since == 4) {
                scan_emit(so, s.seg_start, since, tok_idx, 0, CVY_SEG_CLOSE, s.region);
                s.region = -1;
                s.win = 0;
            } else {
                scan_emit(so, s.seg_start, since, tok_idx, 0, 0, s.region);
            }
            s.seg_start = p;
            s.esc = 0;
        } else if ((int)since == t.max_seg) {
            scan_emit(so, s.seg_start, since, tok_idx, (uint16_t)CVY_DELIM_NONE, CVY_SEG_OVERFLOW, s.region);
            s.seg_start = p;
            s.esc = 4;
        }
        return;
    }
    const int hit = json_step(s, b, true);
    if (hit == 1) {
        scan_emit(so, s.seg_start, since, tok_idx, 1, CVY_SEG_CLOSE, s.region);
        s.seg_start = p;
        s.region = -1;
        s.win = ~0ull;  // the rest of this line is not at a line start
    } else if (hit == 0) {
        scan_emit(so, s.seg_start, since, tok_idx, 0, 0, s.region);
        s.seg_start = p;
    } else if ((int)since == t.max_seg) {
        scan_emit(so, s.seg_start, since, tok_idx, (uint16_t)CVY_DELIM_NONE, CVY_SEG_OVERFLOW, s.region);
        s.seg_start = p;
    }
}

// Feed one byte of the round stream through the slot's trigger scanner (R5-R11).
CVY_DEV void scan_byte(SlotDev& s, const ToolDev& t, uint8_t b, uint32_t tok_idx, ScanOut& so) {
    s.stream_len += 1;
    const uint32_t p = s.stream_len;
    const uint32_t since = p - s.seg_start;
    int hit = -1;
    if (t.kind == CVY_PARSER_PLAN) {
        // R23: per-line DFA over  #E<digits> = <Name>[<args>]\n  in depth (0 = line start,
        // 9 = last byte ']', 10 = dead: mismatch or continuation of a max_seg cut)
        int st = s.depth;
        if (b == '\n') {
            if (st == 9) scan_emit(so, s.seg_start, since, tok_idx, 0, 0, s.tool);
            s.seg_start = p;
            st = 0;
        } else {
            const bool dig = b >= '0' && b <= '9';
            const bool nam = dig || (b >= 'A' && b <= 'Z') || (b >= 'a' && b <= 'z') || b == '_';
            switch (st) {
                case 0: st = b == '#' ? 1 : 10; break;
                case 1: st = b == 'E' ? 2 : 10; break;
                case 2: st = dig ? 3 : 10; break;
                case 3: st = dig ? 3 : (b == ' ' ? 4 : 10); break;
                case 4: st = b == '=' ? 5 : 10; break;
                case 5: st = b == ' ' ? 6 : 10; break;
                case 6: st = nam ? 7 : 10; break;
                case 7: st = nam ? 7 : (b == '[' ? 8 : 10); break;
                case 8: case 9: st = b == ']' ? 9 : 8; break;
                default: break;
            }
            if ((int)since == t.max_seg) {
                s.seg_start = p;
                st = 10;
            }
        }
        s.depth = st;
        return;
    }
    if (t.kind == CVY_PARSER_LITERAL) {
        s.win = (s.win << 8) | b;
        const uint32_t avail = since < 8 ? since : 8;
        for (int i = 0; i < t.n_delims; ++i) {
            if ((uint32_t)t.dlen[i] <= avail && (s.win & t.dmask[i]) == t.dpack[i]) {
                hit = i;
                break;
            }
        }
    } else {
        hit = json_step(s, b, t.kind != CVY_PARSER_JSON_OBJECT);
    }
    if (hit >= 0) {
        scan_emit(so, s.seg_start, since, tok_idx, (uint16_t)hit, 0, s.tool);
        s.seg_start = p;
        s.win = 0;
    } else if ((int)since == t.max_seg) {
        scan_emit(so, s.seg_start, since, tok_idx, (uint16_t)CVY_DELIM_NONE, CVY_SEG_OVERFLOW, s.tool);
        s.seg_start = p;
        s.win = 0;
    }
}

// Run by the 128 epilogue threads of the CTA that completed the last LM-head tile.
CVY_DEV void sample_scan_publish(const StepParams& P, int et, int* sm_i) {
    // sm_i: >= 8 ints of shared scratch
    __threadfence();
    const uint64_t step = *P.step_ctr;
    unsigned long long tail = *P.ring_tail_dev;
    cvy_segment* ring = reinterpret_cast<cvy_segment*>(P.ring);
    uint32_t n_active = 0, n_gen = 0, n_fin = 0, n_seg = 0;
    const int lane = et & 31, warp = et >> 5;
    if (et == 0) sm_i[4] = sm_i[5] = sm_i[6] = 0;
    epi_sync();
    for (int base = 0; base < P.Bp; base += kEpiThreads) {
        const int b = base + et;
        ScanOut so;
        so.n = 0;
        SlotDev s;
        bool live = false;
        if (b < P.Bp) {
            s = P.slots[b];
            unsigned long long key = atomicExch(&P.am_keys[b], 0ULL);
            live = s.active != 0;
            if (live) {
                n_active++;
                const int y = (int)argmax_key_index(key);
                const ToolDev* tool = (s.tool >= 0 && !P.scan_off) ? &P.tools[s.tool] : nullptr;
                bool end = false;
                uint16_t fin_flags = CVY_SEG_FINAL;
                if (s.cancel) {
                    end = true;
                    fin_flags |= CVY_SEG_CANCELLED;
                    s.cancel = 0;
                } else {
                    s.pos += 1;
                    if (s.in_idx < s.in_len) {
                        s.cur_tok = P.in_buf[(size_t)b * P.input_cap + s.in_idx];
                        s.in_idx += 1;
                    } else {
                        const int g = (s.gen < s.force_len) ? P.force_buf[(size_t)b * P.forced_cap + s.gen] : y;
                        const uint32_t ti = (uint32_t)s.gen;
                        s.gen += 1;
                        n_gen++;
                        s.cur_tok = g;
                        if (ti < P.round_tokens) P.tok_log[(size_t)b * P.round_tokens + ti] = g;
                        if (tool) {
                            const int nb = P.vlen[g];
                            for (int k = 0; k < nb; ++k) {
                                const uint8_t byte = P.vtab[(size_t)g * kMaxTokenBytes + k];
                                if (s.stream_len < P.round_bytes) P.byte_log[(size_t)b * P.round_bytes + s.stream_len] = byte;
                                if (s.tool_set) scan_byte_set(s, P.tools, byte, ti, so);
                                else scan_byte(s, *tool, byte, ti, so);
                            }
                        }
                        end = (P.eos >= 0 && g == P.eos) || s.gen >= s.max_new ||
                              (s.force_len > 0 && s.gen >= s.force_len) || s.pos >= s.max_pos;
                    }
                }
                if (end) {
                    const uint32_t last = s.gen > 0 ? (uint32_t)(s.gen - 1) : CVY_NO_TOKEN;
                    scan_emit(so, s.seg_start, s.stream_len - s.seg_start, last, (uint16_t)CVY_DELIM_NONE, fin_flags,
                              (tool && s.tool_set) ? s.region : s.tool);
                    s.active = 0;
                    n_fin++;
                }
                SlotStatus st;
                st.round = s.round;
                st.gen = (uint32_t)s.gen;
                st.state = end ? ((fin_flags & CVY_SEG_CANCELLED) ? 2u : 1u) : 0u;
                st.last_step = (uint32_t)step;
                P.status[b] = st;
            }
        }
        // exclusive prefix sum of record counts over the 128 threads (slot order)
        int cnt = so.n;
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) sm_i[warp] = incl;
        epi_sync();
        int wbase = 0, total = 0;
        for (int w = 0; w < kEpiThreads / 32; ++w) {
            if (w < warp) wbase += sm_i[w];
            total += sm_i[w];
        }
        const unsigned long long first = tail + (unsigned long long)(wbase + incl - cnt);
        for (int r = 0; r < so.n; ++r) {
            cvy_segment rec;
            rec.req_id = s.req_id;
            rec.round = s.round;
            rec.seq = s.seq + r;
            rec.step = (uint32_t)step;
            rec.token_index = so.tok[r];
            rec.byte_offset = so.off[r];
            rec.byte_len = so.len[r];
            rec.delim_id = so.did[r];
            rec.flags = so.flags[r];
            rec.slot = (uint16_t)b;
            rec.tool = so.tool[r];
            ring[(first + r) & P.ring_mask] = rec;
        }
        if (live) {
            s.seq += so.n;
            P.slots[b] = s;
        }
        n_seg += so.n;
        tail += (unsigned long long)total;
        epi_sync();
    }
    // publish: records and bytes become visible to the host before the new tail
    __threadfence_system();
    {
        const uint32_t a = __reduce_add_sync(0xffffffffu, n_active);
        const uint32_t g = __reduce_add_sync(0xffffffffu, n_gen);
        const uint32_t f = __reduce_add_sync(0xffffffffu, n_fin);
        if (lane == 0) {
            atomicAdd(&sm_i[4], (int)a);
            atomicAdd(&sm_i[5], (int)g);
            atomicAdd(&sm_i[6], (int)f);
        }
    }
    epi_sync();
    const int tot_active = sm_i[4], tot_gen = sm_i[5], tot_fin = sm_i[6];
    (void)n_seg;
    if (et == 0) {
        const unsigned long long old_tail = *P.ring_tail_dev;
        *P.ring_tail_dev = tail;
        StepStats ss;
        ss.step = step;
        ss.n_active = (uint32_t)tot_active;
        ss.n_generated = (uint32_t)tot_gen;
        ss.n_segments = (uint32_t)(tail - old_tail);
        ss.n_finished = (uint32_t)tot_fin;
        P.stats[step & 15] = ss;
        fence_sc_sys();
        st_release_sys_u64(reinterpret_cast<uint64_t*>(P.ring_tail_host), tail);
        *P.step_ctr = step + 1;
        *P.lm_done = 0;
    }
}

}  // namespace cvy
