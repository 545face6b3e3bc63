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

CVY_DEV void epi_sync() { named_bar_sync(kEpiBar, kEpiThreads); }

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
            const SlotDev& s = P.slots[b];
            int pos = s.pos;
            long long off = -1;
            if (s.active && pos < s.max_pos) {
                const int page = P.page_table[(size_t)b * P.max_pages + pos / kPageTokens];
                off = (long long)((size_t)page * page_elems + (size_t)(pos % kPageTokens) * P.hd);
            }
            m.pos[b] = min(max(pos, 0), P.max_rope_pos - 1);
            m.kvoff[b] = off;
        }
    }
}

// One 32-column chunk of one 128-row sub-tile.  n0 = first global row of the sub-tile.
template <typename T, int KIND = -1>
CVY_DEV void epilogue_chunk(const StepParams& P, const EpiArgs& E, int n0, int cb, float* v, float* esm,
                            const EpiMeta& M, int et, int width = 32) {
    const float* s_scale = M.scale;
    const int n = n0 + et;
    const int ncols = min(width, P.Bp - cb);
    switch (KIND >= 0 ? KIND : E.kind) {
        case EPI_QKV: {
            const int hd = P.hd, half = hd >> 1;
            const int qk_rows = (P.H + P.Hkv) * hd;
            const int dim = n % hd;
            const int j = dim & (half - 1);
            const bool rot = n < qk_rows;
            // all global inputs first (RoPE cos/sin of every column), then compute, then store:
            // interleaving loads with stores would serialise them (possible aliasing)
            float2 cs[32];
#pragma unroll
            for (int i = 0; i < 32; ++i)
                cs[i] = (rot && i < ncols) ? __ldg(&P.rope[(size_t)M.pos[cb + i] * half + j]) : make_float2(1.f, 0.f);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] *= s_scale[cb + i];
#pragma unroll
            for (int i = 0; i < 32; ++i) esm[et * kEsmLd + i] = v[i];
            epi_sync();
            const int partner = et ^ half;
            float out[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const float pv = esm[partner * kEsmLd + i];
                out[i] = dim < half ? (v[i] * cs[i].x - pv * cs[i].y) : (v[i] * cs[i].x + pv * cs[i].y);
            }
            epi_sync();
            if (n < P.H * hd) {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (i < ncols) P.q[(size_t)(cb + i) * (P.H * hd) + n] = out[i];
            } else if (n < E.N) {
                const int c = n >= qk_rows ? 1 : 0;
                const int rel = n - P.H * hd - c * P.Hkv * hd;
                const int g = rel / hd, e = rel % hd;
                T* kv = reinterpret_cast<T*>(P.kv_pool) + (size_t)E.layer * P.n_pages * (size_t)(2 * P.Hkv * kPageTokens * hd) +
                        (size_t)(c * P.Hkv + g) * (kPageTokens * hd) + e;
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const long long off = (i < ncols) ? M.kvoff[cb + i] : -1;
                    if (off >= 0) kv[off] = DT<T>::from_f(out[i]);
                }
            }
            break;
        }
        case EPI_RESID: {
            T* act = reinterpret_cast<T*>(P.act);
            const bool valid = n < E.N;
            const float w = valid ? E.norm_w[n] : 0.f;
            float xv[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) xv[i] = (valid && i < ncols) ? P.x[(size_t)(cb + i) * P.d + n] : 0.f;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const float xn = xv[i] + v[i];
                xv[i] = xn;
                esm[et * kEsmLd + i] = (valid && i < ncols) ? xn * xn : 0.f;
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                if (valid && i < ncols) {
                    P.x[(size_t)(cb + i) * P.d + n] = xv[i];
                    DT<T>::store_act(act + (size_t)(cb + i) * P.act_ld + n, (size_t)P.act_plane, xv[i] * w);
                }
            }
            epi_sync();
            if (et < 32 && et < ncols) {
                float acc = 0.f;
                for (int r = 0; r < 128; ++r) acc += esm[r * kEsmLd + et];
                if (n0 < E.N) P.ssq[(size_t)(n0 / 128) * P.Bmax + cb + et] = acc;
            }
            epi_sync();
            break;
        }
        case EPI_SWIGLU: {
            // sub-tile rows 0..63: gate rows j0..j0+63; rows 64..127: up rows j0..j0+63
#pragma unroll
            for (int i = 0; i < 32; ++i) esm[et * kEsmLd + i] = v[i] * s_scale[cb + i];
            epi_sync();
            if (et < 64) {
                T* hb = reinterpret_cast<T*>(P.h);
                const int j = (n0 / 128) * 64 + et;
                if (j < P.dff) {
                    for (int i = 0; i < ncols; ++i) {
                        float g = esm[et * kEsmLd + i];
                        float u = esm[(et + 64) * kEsmLd + i];
                        float a = g / (1.f + __expf(-g)) * u;
                        DT<T>::store_act(hb + (size_t)(cb + i) * P.act_ld + j, (size_t)P.act_plane, a);
                    }
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
            if (et < ncols) {
                uint64_t best = 0;
                for (int r = 0; r < 128; ++r) {
                    uint64_t k = argmax_key(esm[r * kEsmLd + et], (uint32_t)(n0 + r));
                    best = k > best ? k : best;
                }
                atomicMax(&P.am_keys[cb + et], (unsigned long long)best);
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
    int n;
};

CVY_DEV void scan_emit(ScanOut& so, uint32_t off, uint32_t len, uint32_t tok, uint16_t did, uint16_t fl) {
    if (so.n < kMaxRecPerSlot) {
        so.off[so.n] = off;
        so.len[so.n] = len;
        so.tok[so.n] = tok;
        so.did[so.n] = did;
        so.flags[so.n] = fl;
        so.n++;
    }
}

// Feed one byte of the round stream through the slot's trigger scanner (R5-R11).
CVY_DEV void scan_byte(SlotDev& s, const ToolDev& t, uint8_t b, uint32_t tok_idx, ScanOut& so) {
    s.stream_len += 1;
    const uint32_t p = s.stream_len;
    const uint32_t since = p - s.seg_start;
    int hit = -1;
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
            else if (b == ',' && s.depth == 1 && t.kind == CVY_PARSER_JSON_MEMBER) hit = 0;
        }
    }
    if (hit >= 0) {
        scan_emit(so, s.seg_start, since, tok_idx, (uint16_t)hit, 0);
        s.seg_start = p;
        s.win = 0;
    } else if ((int)since == t.max_seg) {
        scan_emit(so, s.seg_start, since, tok_idx, (uint16_t)CVY_DELIM_NONE, CVY_SEG_OVERFLOW);
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
                                scan_byte(s, *tool, byte, ti, so);
                            }
                        }
                        end = (P.eos >= 0 && g == P.eos) || s.gen >= s.max_new ||
                              (s.force_len > 0 && s.gen >= s.force_len) || s.pos >= s.max_pos;
                    }
                }
                if (end) {
                    const uint32_t last = s.gen > 0 ? (uint32_t)(s.gen - 1) : CVY_NO_TOKEN;
                    scan_emit(so, s.seg_start, s.stream_len - s.seg_start, last, (uint16_t)CVY_DELIM_NONE, fin_flags);
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
            rec.slot = (uint32_t)b;
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
