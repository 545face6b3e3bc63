// attention_tc.cuh -- paged-KV GQA decode attention for bf16 KV, head_dim 64/128, G <= 4.
//
// One CTA per (kv head g, slot b, split) of the keys [0, pos_b].  A producer warp streams
// the split's KV pages HBM -> shared memory with TMA (2D tensor map over the pool, box =
// 16 tokens x 64 dims, 128B swizzle), 4 pages (64 keys) per pipeline stage, 3 stages.  Four
// consumer warps each take one page of a stage and run it on the tensor cores with
// mma.sync.m16n8k16 (bf16 in, fp32 accumulate):
//   S^T[16 keys][8] = K_page[16][hd] . [q_hi | q_lo]^T   (columns 0-3: q_hi of the G heads,
//                                                        4-7: q_lo -- exact fp32 q, no waste)
//   O^T[hd][8]     += V_page^T[hd][16] . [p_hi | p_lo]^T (probabilities split the same way)
// with an online softmax per warp (exp2 domain) and a cross-warp merge at the end; each KV
// byte is read from HBM once and reused by the G query heads.
#pragma once
#include "common.cuh"
#include "step_params.h"

namespace cvy {

constexpr int kAtcWarps = 4;                 // consumer warps
constexpr int kAtcThreads = (kAtcWarps + 1) * 32;
constexpr int kAtcStages = 3;  // default pipeline depth (template parameter STAGES)
constexpr int kAtcPagesPerStage = 4;
constexpr int kAtcPageBytes = 16 * 128 * 2;  // one (page, K or V) block at hd = 128

CVY_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
CVY_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
CVY_DEV void mma_bf16_16816(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
CVY_DEV uint32_t pack_bf16(float lo_elem, float hi_elem) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo_elem, hi_elem);  // .x = first (lower address)
    return *reinterpret_cast<uint32_t*>(&v);
}
// byte offset of 16-B chunk `c` (0..7) of row `r` in a 16 x 128 B box written by TMA with
// 128B swizzle
CVY_DEV uint32_t sw128(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

// PPS = pages per pipeline stage: 4 (each consumer warp takes one page of every stage) or 2
// (warps 0-1 take the even stages, warps 2-3 the odd ones: half the shared memory per CTA, so
// twice as many CTAs fit on an SM -- one wave for the decode grid -- with the same bytes in flight).
template <int HD, int STAGES = kAtcStages, int PPS = kAtcPagesPerStage>
__global__ void __launch_bounds__(kAtcThreads) attention_tc_kernel(const __grid_constant__ CUtensorMap tmKV,
                                                                   const __grid_constant__ StepParams P, int layer) {
    static_assert(HD == 64 || HD == 128, "head_dim");
    static_assert(PPS == 4 || PPS == 2, "pages per stage");
    // PPS == 2: stage t belongs to warp pair t & 1; an even ring makes every slot belong to one
    // pair, so a pair's parity wait is never more than one phase ahead of the slot's barrier
    static_assert(PPS == 4 || STAGES % 2 == 0, "PPS 2 needs an even number of stages");
    constexpr int HALVES = HD / 64;                      // 64-dim boxes per (page, K/V)
    constexpr int BLK = 16 * HD * 2;                     // bytes of one (page, K/V) block
    constexpr int STAGE = PPS * 2 * BLK;                 // K and V of PPS pages
    constexpr int KSTEPS = HD / 16;
    extern __shared__ __align__(1024) uint8_t asm_raw[];
    uint8_t* sm = asm_raw + ((1024u - (smem_u32(asm_raw) & 1023u)) & 1023u);  // keeps the shared state space
    uint8_t* stages = sm;
    uint16_t* pbuf = reinterpret_cast<uint16_t*>(sm + STAGES * STAGE);  // [warp][8][16] bf16
    float* comb = reinterpret_cast<float*>(pbuf + kAtcWarps * 8 * 16);      // [warp][4 m, 4 l, 4*HD O]
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(comb + kAtcWarps * (8 + 4 * HD));
    uint64_t* empty_bar = full_bar + STAGES;

    pdl_launch_dependents();
    const int g = blockIdx.x, b = blockIdx.y, split = blockIdx.z;
    const int G = P.H / P.Hkv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == kAtcWarps * 32) {
        tma_prefetch_desc(&tmKV);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], PPS);  // the PPS warps that consume the stage
        }
        fence_mbar_init();
    }
    __syncthreads();

    // The split's key range and pages depend only on the slot state and page table (complete
    // before this step's graph starts), so they are read before the grid-dependency wait.
    const int nkeys = row_nkeys(P, b);
    const int nsplit = P.attn_splits;
    const int per = (((nkeys + nsplit - 1) / nsplit) + 16 * PPS - 1) / (16 * PPS) * (16 * PPS);
    const int k_begin = min(split * per, nkeys), k_end = min(nkeys, k_begin + per);
    const int pg_begin = k_begin / 16;
    const int n_pages = (k_end > k_begin) ? (k_end + 15) / 16 - pg_begin : 0;
    const int n_tiles = (n_pages + PPS - 1) / PPS;
    const int32_t* pt = P.page_table + (size_t)row_slot_of(P, b) * P.max_pages;

    if (warp == kAtcWarps) {
        // ============ producer: TMA page blocks into the stage ring ============
        // Pages strictly below the one holding this step's new key (written by the QKV
        // epilogue) were written by earlier steps: the first stages made only of such pages are
        // issued BEFORE griddepcontrol.wait, so their HBM reads overlap the previous kernel's
        // tail (decode rows only; a prefill pass writes several keys per slot).  The page ids
        // are read 32 at a time by the whole warp (no dependent load per TMA issue).
        const int safe_pages = (P.row_slot || !P.attn_early) ? 0 : max(0, (nkeys - 1) / 16 - pg_begin);
        const uint64_t pol = policy_evict_first();
        int chunk_base = -32, my_page = 0;
        auto page_of = [&](int i) {  // page id of split page i (warp-uniform i, increasing)
            if (i >= chunk_base + 32) {
                chunk_base = i & ~31;
                const int j = chunk_base + lane;
                my_page = j < n_pages ? pt[pg_begin + j] : 0;
            }
            return __shfl_sync(0xffffffffu, my_page, i & 31);
        };
        auto issue = [&](int t) {
            const int st = t % STAGES;
            const uint32_t ph = (uint32_t)(t / STAGES) & 1u;
            mbar_wait(&empty_bar[st], ph ^ 1u);
            const int np = min(PPS, n_pages - t * PPS);
            if (lane == 0) mbar_arrive_expect_tx(&full_bar[st], (uint32_t)(np * 2 * BLK));
            for (int p = 0; p < np; ++p) {
                const int page = page_of(t * PPS + p);
                if (lane == 0) {
                    // the (page, kv-head) block: K rows 0-15 then V rows 16-31, contiguous in the
                    // pool ([L][pages][Hkv][K/V][16][hd]); one box lands as [half][32 rows][64]
                    const int row0 = ((layer * P.n_pages + page) * P.Hkv + g) * 32;
                    uint8_t* dst = stages + (size_t)st * STAGE + (size_t)(p * 2) * BLK;
                    if (HALVES == 2 && P.kv_tma3d) {
                        tma_load_3d(dst, &tmKV, &full_bar[st], 0, row0, 0, pol);
                    } else {
                        for (int h = 0; h < HALVES; ++h)
                            tma_load_2d(dst + h * 4096, &tmKV, &full_bar[st], h * 64, row0, pol);
                    }
                }
            }
        };
        int t = 0;
        for (; t < n_tiles && t < STAGES && (t + 1) * PPS <= safe_pages; ++t) issue(t);
        pdl_wait();
        for (; t < n_tiles; ++t) issue(t);
        return;
    }
    pdl_wait();
    if (threadIdx.x == 0) span_begin(P.spans, P.span_base + layer * 8 + 2);

    // ============ consumers ============
    const int grp = lane >> 2, tig = lane & 3;
    // B fragments of [q_hi | q_lo]^T: column n = grp (n < 4: hi of head n, else lo of head n-4)
    uint32_t qb[KSTEPS][2];
    {
        const int n = grp, head = n & 3;
        const bool valid = head < G;
        const float qs = rsqrtf((float)HD) * 1.4426950408889634f;
        const float* qrow = P.q + (size_t)b * (P.H * HD) + (size_t)(g * G + (valid ? head : 0)) * HD;
#pragma unroll
        for (int ks = 0; ks < KSTEPS; ++ks) {
            float v[4];
            const int d0 = ks * 16 + tig * 2;
            const float2 qa = *reinterpret_cast<const float2*>(qrow + d0);      // 8-byte aligned (d0 even)
            const float2 qc = *reinterpret_cast<const float2*>(qrow + d0 + 8);
            v[0] = qa.x;
            v[1] = qa.y;
            v[2] = qc.x;
            v[3] = qc.y;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                float x = valid ? v[u] * qs : 0.f;
                float hi = __bfloat162float(__float2bfloat16_rn(x));
                v[u] = (n < 4) ? hi : (x - hi);
            }
            qb[ks][0] = pack_bf16(v[0], v[1]);
            qb[ks][1] = pack_bf16(v[2], v[3]);
        }
    }
    // per-lane softmax state for heads h0, h0+1 (h0 = 2*(tig&1)), O^T accumulators
    const int h0 = 2 * (tig & 1);
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
    float o[KSTEPS][4];
#pragma unroll
    for (int i = 0; i < KSTEPS; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    uint16_t* pw = pbuf + warp * 128;
    const uint32_t pw_addr = smem_u32(pw);

    for (int t = 0; t < n_tiles; ++t) {
        if (PPS == 2 && (t & 1) != (warp >> 1)) continue;  // the other warp pair's stage
        const int st = t % STAGES;
        const uint32_t ph = (uint32_t)(t / STAGES) & 1u;
        const int wp = PPS == 4 ? warp : (warp & 1);    // this warp's page within the stage
        const int pidx = t * PPS + wp;                  // this warp's page in the split
        // every consumer of the stage waits for its data, even one with no page in it (the last
        // stage of an odd page count): its empty-barrier arrival must not count toward the
        // slot's PREVIOUS phase while the other warp is still reading that phase's pages
        mbar_wait(&full_bar[st], ph);
        if (pidx < n_pages) {
            const uint32_t kbase = smem_u32(stages + (size_t)st * STAGE + (size_t)(wp * 2) * BLK);
            const uint32_t vbase = kbase + 2048;  // [half][K 16 rows | V 16 rows][64]: halves 4 KB apart
            // ---- S^T = K . [q_hi|q_lo]^T
            float s[2][4];  // [key block of 8 cols? no: one n8 block]; s[0] keys grp / grp+8
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int ks = 0; ks < KSTEPS; ++ks) {
                const int r = (lane & 7) + ((lane >> 3) & 1) * 8;    // key row
                const int dchunk = ks * 2 + (lane >> 4);             // 16-B chunk of dims
                const uint32_t addr = kbase + (dchunk >> 3) * 4096 + sw128(r, dchunk & 7);
                uint32_t a0, a1, a2, a3;
                ldsm_x4(addr, a0, a1, a2, a3);
                mma_bf16_16816(acc, a0, a1, a2, a3, qb[ks][0], qb[ks][1]);
            }
            // acc: (key grp, cols 2tig, 2tig+1), (key grp+8, same cols); add hi + lo halves
            s[0][0] = acc[0] + __shfl_xor_sync(0xffffffffu, acc[0], 2);
            s[0][1] = acc[1] + __shfl_xor_sync(0xffffffffu, acc[1], 2);
            s[1][0] = acc[2] + __shfl_xor_sync(0xffffffffu, acc[2], 2);
            s[1][1] = acc[3] + __shfl_xor_sync(0xffffffffu, acc[3], 2);
            // mask keys beyond the split end and heads beyond G
            const int key0 = (pg_begin + pidx) * 16 + grp;
            const bool k0ok = key0 < k_end, k1ok = key0 + 8 < k_end;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                if (!k0ok || h0 + j >= G) s[0][j] = -INFINITY;
                if (!k1ok || h0 + j >= G) s[1][j] = -INFINITY;
            }
            // ---- online softmax over this page's 16 keys (reduce over lanes with equal tig)
            float p[2][2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                float mx = fmaxf(s[0][j], s[1][j]);
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
                const float mnew = fmaxf(m_run[j], mx);
                const float alpha = (mnew == -INFINITY) ? 1.f : exp2f(m_run[j] - mnew);
                p[0][j] = (mnew == -INFINITY) ? 0.f : exp2f(s[0][j] - mnew);
                p[1][j] = (mnew == -INFINITY) ? 0.f : exp2f(s[1][j] - mnew);
                float ps = p[0][j] + p[1][j];
                ps += __shfl_xor_sync(0xffffffffu, ps, 4);
                ps += __shfl_xor_sync(0xffffffffu, ps, 8);
                ps += __shfl_xor_sync(0xffffffffu, ps, 16);
                l_run[j] = l_run[j] * alpha + ps;
                m_run[j] = mnew;
#pragma unroll
                for (int i = 0; i < KSTEPS; ++i) {
                    o[i][j] *= alpha;
                    o[i][2 + j] *= alpha;
                }
            }
            // ---- P^T -> smem as [col n][key]: n < 4 hi, n >= 4 lo (lanes tig<2 write hi, >=2 lo)
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 2; ++j) {
#pragma unroll
                for (int kk = 0; kk < 2; ++kk) {
                    const float x = p[kk][j];
                    const __nv_bfloat16 hi = __float2bfloat16_rn(x);
                    const __nv_bfloat16 val = (tig < 2) ? hi : __float2bfloat16_rn(x - __bfloat162float(hi));
                    const int n = (tig < 2 ? 0 : 4) + h0 + j;
                    pw[n * 16 + grp + kk * 8] = *reinterpret_cast<const uint16_t*>(&val);
                }
            }
            __syncwarp();
            uint32_t pb0, pb1;
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(pb0) : "r"(pw_addr + (uint32_t)((grp * 16 + tig * 2) * 2)));
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(pb1) : "r"(pw_addr + (uint32_t)((grp * 16 + tig * 2 + 8) * 2)));
            // ---- O^T += V^T . [p_hi|p_lo]^T, one m16 block of dims per MMA
#pragma unroll
            for (int i = 0; i < KSTEPS; ++i) {
                const int mtx = lane >> 3, r = lane & 7;
                const int key = r + (mtx >> 1) * 8;
                const int dchunk = i * 2 + (mtx & 1);
                const uint32_t addr = vbase + (dchunk >> 3) * 4096 + sw128(key, dchunk & 7);
                uint32_t a0, a1, a2, a3;
                ldsm_x4_t(addr, a0, a1, a2, a3);
                mma_bf16_16816(o[i], a0, a1, a2, a3, pb0, pb1);
            }
        }
        __syncwarp();
        if (lane == 0 && t < n_tiles) mbar_arrive(&empty_bar[st]);
    }
    // O^T fragment: (dim 16i + grp, cols 2tig, 2tig+1), (dim + 8, same cols); hi + lo halves
#pragma unroll
    for (int i = 0; i < KSTEPS; ++i)
#pragma unroll
        for (int u = 0; u < 4; ++u) o[i][u] += __shfl_xor_sync(0xffffffffu, o[i][u], 2);
    // cross-warp merge through shared memory
    float* cw = comb + warp * (8 + 4 * HD);
    if (lane < 4) {
        // lanes 0..3 hold heads h0(tig), h0+1: tig 0 -> heads 0,1; tig 1 -> heads 2,3
        if (tig < 2) {
            cw[h0] = m_run[0];
            cw[h0 + 1] = m_run[1];
            cw[4 + h0] = l_run[0];
            cw[4 + h0 + 1] = l_run[1];
        }
    }
    if (tig < 2) {
#pragma unroll
        for (int i = 0; i < KSTEPS; ++i) {
            cw[8 + (h0 + 0) * HD + 16 * i + grp] = o[i][0];
            cw[8 + (h0 + 1) * HD + 16 * i + grp] = o[i][1];
            cw[8 + (h0 + 0) * HD + 16 * i + grp + 8] = o[i][2];
            cw[8 + (h0 + 1) * HD + 16 * i + grp + 8] = o[i][3];
        }
    }
    named_bar_sync(2, kAtcWarps * 32);
    const int tid = threadIdx.x;
    for (int idx = tid; idx < G * HD; idx += kAtcWarps * 32) {
        const int j = idx / HD, e = idx % HD;
        float mstar = -INFINITY;
        for (int w = 0; w < kAtcWarps; ++w) mstar = fmaxf(mstar, comb[w * (8 + 4 * HD) + j]);
        float num = 0.f, den = 0.f;
        if (mstar != -INFINITY) {
            for (int w = 0; w < kAtcWarps; ++w) {
                const float* c = comb + w * (8 + 4 * HD);
                if (c[j] == -INFINITY) continue;
                const float sc = exp2f(c[j] - mstar);
                num += sc * c[8 + j * HD + e];
                den += sc * c[4 + j];
            }
        }
        if (nsplit == 1) {
            __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(P.o) + (size_t)b * P.act_ld + (size_t)g * G * HD;
            DT<__nv_bfloat16>::store_act(ob + idx, (size_t)P.act_plane, den > 0.f ? num / den : 0.f);
        } else {
            float* part = P.attn_part + (((size_t)b * P.Hkv + g) * nsplit + split) * (size_t)(G * (HD + 2));
            part[idx] = num;
            if (e == 0) {
                part[G * HD + j] = mstar;
                part[G * HD + G + j] = den;
            }
        }
    }
    if (threadIdx.x == 0) span_end(P.spans, kSpanSlots, P.span_base + layer * 8 + 2);
}

}  // namespace cvy
