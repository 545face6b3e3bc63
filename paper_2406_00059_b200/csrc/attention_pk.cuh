// attention_pk.cuh -- persistent paged GQA decode attention (opt-in CVY_ATTN_PERSISTENT=1;
// bf16 KV, head_dim 128, GQA groups <= 4, decode rows).  DESIGN.md §7.2.
//
// The per-(kv head, slot) kernel (attention_tc.cuh) is latency-bound at short contexts: ~3.5
// CTAs per SM, each with a 2-stage pipeline.  Here one CTA per SM walks a contiguous share of
// 8-page units ((slot, kv head, chunk), shares snapped to whole (slot, kv head) segments, so no
// segment is split and no merge pass exists) through a 3 x 64 KB TMA ring, continuous across
// segments.  8 consumer warps each take one page of every unit (mma.sync m16n8k16 with the
// q / p hi-lo split, online softmax); a segment's 8 partial softmax states are merged through
// shared memory when its last unit is done.  The producer warp reads a unit's page-table
// entries one per lane, a unit ahead.
//
// Measured: slower than attention_tc at the bench shape (1.37 vs 0.90 ms per
// step).  ncu: per-SM transfer rate while active equals attention_tc's (~24 KB/us), the
// whole-segment snap leaves ~29% SM imbalance, and the one-CTA-per-SM grid cannot start
// under the previous GEMM's tail (~4 us per layer).  A second consumer group (16 warps,
// alternate units) was slower still (1.77 ms): it halves the units in flight.
#pragma once
#include "layers_persistent.cuh"

namespace cvy {

constexpr int kApWarps = 8;                       // pages per unit = consumer warps per group
constexpr int kApGroups = 1;                      // consumer groups, alternating units (2 measured slower)
constexpr int kApConsumers = kApWarps * kApGroups;
constexpr uint32_t kApPage = 2u * 16u * 128u * 2u;  // K + V of one 16-token page at hd 128
constexpr uint32_t kApStage = kApWarps * kApPage;   // one unit
constexpr int kApMaxRows = 512;

__host__ __device__ constexpr uint32_t ap_smem_bytes(int stages) {
    return 1024u + (uint32_t)stages * kApStage + kApConsumers * 128u * 2u   // pbuf
           + kApWarps * (8u + 4u * 128u) * 4u                               // comb
           + (3u * kApMaxRows + 8u) * 4u                                     // tables
           + (uint32_t)stages * 16u + 16u;                                   // barriers
}

__global__ void __launch_bounds__((kApConsumers + 1) * 32, 1)
    attention_persistent_kernel(const __grid_constant__ CUtensorMap tmKV, const __grid_constant__ StepParams P,
                                int layer, int nstages) {
    constexpr int HD = 128;
    extern __shared__ __align__(1024) uint8_t ap_raw[];
    uint8_t* sm = ap_raw + ((1024u - (smem_u32(ap_raw) & 1023u)) & 1023u);  // keeps the shared state space
    uint8_t* ring = sm;
    uint16_t* pbuf = reinterpret_cast<uint16_t*>(ring + (size_t)nstages * kApStage);
    float* comb = reinterpret_cast<float*>(pbuf + kApConsumers * 128);
    int* nch = reinterpret_cast<int*>(comb + kApWarps * (8 + 4 * HD));
    int* pre = nch + kApMaxRows;        // [kApMaxRows + 1]
    int* nkeys = pre + kApMaxRows + 1;  // [kApMaxRows]
    uint8_t* bars = reinterpret_cast<uint8_t*>(nkeys + kApMaxRows);
    uint64_t* full = reinterpret_cast<uint64_t*>(bars + ((16u - (smem_u32(bars) & 15u)) & 15u));
    uint64_t* empty = full + nstages;

    pdl_launch_dependents();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int Bp = P.Bp, Hkv = P.Hkv, G = P.H / P.Hkv;
    for (int b = threadIdx.x; b < kApMaxRows; b += blockDim.x) {
        const int nk = b < Bp ? row_nkeys(P, b) : 0;
        nkeys[b] = nk;
        nch[b] = ((nk + 15) / 16 + kApWarps - 1) / kApWarps;
    }
    if (warp == kApConsumers && lane == 0) {
        tma_prefetch_desc(&tmKV);
        for (int s = 0; s < nstages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kApWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        // exclusive prefix of Hkv * nch over kApMaxRows slots (16 per lane)
        constexpr int PER = kApMaxRows / 32;
        int s = 0;
#pragma unroll
        for (int j = 0; j < PER; ++j) s += nch[lane * PER + j] * Hkv;
        int inc = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        int run = inc - s;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            pre[lane * PER + j] = run;
            run += nch[lane * PER + j] * Hkv;
        }
        if (lane == 31) pre[kApMaxRows] = inc;
    }
    __syncthreads();
    pdl_wait();  // q and this step's K, V rows come from the QKV GEMM
    const long long U = pre[kApMaxRows];
    // whole segments per CTA (the snapped even split; a CTA may get none)
    const long long u0 = pk_att_snap(pre, nch, Bp, U, blockIdx.x, gridDim.x);
    const long long u1 = pk_att_snap(pre, nch, Bp, U, blockIdx.x + 1, gridDim.x);

    if (warp == kApConsumers) {
        // ============ producer: one 8-page unit per ring stage ============
        // Lane pg < np owns page pg of the unit: the page-table reads go out in parallel (one
        // L2 round trip per unit, prefetched a unit ahead) and each lane issues its own TMAs.
        const uint64_t pol = policy_evict_first();
        int s = 0;
        uint32_t ph = 0;
        int b = 0, g = 0, chunk = 0, np = 0, page = 0;
        auto fetch = [&](long long u) {
            pk_att_decode(pre, nch, Bp, (int)u, b, g, chunk);
            np = min(kApWarps, (nkeys[b] + 15) / 16 - chunk * kApWarps);
            page = lane < np ? P.page_table[(size_t)row_slot_of(P, b) * P.max_pages + chunk * kApWarps + lane] : 0;
        };
        if (u0 < u1) fetch(u0);
        for (long long u = u0; u < u1; ++u) {
            const int cg = g, cnp = np, cpage = page;
            if (u + 1 < u1) fetch(u + 1);
            if (lane == 0) {
                mbar_wait(&empty[s], ph ^ 1u);
                mbar_arrive_expect_tx(&full[s], (uint32_t)cnp * kApPage);
            }
            __syncwarp();
            if (lane < cnp) {
                uint8_t* dst = ring + (size_t)s * kApStage + (size_t)lane * kApPage;
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int row0 = ((((layer * P.n_pages + cpage) * 2 + c) * Hkv) + cg) * 16;
                    tma_load_2d(dst + (size_t)c * 4096, &tmKV, &full[s], 0, row0, pol);
                    tma_load_2d(dst + (size_t)c * 4096 + 2048, &tmKV, &full[s], 64, row0, pol);
                }
            }
            if (++s == nstages) {
                s = 0;
                ph ^= 1u;
            }
        }
        return;
    }

    // ============ consumers: warp w takes page w of every unit ============
    const int tig = lane & 3, grp = lane >> 2;
    const int h0 = 2 * (tig & 1);
    const int tid = threadIdx.x;
    uint16_t* pw = pbuf + warp * 128;
    PkAttRun R;
    int s = 0;
    uint32_t ph = 0;
    for (long long u = u0; u < u1; ++u) {
        int b, g, chunk;
        pk_att_decode(pre, nch, Bp, (int)u, b, g, chunk);
        if (chunk == 0) pk_att_load_q(P, R, b, g, lane);  // segments start at chunk 0 (whole segments)
        const int nk = nkeys[b];
        const int pidx = chunk * kApWarps + warp;
        mbar_wait(&full[s], ph);
        if (pidx * 16 < nk) {
            const uint32_t kbase = smem_u32(ring + (size_t)s * kApStage + (size_t)warp * kApPage);
            pk_att_page(R, kbase, kbase + 4096, pw, pidx * 16, nk, G, lane);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == nstages) {
            s = 0;
            ph ^= 1u;
        }
        if (chunk == nch[b] - 1) {
            // segment complete: merge the 8 warps' softmax states, store o (hi, lo planes)
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int q = 0; q < 4; ++q) R.o[i][q] += __shfl_xor_sync(0xffffffffu, R.o[i][q], 2);
            float* cw = comb + warp * (8 + 4 * HD);
            if (lane < 2) {
                cw[h0] = R.m_run[0];
                cw[h0 + 1] = R.m_run[1];
                cw[4 + h0] = R.l_run[0];
                cw[4 + h0 + 1] = R.l_run[1];
            }
            if (tig < 2) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    cw[8 + (h0 + 0) * HD + 16 * i + grp] = R.o[i][0];
                    cw[8 + (h0 + 1) * HD + 16 * i + grp] = R.o[i][1];
                    cw[8 + (h0 + 0) * HD + 16 * i + grp + 8] = R.o[i][2];
                    cw[8 + (h0 + 1) * HD + 16 * i + grp + 8] = R.o[i][3];
                }
            }
            named_bar_sync(1, kApWarps * 32);
            __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(P.o) + (size_t)b * P.act_ld + (size_t)g * G * HD;
            for (int idx = tid; idx < G * HD; idx += kApWarps * 32) {
                const int j = idx / HD, e = idx % HD;
                float mstar = -INFINITY;
                for (int w = 0; w < kApWarps; ++w) mstar = fmaxf(mstar, comb[w * (8 + 4 * HD) + j]);
                float num = 0.f, den = 0.f;
                if (mstar != -INFINITY) {
                    for (int w = 0; w < kApWarps; ++w) {
                        const float* c = comb + w * (8 + 4 * HD);
                        if (c[j] == -INFINITY) continue;
                        const float sc = exp2f(c[j] - mstar);
                        num += sc * c[8 + j * HD + e];
                        den += sc * c[4 + j];
                    }
                }
                DT<__nv_bfloat16>::store_act(ob + idx, (size_t)P.act_plane, den > 0.f ? num / den : 0.f);
            }
            named_bar_sync(1, kApWarps * 32);  // comb is rewritten by the next segment
        }
    }
}

}  // namespace cvy
