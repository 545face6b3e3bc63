// layers_persistent.cuh -- all L decoder layers of one decode step in ONE persistent kernel
// (bf16, head_dim 128, GQA groups <= 4, padded batch Bp <= 128).  DESIGN.md §7 "Persistent
// layer kernel".
//
// Why: the step is HBM-bound (14.2 GB of weights + the KV cache per step).
// With one kernel per GEMM / attention, every kernel boundary leaves HBM idle while the last
// CTAs drain their epilogues and the next kernel ramps up (≈5 boundaries per layer, measured
// ≈55 us of ≈137 us per layer at B=64).  Here one CTA per SM runs the whole layer stack and
// the weight stream never stops: a dedicated producer warp walks this CTA's share of every
// projection of every layer in order and keeps a shared-memory ring (plus an L2 look-ahead)
// full, independent of data dependencies.  Only the activation / KV loads wait for the
// phase they depend on, through device-wide "phase done" counters.
//
// Per layer l, five phases p (same order as the paper's decode step):
//   p=0 QKV projection + RoPE + paged-KV append   (X = act, stream-K over (tile, k-block))
//   p=1 paged GQA decode attention                (units = (slot, kv head, 4-page chunk))
//   p=2 O projection + residual + next-norm input (X = o)
//   p=3 gate/up projection + SwiGLU               (X = act)
//   p=4 down projection + residual + next norm    (X = h)
// Phase p of layer l may read its inputs once done[l][p-1] (or done[l-1][4]) == gridDim.x:
// each CTA adds 1 after finishing all of its epilogue work of the phase.  Work of a phase is
// split evenly over the CTAs (stream-K for the GEMMs: a contiguous range of (tile, k-block)
// iterations per CTA; a contiguous range of attention units per CTA), so every SM streams the
// same number of weight / KV bytes.  Tiles (and attention (slot, head) segments) shared by
// several CTAs are combined by the last arriving contributor -- no CTA ever waits for another
// inside a phase; the only cross-CTA waits are the phase-done counters, which every CTA
// reaches (the grid is co-resident: one CTA per SM, cooperative launch).
//
// Warp roles (384 threads, 3 warpgroups; setmaxnreg moves registers from WG1 to WG0):
//   WG0 warps 0-3   GEMM epilogues (TMEM lane = tile row) and attention consumers (mma.sync)
//   WG1 warp 4      weight producer: TMA of W k-blocks into the W ring + L2 prefetch look-ahead
//       warp 5      MMA issuer (tcgen05.mma, one lane) and TMEM owner
//       warp 6      data producer: TMA of activation k-blocks (hi, lo planes) and KV pages into
//                   the D ring, each after its phase dependency
//       warp 7      idle
//   WG2 warps 8-11  attention consumers (the attention phase runs on 8 warps, one KV page each
//                   per 8-page unit: the mma.sync page loop is latency-bound)
#pragma once
#include "attention_tc.cuh"
#include "common.cuh"
#include "epilogue.cuh"
#include "gemm_sm100.cuh"
#include "step_params.h"

namespace cvy {

constexpr int kPkThreads = 384;   // 3 warpgroups (see the role table above)
constexpr int kPkAttWarps = 8;    // attention consumers: warps 0-3 and 8-11
constexpr uint32_t kAttBar = 4;   // named barrier of the 256 attention threads
constexpr uint32_t kWg2Bar = 5;   // named barrier of warpgroup 2
constexpr int kPkPhases = 5;
constexpr int kPkMaxBp = 128;
constexpr uint32_t kPkWStage = 128u * 128u;          // 128 weight rows x 64 bf16 (128B swizzle)
constexpr uint32_t kPkAttStage = 4u * 2u * 16u * 128u * 2u;  // 4 pages x (K, V) x 16 x 128 bf16
constexpr int kPkMaxCon = 6;  // later contributors of one stream-K tile reduced per batch (host checks)
constexpr int kPkTraceStride = 32;  // [0,5) data-producer phase start, [8,13) phase done,
                                      // [16,21) last accumulator received, [24,29) last MMA issued

struct PkGemm {
    int32_t N, K, tiles, kblocks;
};

struct PkParams {
    PkGemm g[4];         // per-layer geometry: QKV, O, gate/up, down
    int32_t w_stages;    // W ring depth (16 KB slots)
    int32_t x_stages;    // D ring depth
    uint32_t x_slot;     // D ring slot bytes = one activation k-block (hi + lo planes: 2*Bp*128);
                         // an attention unit (8 KV pages of 8 KB: one per attention warp) spans
                         // att_su consecutive slots
    int32_t att_ppslot;  // KV pages per D-ring slot (x_slot / 8 KB): 1, 2 or 4
    int32_t att_su;      // D-ring slots per attention unit (8 / att_ppslot)
    int32_t x_arrivals;  // arrivals that release a D-ring slot: att_ppslot (the attention warps
                         // sharing a slot, or as many tcgen05.commit for an activation slot)
    uint32_t tmem_cols;
    int32_t l2_pf;       // weight k-blocks prefetched into L2 ahead of the ring
    int32_t* done;       // [L][5] phase-done counters, zeroed before every launch
    int32_t* att_cnt;    // [Bmax][Hkv] arrival tickets of split attention segments (self-resetting)
    float* att_part;     // [grid][2][G*(hd+2)] partial (num, max, den) of split segments
    float* part;         // [2][grid][Bp/32][8][128][4] fp32: the partial tile of each CTA's first
                         // (shared) segment of a GEMM phase, buffer = GEMM index & 1
    uint32_t* pflag;     // [2][grid] tag of the partial last published by each CTA
    int32_t* err;        // first failing wait (diagnostics before the trap)
    unsigned long long* trace;  // [grid][kPkTraceStride] %globaltimer stamps of trace_layer, or null
    int32_t trace_layer;
    int32_t trace_phase;  // GEMM index (0..3) whose epilogue gets detailed stamps [5,6,7,13,14]
};

struct PkSmem {
    // offsets from the 1024-aligned base; host and device agree
    __host__ __device__ static constexpr uint32_t esm_bytes() { return 128u * kEsmLd * 4u; }
    __host__ __device__ static constexpr uint32_t pbuf_bytes() { return (uint32_t)kPkAttWarps * 8u * 16u * 2u; }
    __host__ __device__ static constexpr uint32_t meta_bytes() { return (uint32_t)kPkMaxBp * 16u; }
    __host__ __device__ static constexpr uint32_t table_bytes() { return (uint32_t)(3 * kPkMaxBp + 4) * 4u; }
    __host__ __device__ static constexpr uint32_t bar_bytes(int ws, int xs) { return (uint32_t)(2 * ws + 2 * xs + 6) * 8u + 64u; }
    __host__ __device__ static constexpr uint32_t total(int ws, int xs, uint32_t x_slot) {
        return 1024u + (uint32_t)ws * kPkWStage + (uint32_t)xs * x_slot + esm_bytes() + pbuf_bytes() + meta_bytes() +
               table_bytes() + bar_bytes(ws, xs);
    }
};

// ------------------------------------------------------------------ device-wide ordering
CVY_DEV int ld_acquire_gpu(const int32_t* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
CVY_DEV void red_release_gpu_add(int32_t* p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
CVY_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

#ifndef K_PK_BACKOFF_NS
#define K_PK_BACKOFF_NS 64
#endif
constexpr unsigned long long kPkTimeoutNs = 4000000000ull;  // a wait this long is a bug: trap

// A wait that exceeds kPkTimeoutNs records (site | progress << 12, CTA) in the host-mapped
// err[2 * role] (role = site >> 8, first recorder wins), keeps waiting another timeout so the
// other stuck roles record theirs too, then traps: the engine reports every stuck site.
CVY_DEV bool pk_fail(int32_t* err, int code, unsigned long long t0) {
    const int r = (code >> 8) & 7;
    if (atomicCAS(&err[2 * r], 0, code) == 0) err[2 * r + 1] = blockIdx.x;
    if (err[0] == 0) atomicCAS(&err[0], 0, code);
    err[16 + blockIdx.x * 8 + r] = code;  // per-CTA, per-role stuck site (diagnostics)
    __threadfence_system();
    if (gtimer() - t0 > 2 * kPkTimeoutNs) __trap();
    return true;
}
CVY_DEV void pk_wait_done(const int32_t* p, int target, int32_t* err, int code) {
    if (ld_acquire_gpu(p) >= target) return;
    const unsigned long long t0 = gtimer();
    while (ld_acquire_gpu(p) < target) {
        __nanosleep(64);
        if (gtimer() - t0 > kPkTimeoutNs) pk_fail(err, code, t0);
    }
}
CVY_DEV void pk_bar_wait(uint64_t* bar, uint32_t parity, int32_t* err, int code) {
    const uint32_t a = smem_u32(bar);
    if (mbar_try_wait(a, parity)) return;
    const unsigned long long t0 = gtimer();
    int n = 0;
    while (!mbar_try_wait(a, parity)) {
        // back off: spinning producer / MMA threads share issue slots with the consumer warps
        // of their SM sub-partition
        if (K_PK_BACKOFF_NS > 0) __nanosleep(K_PK_BACKOFF_NS);
        if (++n == 256) {
            n = 0;
            if (gtimer() - t0 > kPkTimeoutNs) {
                unsigned long long raw;
                asm volatile("ld.shared.b64 %0, [%1];" : "=l"(raw) : "r"(a));
                const int r = (code >> 8) & 7;
                err[16 + gridDim.x * 8 + blockIdx.x * 16 + 2 * r] = (int)(raw & 0xFFFFFFFFu);
                err[16 + gridDim.x * 8 + blockIdx.x * 16 + 2 * r + 1] = (int)(raw >> 32);
                pk_fail(err, code, t0);
            }
        }
    }
}

// 1D bulk copy global -> shared (async proxy), completion on an mbarrier (complete_tx)
CVY_DEV void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(smem_dst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
CVY_DEV void st_release_gpu_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
CVY_DEV uint32_t ld_acquire_gpu_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
CVY_DEV void pk_wait_tag(const uint32_t* p, uint32_t tag, int32_t* err, int code) {
    if (ld_acquire_gpu_u32(p) == tag) return;
    const unsigned long long t0 = gtimer();
    while (ld_acquire_gpu_u32(p) != tag) {
        __nanosleep(32);
        if (gtimer() - t0 > kPkTimeoutNs) pk_fail(err, code, t0);
    }
}

// contiguous share [a0, a1) of T work items for CTA c of G
CVY_DEV void pk_share(long long T, int c, int G, long long& a0, long long& a1) {
    a0 = (T * c) / G;
    a1 = (T * (c + 1)) / G;
}

// number of CTAs owning at least one item of [lo, hi) (CTAs with empty shares are skipped:
// a phase may have fewer items than CTAs)
CVY_DEV int pk_contributors(long long T, int G, long long lo, long long hi) {
    int n = 0;
    for (long long i = lo; i < hi;) {
        const int c = cta_of_iter(i, T, G);
        ++n;
        i = (T * (c + 1)) / G;
    }
    return n;
}

// attention unit u -> (slot b, kv head g, 8-page chunk); pre[b] = units before slot b
CVY_DEV void pk_att_decode(const int* pre, const int* nch, int Bp, int u, int& b, int& g, int& chunk) {
    int lo = 0, hi = Bp;  // pre[lo] <= u < pre[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (pre[mid] <= u) lo = mid;
        else hi = mid;
    }
    b = lo;
    const int rem = u - pre[b];
    g = rem / nch[b];
    chunk = rem - g * nch[b];
}

// Attention share of CTA c.  With at least as many (slot, kv head) segments as CTAs, the even
// split of the U units is snapped to the nearest segment boundary: every CTA then owns whole
// segments (imbalance <= half a segment) and no segment needs a cross-CTA merge.  Otherwise
// (few long segments) the exact even split is used and split segments are merged.
CVY_DEV long long pk_att_snap(const int* pre, const int* nch, int Bp, long long U, int c, int G) {
    if (c <= 0) return 0;
    if (c >= G) return U;
    const long long t = (U * c) / G;
    int lo = 0, hi = Bp;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (pre[mid] <= t) lo = mid;
        else hi = mid;
    }
    const int n = nch[lo];
    if (n == 0) return pre[lo];
    const int g = (int)((t - pre[lo] + n / 2) / n);
    return pre[lo] + (long long)g * n;
}
CVY_DEV void pk_att_range(const int* pre, const int* nch, int Bp, long long U, int nseg, int c, int G, long long& a0,
                          long long& a1) {
    if (nseg >= G) {
        a0 = pk_att_snap(pre, nch, Bp, U, c, G);
        a1 = pk_att_snap(pre, nch, Bp, U, c + 1, G);
    } else {
        pk_share(U, c, G, a0, a1);
    }
}

// GEMM phase index (0..3) of layer phase p (0, 2, 3, 4); X source plane set
CVY_DEV int pk_gp(int p) { return p == 0 ? 0 : p - 1; }

// ------------------------------------------------------------------ GEMM epilogue of one phase
template <int EPI>
CVY_DEV void pk_gemm_epilogue(const StepParams& P, const PkParams& K, const EpiArgs& E, int gp, EpiMeta& meta,
                              float* esm, int* flags, uint64_t* tfull, uint64_t* tempty, uint32_t tmem_base,
                              uint32_t& acnt, int et, int warp, unsigned long long* tr, uint32_t tag,
                              uint64_t* red_bar, uint32_t& red_ph, uint8_t* scratch) {
    const PkGemm& g = K.g[gp];
    const int Gc = gridDim.x;
    const long long T = (long long)g.tiles * g.kblocks;
    long long it, it1;
    pk_share(T, blockIdx.x, Gc, it, it1);
    const int Bp = P.Bp;
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const int buf = gp & 1;
    while (it < it1) {
        const int tile = (int)(it / g.kblocks);
        const long long tb = (long long)tile * g.kblocks, te = tb + g.kblocks;
        const long long seg_b = it;  // this CTA's segment of the tile: [seg_b, seg_e)
        it = min(it1, te);
        const long long seg_e = it;
        const int c_first = cta_of_iter(tb, T, Gc), c_last = cta_of_iter(te - 1, T, Gc);
        const int as = (int)(acnt & 1u);
        pk_bar_wait(&tfull[as], (acnt >> 1) & 1u, K.err, (0x100 + gp) | (int)(min(acnt, 0x7FFFFu) << 12));
        tc_fence_after();
        if (tr && et == 0) tr[16 + (gp == 0 ? 0 : gp + 1)] = gtimer();
        const uint32_t tacc = tmem_base + lane_off + (uint32_t)(as * 2 * Bp);
        const bool dt = tr && et == 0 && gp == K.trace_phase;
        if (dt) tr[15] = gtimer();  // accumulator of the segment received
        if (c_first == c_last) {
            for (int cb = 0; cb < Bp; cb += 32) {
                float v[32], w[32];
                tmem_ld32(tacc + (uint32_t)cb, v);
                tmem_ld32(tacc + (uint32_t)(Bp + cb), w);
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] += w[i];
                epilogue_chunk<__nv_bfloat16, EPI>(P, E, tile * 128, cb, v, esm, meta, et);
            }
            tc_fence_before();
            mbar_arrive(&tempty[as]);
        } else if (seg_b != tb) {
            // a later contributor: publish this partial (coalesced [chunk][q][row][4]) + tag
            float4* mine = reinterpret_cast<float4*>(K.part) + ((size_t)buf * Gc + blockIdx.x) * (size_t)Bp * 32;
            for (int cb = 0; cb < Bp; cb += 32) {
                float v[32], w[32];
                tmem_ld32(tacc + (uint32_t)cb, v);
                tmem_ld32(tacc + (uint32_t)(Bp + cb), w);
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    __stcg(mine + ((size_t)(cb / 32) * 8 + q) * 128 + et,
                           make_float4(v[4 * q] + w[4 * q], v[4 * q + 1] + w[4 * q + 1], v[4 * q + 2] + w[4 * q + 2],
                                       v[4 * q + 3] + w[4 * q + 3]));
            }
            tc_fence_before();
            mbar_arrive(&tempty[as]);
            __threadfence();
            epi_sync();
            if (et == 0) st_release_gpu_u32(K.pflag + (size_t)buf * Gc + blockIdx.x, tag);
        } else {
            // the tile's first CTA (reaches it last in its range): add the later contributors'
            // partials in CTA order -- deterministic -- and run the epilogue.  The partial chunks
            // (16 KB each) are bulk-copied into the data ring, idle here: the next phase's loads
            // wait for this phase's done counter, which this CTA has not bumped yet.
            // tags of every later contributor (one thread each, in parallel), then the proxy fence
            // that orders the bulk copies after them
            {
                int j = 0;
                for (long long i = seg_e; i < te; ++j) {
                    const int c = cta_of_iter(i, T, Gc);
                    if ((j & 127) == et) pk_wait_tag(K.pflag + (size_t)buf * Gc + c, tag, K.err, 0x140 + gp);
                    i = (T * (c + 1)) / Gc;
                }
            }
            fence_proxy_async_global();
            epi_sync();
            if (dt) tr[5] = gtimer();
            for (int cb = 0; cb < Bp; cb += 32) {
                float v[32], w[32];
                tmem_ld32(tacc + (uint32_t)cb, v);
                tmem_ld32(tacc + (uint32_t)(Bp + cb), w);
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] += w[i];
                if (cb + 32 >= Bp) {
                    tc_fence_before();
                    mbar_arrive(&tempty[as]);
                }
                for (long long i = seg_e; i < te;) {
                    // a batch of up to kPkMaxCon contributors' 16 KB chunks, CTA order
                    int con[kPkMaxCon];
                    int n = 0;
                    for (; i < te && n < kPkMaxCon; ++n) {
                        con[n] = cta_of_iter(i, T, Gc);
                        i = (T * (con[n] + 1)) / Gc;
                    }
                    if (et == 0) {
                        mbar_arrive_expect_tx(red_bar, (uint32_t)n * 16384u);
                        for (int j = 0; j < n; ++j)
                            bulk_g2s(scratch + (size_t)j * 16384,
                                     reinterpret_cast<const float4*>(K.part) + ((size_t)buf * Gc + con[j]) * (size_t)Bp * 32 +
                                         (size_t)(cb / 32) * 8 * 128,
                                     16384u, red_bar);
                    }
                    pk_bar_wait(red_bar, red_ph, K.err, 0x150 + gp);
                    red_ph ^= 1u;
                    if (dt) tr[cb == 0 ? 6 : 13] = gtimer();
                    for (int j = 0; j < n; ++j) {
                        const float4* src = reinterpret_cast<const float4*>(scratch + (size_t)j * 16384) + et;
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const float4 t4 = src[(size_t)q * 128];
                            v[4 * q] += t4.x;
                            v[4 * q + 1] += t4.y;
                            v[4 * q + 2] += t4.z;
                            v[4 * q + 3] += t4.w;
                        }
                    }
                    epi_sync();  // scratch is refilled by the next batch
                }
                epilogue_chunk<__nv_bfloat16, EPI>(P, E, tile * 128, cb, v, esm, meta, et);
                if (dt) tr[cb == 0 ? 7 : 14] = gtimer();
            }
        }
        ++acnt;
    }
}

// ------------------------------------------------------------------ attention phase (8 warps)
CVY_DEV void att_sync() { named_bar_sync(kAttBar, kPkAttWarps * 32); }
struct PkAttRun {
    float m_run[2], l_run[2];
    float o[8][4];
    uint32_t qb[8][2];
};

// cross-warp merge of one (slot, kv head) run; complete runs store o, split runs store a
// partial and the last arriving CTA of the segment combines all partials in CTA order
CVY_DEV void pk_att_finish(const StepParams& P, const PkParams& K, PkAttRun& R, float* comb, int* flags, int b, int g,
                           int seg_s, int seg_e, int run_s, int run_e, long long U, int et, int warp, int lane) {
    // et: attention thread index 0..255, warp: attention warp index 0..7
    constexpr int HD = 128, KSTEPS = 8;
    const int G = P.H / P.Hkv;
    const int tig = lane & 3, grp = lane >> 2;
    const int h0 = 2 * (tig & 1);
#pragma unroll
    for (int i = 0; i < KSTEPS; ++i)
#pragma unroll
        for (int u = 0; u < 4; ++u) R.o[i][u] += __shfl_xor_sync(0xffffffffu, R.o[i][u], 2);
    float* cw = comb + warp * (8 + 4 * HD);
    if (lane < 2) {
        cw[h0] = R.m_run[0];
        cw[h0 + 1] = R.m_run[1];
        cw[4 + h0] = R.l_run[0];
        cw[4 + h0 + 1] = R.l_run[1];
    }
    if (tig < 2) {
#pragma unroll
        for (int i = 0; i < KSTEPS; ++i) {
            cw[8 + (h0 + 0) * HD + 16 * i + grp] = R.o[i][0];
            cw[8 + (h0 + 1) * HD + 16 * i + grp] = R.o[i][1];
            cw[8 + (h0 + 0) * HD + 16 * i + grp + 8] = R.o[i][2];
            cw[8 + (h0 + 1) * HD + 16 * i + grp + 8] = R.o[i][3];
        }
    }
    att_sync();
    const bool complete = (run_s == seg_s) && (run_e == seg_e);
    const int Gc = gridDim.x;
    long long u0, u1;
    pk_share(U, blockIdx.x, Gc, u0, u1);
    const size_t pstride = (size_t)G * (HD + 2);
    float* mypart = K.att_part + ((size_t)blockIdx.x * 2 + (run_s == u0 ? 0 : 1)) * pstride;
    __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(P.o) + (size_t)b * P.act_ld + (size_t)g * G * HD;
    for (int idx = et; idx < G * HD; idx += (kPkAttWarps * 32)) {
        const int j = idx / HD, e = idx % HD;
        float mstar = -INFINITY;
        for (int w = 0; w < kPkAttWarps; ++w) mstar = fmaxf(mstar, comb[w * (8 + 4 * HD) + j]);
        float num = 0.f, den = 0.f;
        if (mstar != -INFINITY) {
            for (int w = 0; w < kPkAttWarps; ++w) {
                const float* c = comb + w * (8 + 4 * HD);
                if (c[j] == -INFINITY) continue;
                const float sc = exp2f(c[j] - mstar);
                num += sc * c[8 + j * HD + e];
                den += sc * c[4 + j];
            }
        }
        if (complete) {
            DT<__nv_bfloat16>::store_act(ob + idx, (size_t)P.act_plane, den > 0.f ? num / den : 0.f);
        } else {
            mypart[idx] = num;
            if (e == 0) {
                mypart[G * HD + j] = mstar;
                mypart[G * HD + G + j] = den;
            }
        }
    }
    if (!complete) {
        const int c_first = cta_of_iter(seg_s, U, Gc), c_last = cta_of_iter(seg_e - 1, U, Gc);
        __threadfence();
        att_sync();
        if (et == 0) flags[1] = (atomicAdd(&K.att_cnt[b * P.Hkv + g], 1) == pk_contributors(U, Gc, seg_s, seg_e) - 1);
        att_sync();
        if (flags[1]) {
            __threadfence();
            for (int idx = et; idx < G * HD; idx += (kPkAttWarps * 32)) {
                const int j = idx / HD;
                float M = -INFINITY;
                for (int c = c_first; c <= c_last; ++c) {
                    long long a0, a1;
                    pk_share(U, c, Gc, a0, a1);
                    if (a0 == a1) continue;
                    const int s = (c == c_first && seg_s != a0) ? 1 : 0;
                    const float* pp = K.att_part + ((size_t)c * 2 + s) * pstride;
                    M = fmaxf(M, __ldcg(pp + G * HD + j));
                }
                float num = 0.f, den = 0.f;
                for (int c = c_first; c <= c_last; ++c) {
                    long long a0, a1;
                    pk_share(U, c, Gc, a0, a1);
                    if (a0 == a1) continue;
                    const int s = (c == c_first && seg_s != a0) ? 1 : 0;
                    const float* pp = K.att_part + ((size_t)c * 2 + s) * pstride;
                    const float m = __ldcg(pp + G * HD + j);
                    if (m == -INFINITY) continue;
                    const float sc = exp2f(m - M);
                    num += sc * __ldcg(pp + idx);
                    den += sc * __ldcg(pp + G * HD + G + j);
                }
                DT<__nv_bfloat16>::store_act(ob + idx, (size_t)P.act_plane, den > 0.f ? num / den : 0.f);
            }
            if (et == 0) K.att_cnt[b * P.Hkv + g] = 0;
        }
    }
    att_sync();  // comb / flags reuse
}

CVY_DEV void pk_att_load_q(const StepParams& P, PkAttRun& R, int b, int g, int lane) {
    constexpr int HD = 128, KSTEPS = 8;
    const int G = P.H / P.Hkv;
    const int grp = lane >> 2, tig = lane & 3;
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
            const float x = valid ? v[u] * qs : 0.f;
            const float hi = __bfloat162float(__float2bfloat16_rn(x));
            v[u] = (n < 4) ? hi : (x - hi);
        }
        R.qb[ks][0] = pack_bf16(v[0], v[1]);
        R.qb[ks][1] = pack_bf16(v[2], v[3]);
    }
    R.m_run[0] = R.m_run[1] = -INFINITY;
    R.l_run[0] = R.l_run[1] = 0.f;
#pragma unroll
    for (int i = 0; i < KSTEPS; ++i) R.o[i][0] = R.o[i][1] = R.o[i][2] = R.o[i][3] = 0.f;
}

// one 16-key page of K and V (hd 128) in shared memory -> online-softmax update of the run
CVY_DEV void pk_att_page(PkAttRun& R, uint32_t kbase, uint32_t vbase, uint16_t* pw, int key_base, int nkeys, int G,
                         int lane) {
    constexpr int KSTEPS = 8;
    const int grp = lane >> 2, tig = lane & 3;
    const int h0 = 2 * (tig & 1);
    // two independent accumulator chains (even / odd k-steps) halve the dependent MMA latency
    float acc[4] = {0.f, 0.f, 0.f, 0.f}, acc2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int ks = 0; ks < KSTEPS; ++ks) {
        const int r = (lane & 7) + ((lane >> 3) & 1) * 8;
        const int dchunk = ks * 2 + (lane >> 4);
        const uint32_t addr = kbase + (dchunk >> 3) * 2048 + sw128(r, dchunk & 7);
        uint32_t a0, a1, a2, a3;
        ldsm_x4(addr, a0, a1, a2, a3);
        mma_bf16_16816((ks & 1) ? acc2 : acc, a0, a1, a2, a3, R.qb[ks][0], R.qb[ks][1]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc[u] += acc2[u];
    float s[2][2];
    s[0][0] = acc[0] + __shfl_xor_sync(0xffffffffu, acc[0], 2);
    s[0][1] = acc[1] + __shfl_xor_sync(0xffffffffu, acc[1], 2);
    s[1][0] = acc[2] + __shfl_xor_sync(0xffffffffu, acc[2], 2);
    s[1][1] = acc[3] + __shfl_xor_sync(0xffffffffu, acc[3], 2);
    const int key0 = key_base + grp;
    const bool k0ok = key0 < nkeys, k1ok = key0 + 8 < nkeys;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        if (!k0ok || h0 + j >= G) s[0][j] = -INFINITY;
        if (!k1ok || h0 + j >= G) s[1][j] = -INFINITY;
    }
    float p[2][2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        float mx = fmaxf(s[0][j], s[1][j]);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        const float mnew = fmaxf(R.m_run[j], mx);
        const float alpha = (mnew == -INFINITY) ? 1.f : exp2f(R.m_run[j] - mnew);
        p[0][j] = (mnew == -INFINITY) ? 0.f : exp2f(s[0][j] - mnew);
        p[1][j] = (mnew == -INFINITY) ? 0.f : exp2f(s[1][j] - mnew);
        float ps = p[0][j] + p[1][j];
        ps += __shfl_xor_sync(0xffffffffu, ps, 4);
        ps += __shfl_xor_sync(0xffffffffu, ps, 8);
        ps += __shfl_xor_sync(0xffffffffu, ps, 16);
        R.l_run[j] = R.l_run[j] * alpha + ps;
        R.m_run[j] = mnew;
#pragma unroll
        for (int i = 0; i < KSTEPS; ++i) {
            R.o[i][j] *= alpha;
            R.o[i][2 + j] *= alpha;
        }
    }
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
    const uint32_t pw_addr = smem_u32(pw);
    uint32_t pb0, pb1;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(pb0) : "r"(pw_addr + (uint32_t)((grp * 16 + tig * 2) * 2)));
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(pb1) : "r"(pw_addr + (uint32_t)((grp * 16 + tig * 2 + 8) * 2)));
#pragma unroll
    for (int i = 0; i < KSTEPS; ++i) {
        const int mtx = lane >> 3, r = lane & 7;
        const int key = r + (mtx >> 1) * 8;
        const int dchunk = i * 2 + (mtx & 1);
        const uint32_t addr = vbase + (dchunk >> 3) * 2048 + sw128(key, dchunk & 7);
        uint32_t a0, a1, a2, a3;
        ldsm_x4_t(addr, a0, a1, a2, a3);
        mma_bf16_16816(R.o[i], a0, a1, a2, a3, pb0, pb1);
    }
    __syncwarp();
}

// One layer's attention over this CTA's units [u0, u1) on the 8 attention warps (aw = 0..7,
// at = 0..255).  Unit = 8 KV pages of one (slot, kv head); warp aw takes page aw of the unit,
// which sits in D-ring use xcnt + aw / ppslot; each warp releases its slot itself.
CVY_DEV void pk_attention_phase(const StepParams& P, const PkParams& K, long long u0, long long u1, long long U,
                                const int* att_pre, const int* att_nch, const int* att_nkeys, uint8_t* xring,
                                uint64_t* xfull, uint64_t* xempty, float* comb, uint16_t* pbuf, int* flags,
                                uint32_t& xcnt, int aw, int at, int lane, unsigned long long* tr) {
    const int SX = K.x_stages, Bp = P.Bp, G = P.H / P.Hkv;
    const int ppslot = K.att_ppslot;
    uint16_t* pw = pbuf + aw * 128;
    PkAttRun R;
    int run_s = (int)u0;
    const bool atr = tr != nullptr && at == 0;
    unsigned long long t_wait = 0, t_fin = 0, t_q = 0, t_page = 0;
    int n_runs = 0;
    for (long long u = u0; u < u1; ++u) {
        int b, g, chunk;
        pk_att_decode(att_pre, att_nch, Bp, (int)u, b, g, chunk);
        const int nchb = att_nch[b];
        const int seg_s = att_pre[b] + g * nchb, seg_e = seg_s + nchb;
        if (u == u0 || chunk == 0) {
            run_s = (int)u;
            const unsigned long long ta = atr ? gtimer() : 0;
            pk_att_load_q(P, R, b, g, lane);
            if (atr) {
                t_q += gtimer() - ta;
                ++n_runs;
            }
        }
        const int nkeys = att_nkeys[b];
        const int npg = (nkeys + 15) / 16;
        const int pidx = chunk * 8 + aw;
        const uint32_t use = xcnt + (uint32_t)(aw / ppslot);
        const int s = (int)(use % (uint32_t)SX);
        const unsigned long long tw = atr ? gtimer() : 0;
        pk_bar_wait(&xfull[s], (use / (uint32_t)SX) & 1u, K.err,
                    (pidx < npg ? 0x510 : 0x511) | (int)(min(use, 0x7FFFFu) << 12));
        const unsigned long long tp = atr ? gtimer() : 0;
        if (atr) t_wait += tp - tw;
        if (pidx < npg) {
            const uint32_t kbase = smem_u32(xring + (size_t)s * K.x_slot + (size_t)(aw % ppslot) * 8192);
            pk_att_page(R, kbase, kbase + 4096, pw, pidx * 16, nkeys, G, lane);
        }
        if (atr) t_page += gtimer() - tp;
        __syncwarp();
        if (lane == 0) mbar_arrive(&xempty[s]);
        xcnt += (uint32_t)K.att_su;
        if (u == u1 - 1 || chunk == nchb - 1) {
            const unsigned long long tf = atr ? gtimer() : 0;
            pk_att_finish(P, K, R, comb, flags, b, g, seg_s, seg_e, run_s, (int)u + 1, U, at, aw, lane);
            if (atr) t_fin += gtimer() - tf;
        }
    }
    if (atr) {
        tr[21] = t_wait;
        tr[22] = t_page;
        tr[23] = t_q;
        tr[29] = t_fin;
        tr[30] = (unsigned long long)n_runs;
        tr[31] = (unsigned long long)(u1 - u0);
    }
}

// ------------------------------------------------------------------ the kernel
__global__ void __launch_bounds__(kPkThreads, 1)
    layers_persistent_kernel(const __grid_constant__ CUtensorMap tmWqkv, const __grid_constant__ CUtensorMap tmWo,
                             const __grid_constant__ CUtensorMap tmWgu, const __grid_constant__ CUtensorMap tmWd,
                             const __grid_constant__ CUtensorMap tmXact, const __grid_constant__ CUtensorMap tmXo,
                             const __grid_constant__ CUtensorMap tmXh, const __grid_constant__ CUtensorMap tmKV,
                             const __grid_constant__ StepParams P, const __grid_constant__ PkParams K) {
    extern __shared__ __align__(1024) uint8_t pk_raw[];
    uint8_t* smem = pk_raw + ((1024u - (smem_u32(pk_raw) & 1023u)) & 1023u);  // keeps the shared state space
    const int SW = K.w_stages, SX = K.x_stages;
    uint8_t* wring = smem;
    uint8_t* xring = wring + (size_t)SW * kPkWStage;
    float* esm = reinterpret_cast<float*>(xring + (size_t)SX * K.x_slot);
    uint16_t* pbuf = reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(esm) + PkSmem::esm_bytes());
    uint8_t* metab = reinterpret_cast<uint8_t*>(pbuf) + PkSmem::pbuf_bytes();
    EpiMeta meta;
    meta.kvoff = reinterpret_cast<long long*>(metab);
    meta.scale = reinterpret_cast<float*>(metab + 8 * kPkMaxBp);
    meta.pos = reinterpret_cast<int*>(metab + 12 * kPkMaxBp);
    int* att_nch = reinterpret_cast<int*>(metab + PkSmem::meta_bytes());
    int* att_pre = att_nch + kPkMaxBp;  // [kPkMaxBp + 1]
    int* att_nkeys = att_pre + kPkMaxBp + 1;  // [kPkMaxBp] keys attended by slot b this step
    uint64_t* wfull = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(att_nch) + PkSmem::table_bytes());
    uint64_t* wempty = wfull + SW;
    uint64_t* xfull = wempty + SW;
    uint64_t* xempty = xfull + SX;
    uint64_t* tfull = xempty + SX;
    uint64_t* tempty = tfull + 2;
    uint64_t* red_bar = tempty + 2;  // stream-K reduction bulk copies
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(red_bar + 2);
    int* flags = reinterpret_cast<int*>(tmem_slot + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int Bp = P.Bp, L = P.L, Hkv = P.Hkv;
    const int Gc = gridDim.x, cta = blockIdx.x;

    // attention work table: chunks of 4 pages per (slot, kv head) and unit prefix per slot
    if (threadIdx.x < kPkMaxBp) {
        const int b = threadIdx.x;
        int nch = 0, nkeys = 0;
        if (b < Bp) {
            const SlotDev& s = P.slots[b];
            nkeys = s.active ? min(s.pos, s.max_pos - 1) + 1 : 0;
            nch = ((nkeys + 15) / 16 + 7) / 8;  // units of 8 pages
        }
        att_nch[b] = nch;
        att_nkeys[b] = nkeys;
    }
    if (warp == 4 && lane == 0) {
        tma_prefetch_desc(&tmWqkv);
        tma_prefetch_desc(&tmWo);
        tma_prefetch_desc(&tmWgu);
        tma_prefetch_desc(&tmWd);
        for (int s = 0; s < SW; ++s) {
            mbar_init(&wfull[s], 1);
            mbar_init(&wempty[s], 1);
        }
        for (int s = 0; s < SX; ++s) {
            mbar_init(&xfull[s], 1);
            mbar_init(&xempty[s], K.x_arrivals);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], kEpiThreads);
        }
        mbar_init(red_bar, 1);
        fence_mbar_init();
    }
    if (warp == 6 && lane == 0) {
        tma_prefetch_desc(&tmXact);
        tma_prefetch_desc(&tmXo);
        tma_prefetch_desc(&tmXh);
        tma_prefetch_desc(&tmKV);
    }
    if (warp == 5) tmem_alloc(tmem_slot, K.tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) {
        // exclusive prefix of Hkv * nch over the 128 slots: 4 per lane, warp scan
        int v[4], s = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            v[j] = att_nch[lane * 4 + j] * Hkv;
            s += v[j];
        }
        int inc = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        int run = inc - s;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            att_pre[lane * 4 + j] = run;
            run += v[j];
        }
        if (lane == 31) att_pre[kPkMaxBp] = inc;
        int act = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) act += att_nch[lane * 4 + j] > 0 ? 1 : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) act += __shfl_xor_sync(0xffffffffu, act, o);
        if (lane == 0) att_nkeys[kPkMaxBp] = act * Hkv;  // number of (slot, kv head) segments
    }
    __syncthreads();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t step_tag = (uint32_t)*P.step_ctr;  // distinguishes partial tags across steps
    const long long U = att_pre[kPkMaxBp];
    const int nseg = att_nkeys[kPkMaxBp];
    // note: att_pre[b] for b >= Bp equals U (nch = 0), so decoding may search [0, Bp)
    unsigned long long* tr = (K.trace != nullptr) ? K.trace + (size_t)cta * kPkTraceStride : nullptr;

    if (warp >= 4 && warp < 8) {
    // ===================== WG1: producers + MMA issuer (few registers) =====================
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
    if (warp == 4) {
        // ===================== weight producer =====================
        // Single thread; the per-item path is a handful of integer adds (no divisions: a 64-bit
        // '%' per 16 KB item was measured to cap the stream at ~20 GB/s per SM).
        if (lane == 0) {
            const uint64_t pol_w = policy_evict_first();
            auto wmap = [&](int q) -> const CUtensorMap* {
                return q == 0 ? &tmWqkv : q == 1 ? &tmWo : q == 2 ? &tmWgu : &tmWd;
            };
            // cursor over (layer, GEMM, tile, k-block) of this CTA's shares; an L2-prefetch
            // cursor runs l2_pf items ahead of the load cursor
            struct Cur {
                int l, q, it, it1, tile, kb, row;
            };
            auto start = [&](Cur& c) {
                while (c.l < L) {
                    long long a0, a1;
                    pk_share((long long)K.g[c.q].tiles * K.g[c.q].kblocks, cta, Gc, a0, a1);
                    c.it = (int)a0;
                    c.it1 = (int)a1;
                    if (c.it < c.it1) {
                        c.tile = c.it / K.g[c.q].kblocks;
                        c.kb = c.it - c.tile * K.g[c.q].kblocks;
                        c.row = c.l * K.g[c.q].N + c.tile * 128;
                        return;
                    }
                    if (++c.q == 4) {
                        c.q = 0;
                        ++c.l;
                    }
                }
            };
            auto advance = [&](Cur& c) {
                ++c.it;
                if (++c.kb == K.g[c.q].kblocks) {
                    c.kb = 0;
                    ++c.tile;
                    c.row += 128;
                }
                if (c.it >= c.it1) {
                    if (++c.q == 4) {
                        c.q = 0;
                        ++c.l;
                    }
                    start(c);
                }
            };
            Cur c{0, 0, 0, 0, 0, 0, 0}, pf{0, 0, 0, 0, 0, 0, 0};
            start(c);
            start(pf);
            for (int j = 0; j < K.l2_pf && pf.l < L; ++j) {
                tma_prefetch_l2_2d(wmap(pf.q), pf.kb * 64, pf.row);
                advance(pf);
            }
            int s = 0;
            uint32_t ph = 0, cnt = 0;
            while (c.l < L) {
                if (K.l2_pf > 0 && pf.l < L) {
                    tma_prefetch_l2_2d(wmap(pf.q), pf.kb * 64, pf.row);
                    advance(pf);
                }
                pk_bar_wait(&wempty[s], ph ^ 1u, K.err, 0x200 | (int)(min(cnt, 0x7FFFFu) << 12));
                mbar_arrive_expect_tx(&wfull[s], kPkWStage);
                tma_load_2d(wring + (size_t)s * kPkWStage, wmap(c.q), &wfull[s], c.kb * 64, c.row, pol_w);
                ++cnt;
                if (++s == SW) {
                    s = 0;
                    ph ^= 1u;
                }
                advance(c);
            }
        }
    } else if (warp == 6) {
        // ===================== data producer (activations, KV pages) =====================
        // Activation k-blocks: lane 0.  KV pages: the whole warp -- an 8-page unit is 32 TMA
        // boxes (page, K/V, 64-dim half), one per lane, after lane 0 armed the unit's slots.
        const uint64_t pol_x = policy_evict_last();
        const uint64_t pol_kv = policy_evict_first();
        const uint32_t xrow = (uint32_t)Bp * 128u;  // one plane of one k-block
        long long u0, u1;
        pk_att_range(att_pre, att_nch, Bp, U, nseg, cta, Gc, u0, u1);
        uint32_t cnt = 0;
        for (int l = 0; l < L; ++l) {
            for (int p = 0; p < kPkPhases; ++p) {
                if (p > 0 || l > 0) {
                    if (lane == 0)
                        pk_wait_done(K.done + (p > 0 ? l * kPkPhases + p - 1 : (l - 1) * kPkPhases + 4), Gc, K.err,
                                     (0x300 + p) | ((l * 8 + p) << 12));
                    __syncwarp();
                    fence_proxy_async_global();
                }
                if (tr && l == K.trace_layer && lane == 0) tr[p] = gtimer();
                if (p == 1) {
                    const int ppslot = K.att_ppslot;
                    const int pg = lane >> 2, cc = (lane >> 1) & 1, hh = lane & 1;
                    // software pipeline: each lane's page id of the next unit loads while this
                    // unit's slots are armed
                    int nb = 0, ng = 0, nchunk = 0, nnp = 0, npage = 0;
                    auto fetch = [&](long long uu) {
                        pk_att_decode(att_pre, att_nch, Bp, (int)uu, nb, ng, nchunk);
                        nnp = min(8, (att_nkeys[nb] + 15) / 16 - nchunk * 8);
                        npage = pg < nnp ? __ldg(P.page_table + (size_t)nb * P.max_pages + nchunk * 8 + pg) : 0;
                    };
                    if (u0 < u1) fetch(u0);
                    for (long long u = u0; u < u1; ++u) {
                        const int g = ng, np = nnp, page = npage;
                        if (u + 1 < u1) fetch(u + 1);
                        if (lane == 0) {
                            for (int j = 0; j < K.att_su; ++j) {
                                const uint32_t c2 = cnt + (uint32_t)j;
                                const int s = (int)(c2 % (uint32_t)SX);
                                pk_bar_wait(&xempty[s], ((c2 / (uint32_t)SX) & 1u) ^ 1u, K.err,
                                            0x310 | (int)(min(c2, 0x7FFFFu) << 12));
                                const int pg0 = j * ppslot, pg1 = min(np, pg0 + ppslot);
                                mbar_arrive_expect_tx(&xfull[s], (uint32_t)max(0, pg1 - pg0) * 2u * 4096u);
                            }
                        }
                        __syncwarp();
                        if (pg < np) {
                            const uint32_t c2 = cnt + (uint32_t)(pg / ppslot);
                            const int s = (int)(c2 % (uint32_t)SX);
                            const int row0 = ((((l * P.n_pages + page) * 2 + cc) * Hkv) + g) * 16;
                            uint8_t* dst = xring + (size_t)s * K.x_slot + (size_t)((pg % ppslot) * 2 + cc) * 4096 + hh * 2048;
                            tma_load_2d(dst, &tmKV, &xfull[s], hh * 64, row0, pol_kv);
                        }
                        cnt += (uint32_t)K.att_su;
                    }
                } else {
                    const int q = pk_gp(p);
                    const int kblocks = K.g[q].kblocks;
                    long long a0, a1;
                    pk_share((long long)K.g[q].tiles * kblocks, cta, Gc, a0, a1);
                    if (lane == 0) {
                        const CUtensorMap* xmap = (p == 2) ? &tmXo : (p == 4) ? &tmXh : &tmXact;
                        int kb = (int)(a0 % kblocks);
                        int s = (int)(cnt % (uint32_t)SX);
                        uint32_t ph = (cnt / (uint32_t)SX) & 1u;
                        uint32_t c2 = cnt;
                        for (int it = (int)a0; it < (int)a1; ++it) {
                            pk_bar_wait(&xempty[s], ph ^ 1u, K.err, (0x320 + p) | (int)(min(c2, 0x7FFFFu) << 12));
                            mbar_arrive_expect_tx(&xfull[s], 2u * xrow);
                            uint8_t* dst = xring + (size_t)s * K.x_slot;
                            tma_load_2d(dst, xmap, &xfull[s], kb * 64, 0, pol_x);
                            tma_load_2d(dst + xrow, xmap, &xfull[s], kb * 64, (int)P.Bmax, pol_x);
                            ++c2;
                            if (++kb == kblocks) kb = 0;
                            if (++s == SX) {
                                s = 0;
                                ph ^= 1u;
                            }
                        }
                    }
                    cnt += (uint32_t)(a1 - a0);
                    __syncwarp();
                }
            }
        }
    } else if (warp == 5) {
        // ===================== MMA issuer =====================
        const uint32_t idesc = idesc_bf16_f32(128, (uint32_t)(2 * Bp));
        const uint64_t wd0 = sdesc_kmajor_sw128(smem_u32(wring));
        const uint64_t xd0 = sdesc_kmajor_sw128(smem_u32(xring));
        long long u0, u1;
        pk_att_range(att_pre, att_nch, Bp, U, nseg, cta, Gc, u0, u1);
        uint32_t wcnt = 0, xcnt = 0, acnt = 0;
        for (int l = 0; l < L; ++l) {
            for (int p = 0; p < kPkPhases; ++p) {
                if (p == 1) {
                    // The attention units occupy D-ring uses this warp never consumes.  Before
                    // waiting on the ring again it must know they were all consumed: an mbarrier
                    // parity wait more than one phase ahead of the barrier would pass early.
                    xcnt += (uint32_t)(u1 - u0) * (uint32_t)K.att_su;
                    pk_wait_done(K.done + l * kPkPhases + 1, Gc, K.err, 0x430 | (l << 12));
                    continue;
                }
                const PkGemm& g = K.g[pk_gp(p)];
                long long a0, a1;
                pk_share((long long)g.tiles * g.kblocks, cta, Gc, a0, a1);
                int it = (int)a0;
                const int it1 = (int)a1;
                int ws = (int)(wcnt % (uint32_t)SW), xs = (int)(xcnt % (uint32_t)SX);
                uint32_t wph = (wcnt / (uint32_t)SW) & 1u, xph = (xcnt / (uint32_t)SX) & 1u;
                while (it < it1) {
                    const int tile = it / g.kblocks;
                    const int seg_end = min(it1, (tile + 1) * g.kblocks);
                    const int as = (int)(acnt & 1u);
                    pk_bar_wait(&tempty[as], ((acnt >> 1) & 1u) ^ 1u, K.err, 0x400 | (int)(min(acnt, 0x7FFFFu) << 12));
                    tc_fence_after();
                    const uint32_t dcol = tmem_base + (uint32_t)(as * 2 * Bp);
                    bool first = true;
                    for (; it < seg_end; ++it) {
                        pk_bar_wait(&wfull[ws], wph, K.err, 0x410 | (int)(min(wcnt, 0x7FFFFu) << 12));
                        pk_bar_wait(&xfull[xs], xph, K.err, 0x420 | (int)(min(xcnt, 0x7FFFFu) << 12));
                        tc_fence_after();
                        if (lane == 0) {
                            const uint64_t ad = desc_add(wd0, (uint32_t)ws * kPkWStage);
                            const uint64_t bd = desc_add(xd0, (uint32_t)xs * K.x_slot);
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                umma_bf16(dcol, desc_add(ad, (uint32_t)k * 32u), desc_add(bd, (uint32_t)k * 32u), idesc,
                                          (first && k == 0) ? 0u : 1u);
                            umma_commit(&wempty[ws]);
                            for (int a = 0; a < K.x_arrivals; ++a) umma_commit(&xempty[xs]);
                        }
                        __syncwarp();
                        first = false;
                        ++wcnt;
                        ++xcnt;
                        if (++ws == SW) {
                            ws = 0;
                            wph ^= 1u;
                        }
                        if (++xs == SX) {
                            xs = 0;
                            xph ^= 1u;
                        }
                    }
                    if (lane == 0) umma_commit(&tfull[as]);
                    __syncwarp();
                    ++acnt;
                }
                if (tr && l == K.trace_layer && lane == 0) tr[24 + p] = gtimer();
            }
        }
    }
    } else if (warp < 4) {
        // ===================== WG0: epilogue / attention warps 0-3 =====================
        asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
        const int et = threadIdx.x;
        long long u0, u1;
        pk_att_range(att_pre, att_nch, Bp, U, nseg, cta, Gc, u0, u1);
        uint32_t xcnt = 0, acnt = 0, red_ph = 0;
        for (int l = 0; l < L; ++l) {
            for (int p = 0; p < kPkPhases; ++p) {
                if (p > 0 || l > 0) {
                    if (et == 0)
                        pk_wait_done(K.done + (p > 0 ? l * kPkPhases + p - 1 : (l - 1) * kPkPhases + 4), Gc, K.err,
                                     (0x500 + p) | ((l * 8 + p) << 12));
                    epi_sync();
                }
                if (p == 1) {
                    pk_attention_phase(P, K, u0, u1, U, att_pre, att_nch, att_nkeys, xring, xfull, xempty, esm, pbuf,
                                       flags, xcnt, warp, et, lane, l == K.trace_layer ? tr : nullptr);
                    // warpgroup 2's attention stores are fenced before this barrier too
                    fence_proxy_async_global();
                    __threadfence();
                    att_sync();
                    if (tr && l == K.trace_layer && et == 0) tr[17] = gtimer();
                } else {
                    const int q = pk_gp(p);
                    {
                        long long a0, a1;
                        pk_share((long long)K.g[q].tiles * K.g[q].kblocks, cta, Gc, a0, a1);
                        xcnt += (uint32_t)(a1 - a0);
                    }
                    EpiArgs E;
                    E.layer = l;
                    E.N = K.g[q].N;
                    E.norm_w = nullptr;
                    E.store_out = nullptr;
                    if (p == 0) E.kind = EPI_QKV;
                    else if (p == 3) E.kind = EPI_SWIGLU;
                    else {
                        E.kind = EPI_RESID;
                        E.norm_w = (p == 2) ? P.mlp_norm + (size_t)l * P.d
                                            : ((l + 1 < L) ? P.attn_norm + (size_t)(l + 1) * P.d : P.final_norm);
                    }
                    epilogue_prepare(P, E, meta, et);
                    epi_sync();
                    if (p == 0)
                        pk_gemm_epilogue<EPI_QKV>(P, K, E, q, meta, esm, flags, tfull, tempty, tmem_base, acnt, et, warp,
                                                     l == K.trace_layer ? tr : nullptr, ((step_tag * 128u + (uint32_t)l) << 3) + (uint32_t)q + 1u,
                                                     red_bar, red_ph, xring);
                    else if (p == 3)
                        pk_gemm_epilogue<EPI_SWIGLU>(P, K, E, q, meta, esm, flags, tfull, tempty, tmem_base, acnt, et, warp,
                                                     l == K.trace_layer ? tr : nullptr, ((step_tag * 128u + (uint32_t)l) << 3) + (uint32_t)q + 1u,
                                                     red_bar, red_ph, xring);
                    else
                        pk_gemm_epilogue<EPI_RESID>(P, K, E, q, meta, esm, flags, tfull, tempty, tmem_base, acnt, et, warp,
                                                     l == K.trace_layer ? tr : nullptr, ((step_tag * 128u + (uint32_t)l) << 3) + (uint32_t)q + 1u,
                                                     red_bar, red_ph, xring);
                }
                // phase done: every store of this CTA's phase work is visible (generic and to
                // the async proxy that the next phase's TMA loads use) before the counter moves
                fence_proxy_async_global();
                __threadfence();
                epi_sync();
                if (et == 0) {
                    if (tr && l == K.trace_layer) tr[8 + p] = gtimer();
                    red_release_gpu_add(K.done + l * kPkPhases + p, 1);
                }
            }
        }
    }
    else {
        // ===================== WG2: attention warps 8-11 =====================
        const int at = threadIdx.x - 128;  // 128..255 among the attention threads
        long long u0, u1;
        pk_att_range(att_pre, att_nch, Bp, U, nseg, cta, Gc, u0, u1);
        uint32_t xcnt = 0;
        for (int l = 0; l < L; ++l) {
            for (int p = 0; p < kPkPhases; ++p) {
                if (p != 1) {
                    long long a0, a1;
                    pk_share((long long)K.g[pk_gp(p)].tiles * K.g[pk_gp(p)].kblocks, cta, Gc, a0, a1);
                    xcnt += (uint32_t)(a1 - a0);
                    continue;
                }
                if (at == 128) pk_wait_done(K.done + l * kPkPhases, Gc, K.err, 0x601 | (l << 12));
                named_bar_sync(kWg2Bar, 128);
                pk_attention_phase(P, K, u0, u1, U, att_pre, att_nch, att_nkeys, xring, xfull, xempty, esm, pbuf,
                                   flags, xcnt, warp - 4, at, lane, nullptr);
                fence_proxy_async_global();
                __threadfence();
                att_sync();
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc(tmem_base, K.tmem_cols);
    }
}

}  // namespace cvy
