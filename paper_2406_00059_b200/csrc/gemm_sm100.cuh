// gemm_sm100.cuh -- skinny decode GEMM on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Y^T[n][b] = sum_k W[n][k] * X[b][k]  (swap-AB: the weight rows are the UMMA M=128 side,
// the padded batch is the UMMA N side), bf16 inputs, fp32 accumulation in TMEM.  X is the
// (hi, lo) bf16 pair of the activation: both planes form ONE B
// operand of N = 2*bq rows (TMEM columns [0,bq) = W.x_hi, [bq,2bq) = W.x_lo, summed in the
// epilogue).  Batches above 128 run as Bp/128 batch tiles of bq = 128 columns on grid.y.
//
// Work split (chosen per GEMM by the engine):
//  * whole tiles (split = 1): one CTA per 128- or 256-row tile (gate/up, LM head);
//  * cluster split-K (split = S in 2..4): tile = blockIdx.x / S, its K range split over the S
//    CTAs of a thread-block cluster; partials are staged in the idle pipeline smem and
//    reduce-scattered through DSMEM in rank order (deterministic) -- QKV, O, down;
//  * stream-K (split = 0, batch tiles / forced): contiguous (tile, k-block) ranges per CTA;
//    shared tiles are summed with fp32 red.add into an L2 accumulator and the last arriving
//    contributor (ticket) runs the epilogue (summation order varies run to run).
//
// Warp roles (192 threads): warps 0-3 epilogue (TMEM lanes 0-127), warp 4 TMA producer,
// warp 5 MMA issuer (one lane; descriptors precomputed, loops unrolled) and TMEM owner.
#pragma once
#include "common.cuh"
#include "epilogue.cuh"
#include "step_params.h"

namespace cvy {

// Geometry of the GEMM launched after this one (its weight stream is prefetched into L2 during
// this kernel's epilogue tail, when HBM would otherwise idle).
struct GemmNext {
    int32_t tiles, kblocks, split, rows_per_tile, w_row0, grid, bk;
    int32_t blocks;  // k-blocks prefetched per next-kernel CTA (0: off)
};

constexpr int kMaxSplit = 4;  // cluster split-K ranks the DSMEM reduce-scatter sums (t4[kMaxSplit])

struct GemmTC {
    int32_t N;          // weight rows of this GEMM (one layer)
    int32_t K;
    int32_t nsub;       // 128-row sub-tiles per tile (must equal the kernel's NSUB)
    int32_t mma_n;      // UMMA N of one MMA
    int32_t nbh;        // batch halves (bq / mma_n) when the planes are not merged
    int32_t bq;         // batch columns of one CTA (= Bp, or 128 when the batch is tiled)
    int32_t nbt;        // batch tiles (grid.y): Bp = nbt * bq; each CTA row of the grid runs the
                        // merged 128-column pipeline on its batch tile (CTAs sharing a weight
                        // tile read it through L2)
    int32_t tiles;
    int32_t kblocks;    // K / bk
    int32_t bk;         // K elements per pipeline stage: 64 (128B swizzle) or 32 (64B swizzle)
    int32_t stages;
    int32_t acc_stages; // TMEM accumulator buffers (1 or 2)
    uint32_t tmem_cols;
    int32_t cols_per_sub;  // TMEM columns of one sub-tile accumulator (2*Bp merged, else Bp)
    int32_t merge;      // 1: hi/lo planes merged into one N = 2*Bp MMA
    int32_t split;      // 0: stream-K over all CTAs; S >= 1: tile = blockIdx/S, K split over the S
                        //    CTAs of a thread-block cluster, reduced through DSMEM
    int32_t pair;       // 1: CTA pairs (cta_group::2, clusters of 2): a tile is 256 weight rows, CTA
                        //    rank r holds rows [128r, 128r+128) and activation plane r (hi / lo), the
                        //    leader issues M = 256, N = 2*bq MMAs; split is 1 (whole tiles) or 0
                        //    (stream-K over pairs)
    int32_t w_row0;     // first row of this layer's matrix in the weight tensor map
    int32_t wtiled;     // 1: weights packed tile-major [rows/128][K/64][128][64] (cvy_pack_weights_tiled):
                        //    every 128-row x 64-column box is 16 contiguous KB (row-major boxes
                        //    read 128 B from each of 128 rows; DESIGN.md §7.2 "Weight layout")
    int32_t x_plane_rows;  // row offset of the lo plane in the activation tensor map
    float* part;        // [tiles][nsub*128][Bp] fp32 accumulators of shared tiles (zero between uses)
    int32_t* tile_cnt;  // [tiles] arrival tickets (zero between uses; reset by the last arriver)
    EpiArgs epi;
    int32_t dbg;        // measurement knobs (test hook only): 1 no epilogue work, 2 no MMA issue,
                        // 4 shared tiles: store partial only, 8 skip the epilogue functor
    unsigned long long* trace;  // test hook: [grid][kTraceStride] %globaltimer stamps, or null
    int32_t l2_prefetch;        // k-block stages prefetched into L2 beyond the smem ring
    GemmNext nx;                // next GEMM of the step (prefetched through tmN)
};

CVY_DEV unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

constexpr int kGemmThreads = 192;
// The gate/up GEMM runs its (latency-bound) SwiGLU epilogue on two groups of 4 warps (warps 0-3
// and 6-9 both cover the 4 TMEM lane quadrants), alternating 32-column chunks.
__host__ __device__ constexpr int gemm_epi_groups(int epi) { return epi == EPI_SWIGLU ? 2 : 1; }
__host__ __device__ constexpr int gemm_threads(int epi) { return gemm_epi_groups(epi) == 2 ? 320 : kGemmThreads; }
// threads a launch uses: the second epilogue group only for whole single-tile CTAs (split == 1)
__host__ __device__ constexpr int gemm_launch_threads(int epi, int split) {
    return (gemm_epi_groups(epi) == 2 && split == 1) ? 320 : kGemmThreads;
}
constexpr int kTraceStride = 16;

// shared-memory carve-up (host and device agree); rows are bk*2 bytes (one swizzle atom)
struct GemmSmem {
    __host__ __device__ static constexpr uint32_t w_bytes(int nsub, int bk) { return (uint32_t)nsub * 128u * bk * 2u; }
    __host__ __device__ static constexpr uint32_t x_bytes(int Bp, int bk) { return (uint32_t)Bp * bk * 2u; }
    __host__ __device__ static constexpr uint32_t stage_bytes(int nsub, int Bp, int planes, int bk) {
        return w_bytes(nsub, bk) + (uint32_t)planes * x_bytes(Bp, bk);
    }
    __host__ __device__ static constexpr uint32_t fixed_bytes(int Bp) {
        return 128u * kEsmLd * 4u      // esm
               + 16u                    // alignment pad
               + (uint32_t)Bp * 16u     // EpiMeta: scale, pos, kvoff
               + 64u * 8u               // barriers
               + 64u;                   // tmem addr + flags
    }
};

// Issue L2 prefetches of the next GEMM's first k-blocks (the ones its CTAs load first),
// spread over the 32 lanes of one warp; this CTA covers next-kernel CTAs blockIdx.x + j*grid.
CVY_DEV void prefetch_next_gemm(const GemmTC& G, const CUtensorMap* tmN, int lane) {
    const GemmNext& nx = G.nx;
    if (nx.blocks <= 0) return;
    if (lane == 0) tma_prefetch_desc(tmN);
    int j = 0;
    for (int c = blockIdx.x; c < nx.grid; c += gridDim.x) {
        long long a0, a1;
        if (nx.split > 0) {
            const int t = c / nx.split, r = c % nx.split;
            a0 = (long long)t * nx.kblocks + ((long long)r * nx.kblocks) / nx.split;
            a1 = (long long)t * nx.kblocks + ((long long)(r + 1) * nx.kblocks) / nx.split;
        } else {
            const long long T = (long long)nx.tiles * nx.kblocks;
            a0 = ((long long)c * T) / nx.grid;
            a1 = ((long long)(c + 1) * T) / nx.grid;
        }
        a1 = min(a1, a0 + (long long)nx.blocks);
        for (long long i = a0; i < a1; ++i, ++j)
            if ((j & 31) == lane)
                tma_prefetch_l2_2d(tmN, (int)(i % nx.kblocks) * nx.bk, nx.w_row0 + (int)(i / nx.kblocks) * nx.rows_per_tile);
    }
}

// Weight k-block kb of row tile `tile` (128 * nsub rows) into the stage's weight slot.
template <int NSUB, int BK>
CVY_DEV void load_w_tile(void* dst, const CUtensorMap* tmW, uint64_t* bar, const GemmTC& G, int tile, int kb,
                         uint64_t pol) {
    if (!G.wtiled) {
        tma_load_2d(dst, tmW, bar, kb * BK, G.w_row0 + tile * 128 * NSUB, pol);
    } else {
#pragma unroll
        for (int s = 0; s < NSUB; ++s) {
            const int rt = G.w_row0 / 128 + tile * NSUB + s;
            tma_load_2d(static_cast<uint8_t*>(dst) + s * 16384, tmW, bar, 0, (rt * G.kblocks + kb) * 128, pol);
        }
    }
}

CVY_DEV int cta_of_iter(long long i, long long T, int G) {
    long long c = (i * G) / T;
    while (c + 1 < G && ((c + 1) * T) / G <= i) ++c;
    while (c > 0 && (c * T) / G > i) --c;
    return (int)c;
}

// fp32 x4 reduction into global memory at L2, no return value
CVY_DEV void red_add_v4(float* p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// descriptor arithmetic: adding `bytes` (multiple of 16) to the start address field
CVY_DEV uint64_t desc_add(uint64_t d, uint32_t bytes) { return d + (uint64_t)(bytes >> 4); }

template <typename T, int NSUB, bool MERGE, int BK, int EPI, bool PAIR = false>
__global__ void __launch_bounds__(gemm_threads(EPI), 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                   const __grid_constant__ StepParams P, const __grid_constant__ GemmTC G,
                   const __grid_constant__ CUtensorMap tmN) {
    constexpr uint32_t ROW = BK * 2;                  // bytes per smem row
    // a pair stage holds two BK-column k-blocks (8 MMAs per barrier round trip, as a 256-row
    // single-CTA stage); G.kblocks counts stages
    constexpr int KB2 = PAIR ? 2 : 1;
    constexpr uint32_t WB = NSUB * 128u * ROW * KB2;  // weight bytes per stage
    constexpr int KSTEPS = BK / 16 * KB2;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // aligned by an offset from smem_raw (not a uintptr round trip), so the compiler keeps the
    // shared state space and the epilogue's exchange / metadata accesses compile to LDS / STS
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int Bp = G.bq;                              // this CTA's batch columns
    const int cbase = (int)blockIdx.y * G.bq;         // first batch column of this CTA
    const uint32_t XB = (uint32_t)Bp * ROW * KB2;     // one activation plane per stage
    // a pair CTA holds one activation plane (its half of the MMA's N = 2*bq B operand)
    const uint32_t stage_bytes = WB + (PAIR ? 1u : 2u) * XB;
    uint8_t* fixed = smem + (size_t)G.stages * stage_bytes;
    constexpr int EG = gemm_epi_groups(EPI);
    float* esm0 = reinterpret_cast<float*>(fixed);
    EpiMeta meta;
    meta.kvoff = reinterpret_cast<long long*>(esm0 + 128 * kEsmLd + 4);
    meta.scale = reinterpret_cast<float*>(meta.kvoff + P.Bp);
    meta.pos = reinterpret_cast<int*>(meta.scale + P.Bp);
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(meta.pos + P.Bp + 2);
    uint64_t* empty_bar = full_bar + G.stages;
    uint64_t* tfull_bar = empty_bar + G.stages;
    uint64_t* tempty_bar = tfull_bar + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
    int* flags = reinterpret_cast<int*>(tmem_slot + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // epilogue group of this warp (0: warps 0-3, 1: warps 6-9).  The second group works only when
    // the CTA owns exactly one whole tile (split == 1): its epilogue starts after the tile's last
    // MMA, so the pipeline ring is idle and holds group 1's exchange buffer (no shared memory
    // taken from the ring's stages)
    const int egroup = warp >= 6 ? 1 : 0;
    const int n_egroups = (EG == 2 && G.split == 1 && blockDim.x >= 320) ? 2 : 1;
    float* esm = egroup ? reinterpret_cast<float*>(smem) : esm0;
    const long long T_iters = (long long)G.tiles * G.kblocks;
    // pair mode: work is assigned per CTA pair (both CTAs of a pair run the same k-range)
    const int prank = PAIR ? (int)(blockIdx.x & 1u) : 0;
    const int bx = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    const int Gc = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
    long long it0, it1;
    int crank = 0;
    if (G.split > 0) {
        // cluster split-K: CTA (tile, rank) owns k-blocks [rank*KB/S, (rank+1)*KB/S) of one tile
        const int tile = bx / G.split;
        crank = bx % G.split;
        it0 = (long long)tile * G.kblocks + ((long long)crank * G.kblocks) / G.split;
        it1 = (long long)tile * G.kblocks + ((long long)(crank + 1) * G.kblocks) / G.split;
    } else {
        it0 = ((long long)bx * T_iters) / Gc;
        it1 = ((long long)(bx + 1) * T_iters) / Gc;
    }
    // 128-row weight tile (of the whole matrix) that sub-tile s of `tile` covers in this CTA
    auto row_tile = [&](int tile, int s) { return PAIR ? tile * 2 + prank : tile * NSUB + s; };

    if (warp == 4 && lane == 0) {
        tma_prefetch_desc(&tmW);
        tma_prefetch_desc(&tmX);
        for (int s = 0; s < G.stages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull_bar[s], 1);
            // pair: the leader's accumulator is released by both CTAs' epilogue threads
            mbar_init(&tempty_bar[s], kEpiThreads * n_egroups * (PAIR ? 2 : 1));
        }
        fence_mbar_init();
    }
    if (warp == 5) {
        if (PAIR) tmem_alloc_pair(tmem_slot, G.tmem_cols);
        else tmem_alloc(tmem_slot, G.tmem_cols);
    }
    tc_fence_before();
    // pair: the peer's TMA loads complete on the leader's barriers -- both initialised first
    if (PAIR) cluster_sync_all();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_launch_dependents();
    unsigned long long* tr = (G.trace && blockIdx.y == 0) ? G.trace + (size_t)blockIdx.x * kTraceStride : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = gtimer();

    if (warp == 4) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            const uint64_t pol_w = policy_evict_first();
            const uint64_t pol_x = policy_evict_last();
            const int rows_per_tile = 128 * NSUB;
            const int xh = MERGE ? 1 : G.nbh;
            const int xrows = MERGE ? Bp : G.mma_n;
            // stage s's transaction barrier: the leader's (both halves of a pair count there)
            auto bar_cl = [&](int s) -> uint32_t {
                return PAIR ? mapa_shared(smem_u32(&full_bar[s]), 0u) : smem_u32(&full_bar[s]);
            };
            auto expect = [&](int s) {
                if (!PAIR) mbar_arrive_expect_tx(&full_bar[s], stage_bytes);
                else if (prank == 0) mbar_arrive_expect_tx(&full_bar[s], 2u * stage_bytes);
            };
            auto load_w = [&](uint8_t* dst, int s, int tile, int kb) {
                if (PAIR) {
                    const int rt = row_tile(tile, 0);
#pragma unroll
                    for (int j = 0; j < KB2; ++j) {
                        const int kc = kb * KB2 + j;  // BK-column k-block
                        uint8_t* d = dst + j * 128 * ROW;
                        if (!G.wtiled) tma_load_2d_pair(d, &tmW, bar_cl(s), kc * BK, G.w_row0 + rt * 128, pol_w);
                        else tma_load_2d_pair(d, &tmW, bar_cl(s), 0, ((G.w_row0 / 128 + rt) * G.kblocks * KB2 + kc) * 128, pol_w);
                    }
                } else {
                    load_w_tile<NSUB, BK>(dst, &tmW, &full_bar[s], G, tile, kb, pol_w);
                }
            };
            auto load_x = [&](uint8_t* sx, int s, int kb) {
                if (PAIR) {
#pragma unroll
                    for (int j = 0; j < KB2; ++j)
                        tma_load_2d_pair(sx + (size_t)j * Bp * ROW, &tmX, bar_cl(s), (kb * KB2 + j) * BK,
                                         prank * G.x_plane_rows + cbase, pol_x);
                } else {
                    for (int pl = 0; pl < 2; ++pl)
                        for (int h = 0; h < xh; ++h)
                            tma_load_2d(sx + (size_t)(pl * Bp + h * xrows) * ROW, &tmX, &full_bar[s], kb * BK,
                                        pl * G.x_plane_rows + cbase + h * xrows, pol_x);
                }
            };
            // weights do not depend on the previous kernel: issue the first stages before the
            // grid-dependency wait so the weight stream starts under the previous kernel's tail
            const long long n_it = it1 - it0;
            const int pre = (int)(n_it < G.stages ? n_it : G.stages);
            for (int i = 0; i < pre; ++i) {
                const long long it = it0 + i;
                const int tile = (int)(it / G.kblocks), kb = (int)(it % G.kblocks);
                expect(i);
                load_w(smem + (size_t)i * stage_bytes, i, tile, kb);
            }
            // look-ahead into L2 beyond the smem ring (l2_prefetch k-blocks, rolling with the main
            // loop): more weight bytes in flight per SM than the ring holds
            auto l2_pf = [&](long long it) {
                const int tile = (int)(it / G.kblocks), kb = (int)(it % G.kblocks);
                if (!G.wtiled) {
                    tma_prefetch_l2_2d(&tmW, kb * BK, G.w_row0 + tile * rows_per_tile);
                } else {
#pragma unroll
                    for (int s = 0; s < NSUB; ++s)
                        tma_prefetch_l2_2d(&tmW, 0, ((G.w_row0 / 128 + tile * NSUB + s) * G.kblocks + kb) * 128);
                }
            };
            long long pf_next = it0 + pre;
            const long long pf_end = PAIR ? pf_next : min(it1, it0 + pre + (long long)G.l2_prefetch);
            for (; pf_next < pf_end; ++pf_next) l2_pf(pf_next);
            pdl_wait();
            if (G.epi.span_kind >= 0) span_begin(P.spans, P.span_base + G.epi.layer * 8 + G.epi.span_kind);
            for (int i = 0; i < pre; ++i) {
                const int kb = (int)((it0 + i) % G.kblocks);
                load_x(smem + (size_t)i * stage_bytes + WB, i, kb);
            }
            int stage = pre % G.stages;
            uint32_t phase = (pre == G.stages) ? 1u : 0u;
            for (long long it = it0 + pre; it < it1; ++it) {
                const int tile = (int)(it / G.kblocks), kb = (int)(it % G.kblocks);
                mbar_wait(&empty_bar[stage], phase ^ 1u);
                if (!PAIR && G.l2_prefetch > 0 && pf_next < it1) l2_pf(pf_next++);
                uint8_t* sw = smem + (size_t)stage * stage_bytes;
                expect(stage);
                load_w(sw, stage, tile, kb);
                load_x(sw + WB, stage, kb);
                if (++stage == G.stages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
            if (tr) tr[1] = gtimer();
        }
        // non-split: warm L2 with the next GEMM's first k-blocks right behind our own stream
        __syncwarp();
        if (G.split <= 1 && blockIdx.y == 0) prefetch_next_gemm(G, &tmN, lane);
    } else if (warp == 5 && (!PAIR || prank == 0)) {
        // ===================== MMA issuer (pair: the leader CTA only) =====================
        const uint32_t idesc = idesc_bf16_f32(PAIR ? 256 : 128, (uint32_t)G.mma_n);
        const uint64_t d0 = (BK == 64) ? sdesc_kmajor_sw128(smem_u32(smem)) : sdesc_kmajor_sw64(smem_u32(smem));
        int stage = 0;
        uint32_t phase = 0;
        int as = 0;
        uint32_t aphase = 0;
        long long it = it0;
        while (it < it1) {
            const int tile = (int)(it / G.kblocks);
            const long long seg_end = min(it1, (long long)(tile + 1) * G.kblocks);
            mbar_wait(&tempty_bar[as], aphase ^ 1u);
            tc_fence_after();
            const uint32_t dcol = tmem_base + (uint32_t)(as * NSUB * G.cols_per_sub);
            bool first = true;
            for (; it < seg_end; ++it) {
                mbar_wait(&full_bar[stage], phase);
                tc_fence_after();
                if (lane == 0 && !(G.dbg & 2)) {
                    const uint64_t ws = desc_add(d0, (uint32_t)stage * stage_bytes);
                    const uint64_t xs = desc_add(ws, WB);
#pragma unroll
                    for (int k = 0; k < KSTEPS; ++k) {
#pragma unroll
                        for (int s = 0; s < NSUB; ++s) {
                            const uint64_t ad = desc_add(ws, (uint32_t)s * 128u * ROW + (uint32_t)k * 32u);
                            if (PAIR) {
                                // k-step k: k-block k / 4 of the stage, 16-column step k % 4
                                const uint32_t j = (uint32_t)k / (BK / 16), kk = (uint32_t)k % (BK / 16);
                                umma_bf16_pair(dcol, desc_add(ws, j * 128u * ROW + kk * 32u),
                                               desc_add(xs, j * (uint32_t)Bp * ROW + kk * 32u), idesc,
                                               (first && k == 0) ? 0u : 1u);
                            } else if (MERGE) {
                                umma_bf16(dcol + (uint32_t)(s * G.cols_per_sub), ad, desc_add(xs, (uint32_t)k * 32u),
                                          idesc, (first && k == 0) ? 0u : 1u);
                            } else {
                                for (int h = 0; h < G.nbh; ++h)
#pragma unroll
                                    for (int pl = 0; pl < 2; ++pl)
                                        umma_bf16(dcol + (uint32_t)(s * G.cols_per_sub + h * G.mma_n), ad,
                                                  desc_add(xs, (uint32_t)(pl * Bp + h * G.mma_n) * ROW + (uint32_t)k * 32u),
                                                  idesc, (first && k == 0 && pl == 0) ? 0u : 1u);
                            }
                        }
                    }
                }
                if (lane == 0) {
                    if (PAIR) umma_commit_pair(&empty_bar[stage], 3);  // both CTAs' producers
                    else umma_commit(&empty_bar[stage]);
                }
                __syncwarp();
                first = false;
                if (++stage == G.stages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
            if (lane == 0) {
                if (PAIR) umma_commit_pair(&tfull_bar[as], 3);  // both CTAs' epilogues
                else umma_commit(&tfull_bar[as]);
            }
            __syncwarp();
            if (++as == G.acc_stages) {
                as = 0;
                aphase ^= 1u;
            }
        }
    } else if (warp != 5) {
        // ===================== epilogue (warps 0-3, and 6-9 for the gate/up GEMM) =====================
        const int et = (warp & 3) * 32 + lane;  // 0..127 == TMEM lane == tile row
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        // both groups meet here (prepare, stream-K ticket); one group: its own barrier
        auto grp_sync = [&]() {
            if (n_egroups == 2) named_bar_sync(4, 2 * kEpiThreads); else epi_sync();
        };
        if (egroup >= n_egroups) it0 = it1;  // second group idle in split-K mode
        // release accumulator stage a to the MMA issuer (pair: the leader's barrier)
        auto release_acc = [&](int a) {
            if (PAIR && prank != 0) mbar_arrive_cluster(mapa_shared(smem_u32(&tempty_bar[a]), 0u));
            else mbar_arrive(&tempty_bar[a]);
        };
        const int rows = NSUB * 128;
        bool prepared = false;
        int as = 0;
        uint32_t aphase = 0;
        long long it = it0;
        while (it < it1) {
            const int tile = (int)(it / G.kblocks);
            const long long tb = (long long)tile * G.kblocks, te = tb + G.kblocks;
            it = min(it1, te);
            const int c_first = G.split > 0 ? 0 : cta_of_iter(tb, T_iters, Gc);
            const int c_last = G.split > 0 ? 0 : cta_of_iter(te - 1, T_iters, Gc);
            if (!prepared) {
                pdl_wait();
                if (egroup == 0) epilogue_prepare(P, G.epi, meta, et);
                grp_sync();
                prepared = true;
            }
            mbar_wait(&tfull_bar[as], aphase);
            tc_fence_after();
            if (tr && et == 0 && egroup == 0) tr[2 + (it >= it1 ? 1 : 0)] = gtimer();  // [2] first / [3] last segment's MMA done
            if (G.dbg & 1) {
                tc_fence_before();
                release_acc(as);
                if (++as == G.acc_stages) {
                    as = 0;
                    aphase ^= 1u;
                }
                continue;
            }
            const uint32_t tacc = tmem_base + lane_off + (uint32_t)(as * NSUB * G.cols_per_sub);
            bool did_epi = false;
            if (G.split > 1) {
                // stage this CTA's partial in its (now idle) pipeline smem as 16-column units
                // [sub][unit][row][16] for the cluster reduce-scatter after the role branches
                float* stagep = reinterpret_cast<float*>(smem);
                for (int s = 0; s < NSUB; ++s)
                    for (int cb = 0; cb < Bp; cb += 32) {
                        float v[32];
                        if (MERGE) {
                            float w[32];
                            tmem_ld32x2(tacc + (uint32_t)(s * G.cols_per_sub + cb),
                                        tacc + (uint32_t)(s * G.cols_per_sub + Bp + cb), v, w);
#pragma unroll
                            for (int i = 0; i < 32; ++i) v[i] += w[i];
                        } else {
                            tmem_ld32(tacc + (uint32_t)(s * G.cols_per_sub + cb), v);
                        }
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            // [unit][q][row][4]: a warp's float4 stores (and the peers' loads)
                            // cover 512 contiguous bytes -- no bank conflicts
                            float4* dst = reinterpret_cast<float4*>(stagep) +
                                          (size_t)(s * (Bp / 16) + cb / 16 + h) * 512 + et;
#pragma unroll
                            for (int q = 0; q < 4; ++q)
                                dst[q * 128] = make_float4(v[16 * h + 4 * q], v[16 * h + 4 * q + 1], v[16 * h + 4 * q + 2],
                                                           v[16 * h + 4 * q + 3]);
                        }
                    }
                tc_fence_before();
                release_acc(as);
            } else if (c_first == c_last) {
                // sole contributor: epilogue straight from TMEM (hi + lo planes summed); with two
                // epilogue groups, group g takes the chunks ci = g, g + 2, ...
                for (int s = 0; s < NSUB; ++s)
                    for (int cb = 0; cb < Bp; cb += 32) {
                        if (n_egroups == 2 && (((s * Bp + cb) >> 5) & 1) != egroup) continue;
                        float v[32];
                        if (MERGE) {
                            float w[32];
                            tmem_ld32x2(tacc + (uint32_t)(s * G.cols_per_sub + cb),
                                        tacc + (uint32_t)(s * G.cols_per_sub + Bp + cb), v, w);
#pragma unroll
                            for (int i = 0; i < 32; ++i) v[i] += w[i];
                        } else {
                            tmem_ld32(tacc + (uint32_t)(s * G.cols_per_sub + cb), v);
                        }
                        if (!(G.dbg & 8))
                            epilogue_chunk<T, EPI>(P, G.epi, row_tile(tile, s) * 128, cbase + cb, v, esm, meta, et);
                    }
                tc_fence_before();
                release_acc(as);
                did_epi = true;
            } else {
                // Shared tile: add this CTA's partial into the tile's fp32 accumulator with L2
                // vector reductions (no return, nobody waits), take an arrival ticket; the last
                // arriver reads the completed sum, re-zeroes it, and runs the epilogue.
                // pair: each CTA's 128-row half has its own accumulator and ticket
                const size_t ai = PAIR ? ((size_t)tile * G.nbt + blockIdx.y) * 2 + prank : (size_t)tile * G.nbt + blockIdx.y;
                float* acc = G.part + ai * rows * Bp;
                int32_t* ticket = G.tile_cnt + ai;
                for (int s = 0; s < NSUB; ++s)
                    for (int cb = 0; cb < Bp; cb += 32) {
                        if (n_egroups == 2 && (((s * Bp + cb) >> 5) & 1) != egroup) continue;
                        float v[32];
                        if (MERGE) {
                            float w[32];
                            tmem_ld32x2(tacc + (uint32_t)(s * G.cols_per_sub + cb),
                                        tacc + (uint32_t)(s * G.cols_per_sub + Bp + cb), v, w);
#pragma unroll
                            for (int i = 0; i < 32; ++i) v[i] += w[i];
                        } else {
                            tmem_ld32(tacc + (uint32_t)(s * G.cols_per_sub + cb), v);
                        }
                        float* dst = acc + (size_t)(s * 128 + et) * Bp + cb;
#pragma unroll
                        for (int q = 0; q < 8; ++q) red_add_v4(dst + 4 * q, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                    }
                tc_fence_before();
                release_acc(as);
                __threadfence();
                grp_sync();
                if (et == 0 && egroup == 0) flags[0] = (atomicAdd(ticket, 1) == c_last - c_first) && !(G.dbg & 4);
                grp_sync();
                if (flags[0]) {
                    __threadfence();
                    for (int s = 0; s < NSUB; ++s)
                        for (int cb = 0; cb < Bp; cb += 32) {
                            if (n_egroups == 2 && (((s * Bp + cb) >> 5) & 1) != egroup) continue;
                            float v[32];
                            float4* src = reinterpret_cast<float4*>(acc + (size_t)(s * 128 + et) * Bp + cb);
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const float4 t4 = __ldcg(src + q);
                                v[4 * q] = t4.x;
                                v[4 * q + 1] = t4.y;
                                v[4 * q + 2] = t4.z;
                                v[4 * q + 3] = t4.w;
                            }
#pragma unroll
                            for (int q = 0; q < 8; ++q) __stcg(src + q, make_float4(0.f, 0.f, 0.f, 0.f));
                            if (!(G.dbg & 8))
                                epilogue_chunk<T, EPI>(P, G.epi, row_tile(tile, s) * 128, cbase + cb, v, esm, meta, et);
                        }
                    // both groups have read the accumulator before the ticket is re-armed
                    grp_sync();
                    if (et == 0 && egroup == 0) *ticket = 0;
                    did_epi = true;
                }
            }
            if (EPI == EPI_LMHEAD && did_epi) {
                __threadfence();
                epi_sync();
                if (et == 0) flags[1] = (atomicAdd(P.lm_done, 1) == G.tiles * G.nbt - 1);
                epi_sync();
                if (flags[1]) sample_scan_publish(P, et, reinterpret_cast<int*>(esm));
            }
            if (++as == G.acc_stages) {
                as = 0;
                aphase ^= 1u;
            }
        }
    }
    if (G.split > 1) {
        // DSMEM reduce-scatter: rank r finishes the 16-column units u with u % S == r, summing
        // the S partials in rank order (deterministic), then runs the epilogue on them
        cluster_sync_all();
        if (tr && threadIdx.x == 0) tr[6] = gtimer();  // partials staged cluster-wide
        if (warp == 4 && blockIdx.y == 0) prefetch_next_gemm(G, &tmN, lane);  // overlaps the reduce below
        if (warp < 4) {
            const int et = threadIdx.x;
            const int units = NSUB * (Bp / 16);
            const int tile = blockIdx.x / G.split;
            const uint32_t base = smem_u32(smem);
            // all S*4 remote loads of a unit in flight at once (DSMEM round trips are ~200
            // cycles), then the sum in rank order; the next unit's loads are issued before this
            // unit's epilogue so their latency overlaps it
            float4 t4[kMaxSplit][4];
            auto issue = [&](int uu) {
                const uint32_t off = (uint32_t)(((size_t)uu * 512 + et) * 16);
#pragma unroll
                for (int r = 0; r < kMaxSplit; ++r)
                    if (r < G.split) {
                        const uint32_t a = mapa_shared(base + off, (uint32_t)r);
#pragma unroll
                        for (int q = 0; q < 4; ++q) t4[r][q] = ld_dsmem_f4(a + 2048u * q);
                    }
            };
            if (crank < units) issue(crank);
            for (int u = crank; u < units; u += G.split) {
                float v[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = 0.f;
#pragma unroll
                for (int r = 0; r < kMaxSplit; ++r)
                    if (r < G.split) {
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            v[4 * q] += t4[r][q].x;
                            v[4 * q + 1] += t4[r][q].y;
                            v[4 * q + 2] += t4[r][q].z;
                            v[4 * q + 3] += t4[r][q].w;
                        }
                    }
                if (u + G.split < units) issue(u + G.split);
                const int s = u / (Bp / 16), cb = (u % (Bp / 16)) * 16;
                if (tr && et == 0 && u == crank) tr[8] = gtimer();
                if (!(G.dbg & 8))
                    epilogue_chunk<T, EPI, 16>(P, G.epi, (tile * NSUB + s) * 128, cbase + cb, v, esm, meta, threadIdx.x);
                if (tr && et == 0 && u == crank) tr[9] = gtimer();
            }
        }
        if (tr && threadIdx.x == 0) tr[7] = gtimer();  // own units reduced + epilogued
        cluster_sync_all();  // peers may still be reading this CTA's partial
    }
    if (tr && threadIdx.x == 0) tr[4] = gtimer();  // epilogue warps done
    tc_fence_before();
    // pair: the leader's MMAs write the peer's TMEM and its commits / the peer's releases cross
    // CTAs -- neither CTA frees TMEM or exits before both are done
    if (PAIR) cluster_sync_all();
    else __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        if (PAIR) tmem_dealloc_pair(tmem_base, G.tmem_cols);
        else tmem_dealloc(tmem_base, G.tmem_cols);
    }
    if (threadIdx.x == 0 && G.epi.span_kind >= 0)
        span_end(P.spans, kSpanSlots, P.span_base + G.epi.layer * 8 + G.epi.span_kind);
    if (tr && threadIdx.x == 0) tr[5] = gtimer();
}

// Host-side selection of the kernel instantiation for a plan (split mode is a runtime field).
template <typename T, int EPI>
inline const void* gemm_tc_kernel_ptr_k(int nsub, bool merge, int bk, bool pair) {
    if (pair) return (const void*)gemm_tc_kernel<T, 1, true, 64, EPI, true>;
    if (merge) return nsub == 2 ? (const void*)gemm_tc_kernel<T, 2, true, 64, EPI> : (const void*)gemm_tc_kernel<T, 1, true, 64, EPI>;
    if (bk == 32)
        return nsub == 2 ? (const void*)gemm_tc_kernel<T, 2, false, 32, EPI> : (const void*)gemm_tc_kernel<T, 1, false, 32, EPI>;
    return nsub == 2 ? (const void*)gemm_tc_kernel<T, 2, false, 64, EPI> : (const void*)gemm_tc_kernel<T, 1, false, 64, EPI>;
}
template <typename T>
inline const void* gemm_tc_kernel_ptr(int nsub, bool merge, int bk, int epi, bool pair = false) {
    switch (epi) {
        case EPI_QKV: return gemm_tc_kernel_ptr_k<T, EPI_QKV>(nsub, merge, bk, pair);
        case EPI_RESID: return gemm_tc_kernel_ptr_k<T, EPI_RESID>(nsub, merge, bk, pair);
        case EPI_SWIGLU: return gemm_tc_kernel_ptr_k<T, EPI_SWIGLU>(nsub, merge, bk, pair);
        case EPI_LMHEAD: return gemm_tc_kernel_ptr_k<T, EPI_LMHEAD>(nsub, merge, bk, false);
        default: return gemm_tc_kernel_ptr_k<T, EPI_STORE>(nsub, merge, bk, pair);
    }
}

}  // namespace cvy
