// gemm_sm100.cuh -- skinny decode GEMM on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Y^T[n][b] = sum_k W[n][k] * X[b][k]  (swap-AB: the weight rows are the UMMA M=128 side,
// the padded batch Bp is the UMMA N side), bf16 inputs, fp32 accumulation in TMEM.
// Work split: stream-K over (tile, k-block) iterations -- exactly one persistent CTA per
// SM, each owning a contiguous range of iterations, so every SM streams the same number
// of weight bytes (HBM-bound for Bp <= ~200).  A tile finished by one CTA is epilogued
// straight from TMEM; a tile shared by several CTAs is reduced with fp32 vector atomics
// in an L2-resident workspace and epilogued by the last contributor (arrival ticket).
//
// Warp roles (192 threads): warps 0-3 epilogue (TMEM lanes 0-127), warp 4 TMA producer,
// warp 5 MMA issuer (one elected lane) and TMEM owner.
#pragma once
#include "common.cuh"
#include "epilogue.cuh"
#include "step_params.h"

namespace cvy {

struct GemmTC {
    int32_t N;          // weight rows of this GEMM (one layer)
    int32_t K;
    int32_t nsub;       // 128-row sub-tiles per tile (1 or 2)
    int32_t mma_n;      // UMMA N (<= 256)
    int32_t nbh;        // Bp / mma_n (1 or 2)
    int32_t tiles;
    int32_t kblocks;    // K / bk
    int32_t bk;         // K elements per pipeline stage: 64 (128B swizzle) or 32 (64B swizzle)
    int32_t stages;
    int32_t acc_stages; // TMEM accumulator buffers (1 or 2)
    uint32_t tmem_cols;
    int32_t w_row0;     // first row of this layer's matrix in the weight tensor map
    int32_t xplanes;    // activation planes (2: hi/lo bf16 pair, both multiplied into D)
    int32_t x_plane_rows;  // row offset of the lo plane in the activation tensor map
    float* acc;         // [tiles][nsub*128][Bp] zeroed fp32 workspace
    int32_t* tile_cnt;  // [tiles] arrival tickets (zeroed)
    EpiArgs epi;
};

constexpr int kGemmThreads = 192;
// shared-memory carve-up (host and device agree); rows are bk*2 bytes (one swizzle atom)
struct GemmSmem {
    __host__ __device__ static constexpr uint32_t w_bytes(int nsub, int bk) { return (uint32_t)nsub * 128u * bk * 2u; }
    __host__ __device__ static constexpr uint32_t x_bytes(int Bp, int bk) { return (uint32_t)Bp * bk * 2u; }
    __host__ __device__ static constexpr uint32_t stage_bytes(int nsub, int Bp, int planes, int bk) {
        return w_bytes(nsub, bk) + (uint32_t)planes * x_bytes(Bp, bk);
    }
    __host__ __device__ static constexpr uint32_t fixed_bytes(int Bp) {
        return 128u * kEsmLd * 4u      // esm
               + (uint32_t)Bp * 4u      // s_scale
               + 64u * 8u               // barriers
               + 64u;                   // tmem addr + flags
    }
};

CVY_DEV int cta_of_iter(long long i, long long T, int G) {
    long long c = (i * G) / T;
    while (c + 1 < G && ((c + 1) * T) / G <= i) ++c;
    while (c > 0 && (c * T) / G > i) --c;
    return (int)c;
}

template <typename T>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                   const __grid_constant__ StepParams P, const __grid_constant__ GemmTC G) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t stage_bytes = GemmSmem::stage_bytes(G.nsub, P.Bp, G.xplanes, G.bk);
    const uint32_t row_bytes = (uint32_t)G.bk * 2u;
    uint8_t* fixed = smem + (size_t)G.stages * stage_bytes;
    float* esm = reinterpret_cast<float*>(fixed);
    float* s_scale = esm + 128 * kEsmLd;
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_scale + P.Bp + ((P.Bp & 1) ? 1 : 0));
    uint64_t* full_bar = bars;
    uint64_t* empty_bar = bars + G.stages;
    uint64_t* tfull_bar = empty_bar + G.stages;
    uint64_t* tempty_bar = tfull_bar + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
    int* flags = reinterpret_cast<int*>(tmem_slot + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long T_iters = (long long)G.tiles * G.kblocks;
    const int Gc = gridDim.x;
    const long long it0 = ((long long)blockIdx.x * T_iters) / Gc;
    const long long it1 = ((long long)(blockIdx.x + 1) * T_iters) / Gc;

    if (warp == 4 && lane == 0) {
        tma_prefetch_desc(&tmW);
        tma_prefetch_desc(&tmX);
        for (int s = 0; s < G.stages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull_bar[s], 1);
            mbar_init(&tempty_bar[s], kEpiThreads);
        }
        fence_mbar_init();
    }
    if (warp == 5) tmem_alloc(tmem_slot, G.tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_launch_dependents();

    if (warp == 4) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            const uint64_t pol_w = policy_evict_first();
            const uint64_t pol_x = policy_evict_last();
            const uint32_t wb = GemmSmem::w_bytes(G.nsub, G.bk);
            const int rows_per_tile = 128 * G.nsub;
            // prologue: weights do not depend on the previous kernel -> issue them before
            // the grid-dependency wait so the weight stream starts under the previous tail
            const long long n_it = it1 - it0;
            const int pre = (int)(n_it < G.stages ? n_it : G.stages);
            for (int i = 0; i < pre; ++i) {
                const long long it = it0 + i;
                const int tile = (int)(it / G.kblocks), kb = (int)(it % G.kblocks);
                uint8_t* sw = smem + (size_t)i * stage_bytes;
                mbar_arrive_expect_tx(&full_bar[i], stage_bytes);
                tma_load_2d(sw, &tmW, &full_bar[i], kb * G.bk, G.w_row0 + tile * rows_per_tile, pol_w);
            }
            pdl_wait();
            for (int i = 0; i < pre; ++i) {
                const long long it = it0 + i;
                const int kb = (int)(it % G.kblocks);
                uint8_t* sx = smem + (size_t)i * stage_bytes + wb;
                for (int pl = 0; pl < G.xplanes; ++pl)
                    for (int h = 0; h < G.nbh; ++h)
                        tma_load_2d(sx + (size_t)(pl * P.Bp + h * G.mma_n) * row_bytes, &tmX, &full_bar[i], kb * G.bk,
                                    pl * G.x_plane_rows + h * G.mma_n, pol_x);
            }
            int stage = pre % G.stages;
            uint32_t phase = (pre == G.stages) ? 1u : 0u;
            for (long long it = it0 + pre; it < it1; ++it) {
                const int tile = (int)(it / G.kblocks), kb = (int)(it % G.kblocks);
                mbar_wait(&empty_bar[stage], phase ^ 1u);
                uint8_t* sw = smem + (size_t)stage * stage_bytes;
                mbar_arrive_expect_tx(&full_bar[stage], stage_bytes);
                tma_load_2d(sw, &tmW, &full_bar[stage], kb * G.bk, G.w_row0 + tile * rows_per_tile, pol_w);
                for (int pl = 0; pl < G.xplanes; ++pl)
                    for (int h = 0; h < G.nbh; ++h)
                        tma_load_2d(sw + wb + (size_t)(pl * P.Bp + h * G.mma_n) * row_bytes, &tmX, &full_bar[stage],
                                    kb * G.bk, pl * G.x_plane_rows + h * G.mma_n, pol_x);
                if (++stage == G.stages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
    } else if (warp == 5) {
        // ===================== MMA issuer =====================
        const uint32_t idesc = idesc_bf16_f32(128, (uint32_t)G.mma_n);
        const uint32_t wb = GemmSmem::w_bytes(G.nsub, G.bk);
        const bool sw128 = G.bk == 64;
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
            const uint32_t dcol = tmem_base + (uint32_t)(as * G.nsub * P.Bp);
            for (; it < seg_end; ++it) {
                mbar_wait(&full_bar[stage], phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t sw = smem_u32(smem + (size_t)stage * stage_bytes);
                    const uint32_t sx = sw + wb;
                    const bool first = (it == (long long)tile * G.kblocks) || (it == it0);
                    for (int k = 0; k < G.bk / 16; ++k) {
                        for (int s = 0; s < G.nsub; ++s) {
                            const uint32_t aaddr = sw + (uint32_t)s * 128u * row_bytes + (uint32_t)k * 32u;
                            const uint64_t ad = sw128 ? sdesc_kmajor_sw128(aaddr) : sdesc_kmajor_sw64(aaddr);
                            for (int h = 0; h < G.nbh; ++h)
                                for (int pl = 0; pl < G.xplanes; ++pl) {
                                    const uint32_t baddr =
                                        sx + (uint32_t)(pl * P.Bp + h * G.mma_n) * row_bytes + (uint32_t)k * 32u;
                                    const uint64_t bd = sw128 ? sdesc_kmajor_sw128(baddr) : sdesc_kmajor_sw64(baddr);
                                    umma_bf16(dcol + (uint32_t)(s * P.Bp + h * G.mma_n), ad, bd, idesc,
                                              (first && k == 0 && pl == 0) ? 0u : 1u);
                                }
                        }
                    }
                    umma_commit(&empty_bar[stage]);
                }
                __syncwarp();
                if (++stage == G.stages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
            if (lane == 0) umma_commit(&tfull_bar[as]);
            __syncwarp();
            if (++as == G.acc_stages) {
                as = 0;
                aphase ^= 1u;
            }
        }
    } else {
        // ===================== epilogue (warps 0-3) =====================
        const int et = threadIdx.x;  // 0..127 == TMEM lane == tile row
        const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
        bool scales_ready = false;
        int as = 0;
        uint32_t aphase = 0;
        long long it = it0;
        while (it < it1) {
            const int tile = (int)(it / G.kblocks);
            const long long tb = (long long)tile * G.kblocks, te = tb + G.kblocks;
            const long long seg_end = min(it1, te);
            const int ncontrib = cta_of_iter(te - 1, T_iters, Gc) - cta_of_iter(tb, T_iters, Gc) + 1;
            it = seg_end;
            if (!scales_ready) {
                pdl_wait();
                if (G.epi.kind != EPI_RESID && G.epi.kind != EPI_STORE) compute_row_scales(P, s_scale, et);
                epi_sync();
                scales_ready = true;
            }
            mbar_wait(&tfull_bar[as], aphase);
            tc_fence_after();
            const uint32_t tacc = tmem_base + lane_off + (uint32_t)(as * G.nsub * P.Bp);
            float* accw = G.acc + (size_t)tile * (G.nsub * 128) * P.Bp;
            bool do_epi = true;
            bool from_tmem = true;
            if (ncontrib > 1) {
                // contribute this CTA's partial sums (fp32 vector atomics, L2-resident)
                for (int s = 0; s < G.nsub; ++s)
                    for (int cb = 0; cb < P.Bp; cb += 32) {
                        float v[32];
                        tmem_ld32(tacc + (uint32_t)(s * P.Bp + cb), v);
                        float4* dst = reinterpret_cast<float4*>(accw + (size_t)(s * 128 + et) * P.Bp + cb);
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            atomicAdd(dst + q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
                    }
                tc_fence_before();
                mbar_arrive(&tempty_bar[as]);
                __threadfence();
                epi_sync();
                if (et == 0) flags[0] = (atomicAdd(&G.tile_cnt[tile], 1) == ncontrib - 1);
                epi_sync();
                do_epi = flags[0] != 0;
                from_tmem = false;
                if (do_epi) __threadfence();
            }
            if (do_epi) {
                for (int s = 0; s < G.nsub; ++s) {
                    const int n0 = (tile * G.nsub + s) * 128;
                    for (int cb = 0; cb < P.Bp; cb += 32) {
                        float v[32];
                        if (from_tmem) {
                            tmem_ld32(tacc + (uint32_t)(s * P.Bp + cb), v);
                        } else {
                            float4* src = reinterpret_cast<float4*>(accw + (size_t)(s * 128 + et) * P.Bp + cb);
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                float4 t4 = __ldcg(src + q);
                                v[4 * q] = t4.x;
                                v[4 * q + 1] = t4.y;
                                v[4 * q + 2] = t4.z;
                                v[4 * q + 3] = t4.w;
                                __stcg(src + q, make_float4(0.f, 0.f, 0.f, 0.f));
                            }
                        }
                        epilogue_chunk<T>(P, G.epi, n0, cb, v, esm, s_scale, et);
                    }
                }
                if (from_tmem) {
                    tc_fence_before();
                    mbar_arrive(&tempty_bar[as]);
                } else if (et == 0) {
                    G.tile_cnt[tile] = 0;
                }
                if (G.epi.kind == EPI_LMHEAD) {
                    __threadfence();
                    epi_sync();
                    if (et == 0) flags[1] = (atomicAdd(P.lm_done, 1) == G.tiles - 1);
                    epi_sync();
                    if (flags[1]) sample_scan_publish(P, et, reinterpret_cast<int*>(esm));
                }
            }
            if (++as == G.acc_stages) {
                as = 0;
                aphase ^= 1u;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc(tmem_base, G.tmem_cols);
    }
}

}  // namespace cvy
