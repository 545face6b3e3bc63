// tma_read_micro.cu -- HBM read bandwidth by transfer mechanism (DESIGN.md §7.2 diagnostics).
// Reads a 2 GiB bf16 [rows][128] buffer (256 B rows, > L2) once per rep with one CTA per SM:
//   tma  : 2D TMA boxes of {64 cols, box_rows} with 128B swizzle (the KV / weight load shape),
//          two boxes per row block, S-stage ring of stage_kb each (producer lane -> consumer)
//   bulk : 1D cp.async.bulk of chunk bytes
//   ldg  : plain 16-byte loads, grid 148 x 4, 512 threads
// "scatter" visits the 16-row (4 KB) blocks in a fixed pseudo-random order (the paged-KV pattern).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/tma_read_micro.cu -lcuda -o /tmp/trm
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cudaTypedefs.h>
#include "../paper_2406_00059_b200/csrc/common.cuh"

using namespace cvy;

__device__ __forceinline__ uint32_t blk_of(uint32_t i, uint32_t nblk, bool scatter) {
    // odd multiplier mod a power of two is a bijection
    return scatter ? (uint32_t)(((uint64_t)i * 2654435761ull) & (nblk - 1)) : i;
}

__global__ void __launch_bounds__(64, 1) rd_tma(const __grid_constant__ CUtensorMap tm, uint32_t nblk16, int box_rows,
                                                 int stages, int stage_bytes, int scatter, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[16], empty[16];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int box_bytes = box_rows * 128;
    const int per_stage = stage_bytes / box_bytes;  // boxes per stage
    const uint32_t blk_rows = (uint32_t)box_rows;   // rows per "block" of work (2 boxes: cols 0, 64)
    const uint32_t nblk = nblk16 * 16u / blk_rows;
    const uint32_t b0 = (uint64_t)nblk * blockIdx.x / gridDim.x, b1 = (uint64_t)nblk * (blockIdx.x + 1) / gridDim.x;
    const uint32_t nbox = (b1 - b0) * 2u;
    const uint32_t nst = (nbox + per_stage - 1) / per_stage;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int s = 0;
            uint32_t ph = 0, bx = 0;
            for (uint32_t t = 0; t < nst; ++t) {
                const uint32_t n = min((uint32_t)per_stage, nbox - bx);
                mbar_wait(&empty[s], ph ^ 1u);
                mbar_arrive_expect_tx(&full[s], n * box_bytes);
                for (uint32_t j = 0; j < n; ++j, ++bx) {
                    const uint32_t blk = blk_of(b0 + bx / 2, nblk, scatter != 0 && box_rows == 16);
                    tma_load_2d(ring + (size_t)s * stage_bytes + (size_t)j * box_bytes, &tm, &full[s], (bx & 1) * 64,
                                (int)(blk * blk_rows), pol);
                }
                if (++s == stages) { s = 0; ph ^= 1u; }
            }
        }
    } else if (lane == 0) {
        int s = 0;
        uint32_t ph = 0;
        unsigned long long acc = 0;
        for (uint32_t t = 0; t < nst; ++t) {
            mbar_wait(&full[s], ph);
            acc += *reinterpret_cast<volatile uint32_t*>(ring + (size_t)s * stage_bytes);
            mbar_arrive(&empty[s]);
            if (++s == stages) { s = 0; ph ^= 1u; }
        }
        if (acc == 0x123456789ull) *sink = acc;
    }
}

__global__ void __launch_bounds__(64, 1) rd_bulk(const uint8_t* src, size_t bytes, int chunk, int stages, int stage_bytes,
                                                  int scatter, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[16], empty[16];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t nch = (uint32_t)(bytes / chunk);
    const uint32_t c0 = (uint64_t)nch * blockIdx.x / gridDim.x, c1 = (uint64_t)nch * (blockIdx.x + 1) / gridDim.x;
    const int per_stage = stage_bytes / chunk;
    const uint32_t nst = (c1 - c0 + per_stage - 1) / per_stage;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0, c = c0;
            for (uint32_t t = 0; t < nst; ++t) {
                const uint32_t n = min((uint32_t)per_stage, c1 - c);
                mbar_wait(&empty[s], ph ^ 1u);
                mbar_arrive_expect_tx(&full[s], n * chunk);
                for (uint32_t j = 0; j < n; ++j, ++c) {
                    const uint32_t cc = blk_of(c, nch, scatter != 0);
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            smem_u32(ring + (size_t)s * stage_bytes + (size_t)j * chunk)),
                        "l"(src + (size_t)cc * chunk), "r"(chunk), "r"(smem_u32(&full[s]))
                        : "memory");
                }
                if (++s == stages) { s = 0; ph ^= 1u; }
            }
        }
    } else if (lane == 0) {
        int s = 0;
        uint32_t ph = 0;
        unsigned long long acc = 0;
        for (uint32_t t = 0; t < nst; ++t) {
            mbar_wait(&full[s], ph);
            acc += *reinterpret_cast<volatile uint32_t*>(ring + (size_t)s * stage_bytes);
            mbar_arrive(&empty[s]);
            if (++s == stages) { s = 0; ph ^= 1u; }
        }
        if (acc == 0x123456789ull) *sink = acc;
    }
}

// GEMM-shaped stream: per stage, 2 boxes of 128 rows x 64 cols (32 KB, this CTA's weight rows,
// k-block kb) + 1 box of 128 rows of a shared 128-row x K "activation" matrix (16 KB, the same
// for every CTA at the same kb).  rot != 0 starts CTA c at k-block (c * rot) % KB.
__global__ void __launch_bounds__(64, 1) rd_gemmlike(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap tx,
                                                      int KB, int stages, int rot, int with_x, int layout,
                                                      unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[16], empty[16];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int SB = 48 * 1024;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int s = 0;
            uint32_t ph = 0;
            for (int i = 0; i < KB; ++i) {
                const int kb = (i + blockIdx.x * rot) % KB;
                mbar_wait(&empty[s], ph ^ 1u);
                mbar_arrive_expect_tx(&full[s], with_x ? SB : 32768);
                uint8_t* d = ring + (size_t)s * SB;
                if (layout == 0) {  // row-major [N][K]: 128 rows x 128 B per box
                    tma_load_2d(d, &tw, &full[s], kb * 64, blockIdx.x * 256, pol);
                    tma_load_2d(d + 16384, &tw, &full[s], kb * 64, blockIdx.x * 256 + 128, pol);
                } else if (layout == 1) {  // row-major, one 128-row sub x two adjacent k-blocks
                    const int sub = i & 1, kp = (i >> 1) * 2;
                    tma_load_2d(d, &tw, &full[s], kp * 64, blockIdx.x * 256 + sub * 128, pol);
                    tma_load_2d(d + 16384, &tw, &full[s], kp * 64 + 64, blockIdx.x * 256 + sub * 128, pol);
                } else {  // tile-major [N/128][K/64][128][64]: each box is 16 contiguous KB
                    tma_load_2d(d, &tw, &full[s], 0, ((blockIdx.x * 2 + 0) * KB + kb) * 128, pol);
                    tma_load_2d(d + 16384, &tw, &full[s], 0, ((blockIdx.x * 2 + 1) * KB + kb) * 128, pol);
                }
                if (with_x) tma_load_2d(d + 32768, &tx, &full[s], kb * 64, 0, policy_evict_last());
                if (++s == stages) { s = 0; ph ^= 1u; }
            }
        }
    } else if (lane == 0) {
        int s = 0;
        uint32_t ph = 0;
        unsigned long long acc = 0;
        for (int i = 0; i < KB; ++i) {
            mbar_wait(&full[s], ph);
            acc += *reinterpret_cast<volatile uint32_t*>(ring + (size_t)s * SB);
            mbar_arrive(&empty[s]);
            if (++s == stages) { s = 0; ph ^= 1u; }
        }
        if (acc == 0x123456789ull) *sink = acc;
    }
}

__global__ void rd_ldg(const int4* src, size_t n16, unsigned long long* sink) {
    unsigned long long acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        int4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride),
             d = __ldcs(src + i + 3 * stride);
        acc += (unsigned)(a.x ^ b.y ^ c.z ^ d.w);
    }
    for (; i < n16; i += stride) acc += (unsigned)__ldcs(src + i).x;
    if (acc == 0x123456789ull) *sink = acc;
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

int main() {
    const size_t bytes = 2ull << 30, rows = bytes / 256;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    uint8_t* buf;
    unsigned long long* sink;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&sink, 8);
    cudaMemset(buf, 1, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char* name, auto&& launch) {
        launch();
        cudaDeviceSynchronize();
        const int reps = 5;
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) launch();
        cudaEventRecord(e1);
        cudaError_t err = cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-40s %8.1f GB/s  %s\n", name, bytes * reps / (ms * 1e-3) / 1e9, cudaGetErrorString(err));
        fflush(stdout);
    };
    const int box_rows_list[] = {16, 64, 128, 256};
    for (int br : box_rows_list) {
        CUtensorMap tm;
        cuuint64_t gdim[2] = {128, rows}, gstride[1] = {256};
        cuuint32_t box[2] = {64, (cuuint32_t)br}, es[2] = {1, 1};
        if (enc()(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS) {
            printf("encode failed %d\n", br);
            continue;
        }
        const int cfg[][2] = {{2, 64}, {3, 64}, {6, 32}, {4, 48}};
        for (auto& c : cfg) {
            const int st = c[0], sb = c[1] * 1024;
            if (sb < br * 128) continue;
            const size_t smem = (size_t)st * sb + 1024;
            cudaFuncSetAttribute(rd_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            for (int sc = 0; sc < (br == 16 ? 2 : 1); ++sc) {
                char name[96];
                snprintf(name, sizeof name, "tma box%dx64 %dx%dKB%s", br, st, c[1], sc ? " scatter" : "");
                timeit(name, [&] { rd_tma<<<nsm, 64, smem>>>(tm, (uint32_t)(rows / 16), br, st, sb, sc, sink); });
            }
        }
    }
    // per-SM ceiling: the same stream on fewer CTAs (one per SM)
    {
        CUtensorMap tm;
        cuuint64_t gdim[2] = {128, rows}, gstride[1] = {256};
        cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
        enc()(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int cfg[][2] = {{3, 64}, {6, 32}, {12, 16}};
        for (auto& c : cfg) {
            const int st = c[0], sb = c[1] * 1024;
            const size_t smem = (size_t)st * sb + 1024;
            cudaFuncSetAttribute(rd_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            for (int grid : {148, 128, 112, 96, 74}) {
                char name[96];
                snprintf(name, sizeof name, "tma box128x64 %dx%dKB grid %d", st, c[1], grid);
                timeit(name, [&] { rd_tma<<<grid, 64, smem>>>(tm, (uint32_t)(rows / 16), 128, st, sb, 0, sink); });
            }
        }
    }
    // gate/up-shaped: 112 CTAs x 256 weight rows x K = 4096 (bf16) = 235 MB, + shared X (128 x 4096)
    {
        const int K = 4096, KB = K / 64, NR = 28672;
        CUtensorMap tw, tx;
        cuuint64_t gw[2] = {(cuuint64_t)K, (cuuint64_t)NR}, sw[1] = {(cuuint64_t)K * 2};
        cuuint64_t gx[2] = {(cuuint64_t)K, 128}, sx[1] = {(cuuint64_t)K * 2};
        cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
        enc()(&tw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, gw, sw, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        CUtensorMap tt;  // tile-major view of the same bytes: rows of 64 elements
        cuuint64_t gt[2] = {64, (cuuint64_t)NR * K / 64}, st_[1] = {128};
        enc()(&tt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, gt, st_, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        enc()(&tx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf + (size_t)NR * K * 2, gx, sx, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const size_t wbytes = (size_t)NR * K * 2;
        for (int st : {3, 4}) {
            const size_t smem = (size_t)st * 48 * 1024 + 1024;
            cudaFuncSetAttribute(rd_gemmlike, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            for (int lay = 0; lay < 3; ++lay)
            for (int wx = 0; wx < 2; ++wx)
                for (int rot : {0, 1}) {
                    if (!wx && rot) continue;
                    const int reps = 10;
                    rd_gemmlike<<<112, 64, smem>>>(lay == 2 ? tt : tw, tx, KB, st, rot, wx, lay, sink);
                    cudaDeviceSynchronize();
                    cudaEventRecord(e0);
                    for (int r = 0; r < reps; ++r) rd_gemmlike<<<112, 64, smem>>>(lay == 2 ? tt : tw, tx, KB, st, rot, wx, lay, sink);
                    cudaEventRecord(e1);
                    cudaError_t err = cudaEventSynchronize(e1);
                    float ms = 0;
                    cudaEventElapsedTime(&ms, e0, e1);
                    printf("gemmlike 112 CTAs layout %d %d x 48KB x=%d rot=%d: %.1f us/launch, weights %.1f GB/s  %s\n",
                           lay, st, wx, rot, ms * 1e3 / reps, wbytes * reps / (ms * 1e-3) / 1e9, cudaGetErrorString(err));
                }
        }
    }
    const int chunks[] = {4096, 8192, 16384};
    for (int ch : chunks) {
        const int cfg[][2] = {{3, 64}, {6, 32}};
        for (auto& c : cfg) {
            const int st = c[0], sb = c[1] * 1024;
            const size_t smem = (size_t)st * sb + 1024;
            cudaFuncSetAttribute(rd_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            for (int sc = 0; sc < 2; ++sc) {
                char name[96];
                snprintf(name, sizeof name, "bulk %dB %dx%dKB%s", ch, st, c[1], sc ? " scatter" : "");
                timeit(name, [&] { rd_bulk<<<nsm, 64, smem>>>(buf, bytes, ch, st, sb, sc, sink); });
            }
        }
    }
    for (int k : {2, 4, 8}) {
        char name[64];
        snprintf(name, sizeof name, "ldg int4 grid %dx%d x512", nsm, k);
        timeit(name, [&] { rd_ldg<<<nsm * k, 512>>>((const int4*)buf, bytes / 16, sink); });
    }
    return 0;
}
