// Standalone: cycles per tcgen05.mma (kind::f16, M=128, SS operands, K-major SW128) for
// several N, issued back to back by one thread into one or two accumulators.
#include "../paper_2406_00059_b200/csrc/common.cuh"
#include <cstdio>
using namespace cvy;

__global__ void __launch_bounds__(128, 1) mma_bench(int N, int n_mma, int nacc, int lbo0, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // zero the operand tiles (A: 128 x 128 B, B: N x 128 B)
    for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (warp == 0) tmem_alloc(&tslot, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tslot;
    if (warp == 1 && lane == 0) {
        const uint32_t a = smem_u32(smem), b = a + 128 * 128;
        const uint32_t idesc = idesc_bf16_f32(128, N);
        long long t0 = clock64();
        for (int i = 0; i < n_mma; ++i) {
            const int k = i & 3;
            uint64_t ad = sdesc_kmajor_sw128(a + k * 32), bd = sdesc_kmajor_sw128(b + k * 32);
            if (lbo0) { ad &= ~(0x3FFFull << 16); bd &= ~(0x3FFFull << 16); }
            umma_bf16(tbase + (uint32_t)((i % nacc) * N), ad, bd, idesc, i >= nacc ? 1u : 0u);
        }
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        out[0] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(mma_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    int Ns[] = {16, 32, 64, 128, 256};
    for (int lbo0 = 0; lbo0 < 2; ++lbo0)
    for (int nacc = 1; nacc <= 2; ++nacc)
        for (int N : Ns) {
            if (N * nacc > 512) continue;
            long long best = 1LL << 60;
            for (int rep = 0; rep < 3; ++rep) {
                mma_bench<<<1, 128, 100 * 1024>>>(N, 2000, nacc, lbo0, d);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
                long long h;
                cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
                best = h < best ? h : best;
            }
            printf("lbo0=%d nacc=%d N=%3d: %.1f cycles/MMA (%.0f MAC/cycle)\n", lbo0, nacc, N, best / 2000.0,
                   128.0 * N * 16 * 2000 / best);
        }
    // full chip: 148 CTAs concurrently
    return 0;
}
