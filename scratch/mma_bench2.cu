#include "../paper_2406_00059_b200/csrc/common.cuh"
#include <cstdio>
using namespace cvy;

// all lanes execute; one elected lane issues; descriptors passed as 64-bit values
CVY_DEV void umma_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}

template <int V>
__global__ void __launch_bounds__(128, 1) mma_bench(int N, int n_iter, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (warp == 0) tmem_alloc(&tslot, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tslot;
    if (warp == 1) {
        const uint32_t a = smem_u32(smem), b = a + 128 * 128;
        const uint32_t idesc = idesc_bf16_f32(128, N);
        const uint64_t ad0 = sdesc_kmajor_sw128(a), bd0 = sdesc_kmajor_sw128(b);
        long long t0 = clock64();
        if (V == 2) {
            if (lane == 0) {
                for (int i = 0; i < n_iter; ++i) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        umma_bf16(tbase, ad0 + 2 * k, bd0 + 2 * k, idesc, (i | k) ? 1u : 0u);
                }
            }
        } else if (V == 3) {
            for (int i = 0; i < n_iter; ++i) {
#pragma unroll
                for (int k = 0; k < 4; ++k) umma_elect(tbase, ad0 + 2 * k, bd0 + 2 * k, idesc, (i | k) ? 1u : 0u);
            }
        }
        __syncwarp();
        if (lane == 0) {
            umma_commit(&bar);
            mbar_wait(&bar, 0);
            long long t1 = clock64();
            out[0] = t1 - t0;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tbase, 512); }
}

template <int V> void run(const char* name) {
    long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(mma_bench<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    int Ns[] = {32, 64, 128, 256};
    for (int N : Ns) {
        long long best = 1LL << 60;
        for (int rep = 0; rep < 3; ++rep) {
            mma_bench<V><<<1, 128, 100 * 1024>>>(N, 500, d);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
            long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            best = h < best ? h : best;
        }
        printf("%s N=%3d: %.1f cycles/MMA (%.0f MAC/cycle)\n", name, N, best / 2000.0, 128.0 * N * 16 * 2000 / best);
    }
}
int main() { run<2>("lane0-unrolled-precomp"); run<3>("warp-elect-unrolled"); return 0; }
