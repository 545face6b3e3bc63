// l2_ingest_micro.cu -- L2 -> shared-memory ingest rate per SM (DESIGN.md §7.3 diagnostics).
// One CTA per SM (or `ctas` CTAs) streams 1D cp.async.bulk chunks of an L2-resident buffer into a
// shared-memory ring (`stages` x `chunk` bytes in flight), nothing consumes the data.  Reports the
// aggregate GB/s and bytes per SM clock (clock sampled with clock64 over the run).
//   mode 0: every CTA walks its own region of the buffer
//   mode 1: groups of 4 CTAs read the same chunks at the same time (the batch-tile GEMM pattern)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/l2_ingest_micro.cu -o /tmp/l2i
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 1) ingest(const uint8_t* buf, size_t buf_bytes, int chunk, int stages, int iters,
                                                 int mode, int producers, unsigned long long* clk) {
    extern __shared__ __align__(1024) uint8_t ring_all[];
    __shared__ __align__(8) uint64_t full_all[4][16];
    // `producers` warps, each with its own ring of `stages` chunks
    if ((threadIdx.x & 31) != 0 || (int)(threadIdx.x >> 5) >= producers) return;
    const int w = threadIdx.x >> 5;
    uint8_t* ring = ring_all + (size_t)w * stages * chunk;
    uint64_t* full = full_all[w];
    for (int s = 0; s < stages; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const size_t nchunks = buf_bytes / chunk;
    const size_t base = (mode == 0 ? (size_t)blockIdx.x * 977 : (size_t)(blockIdx.x / 4) * 977) + (size_t)w * 131;
    const unsigned long long c0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const int s = i % stages;
        if (i >= stages) {
            const uint32_t ph = (uint32_t)((i / stages) - 1) & 1u;
            asm volatile(
                "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                "@!p bra WAIT_%=;\n\t}" ::"r"(su32(&full[s])), "r"(ph) : "memory");
        }
        const uint8_t* src = buf + ((base + (size_t)i) % nchunks) * chunk;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(chunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(ring + (size_t)s * chunk)),
                     "l"(src), "r"(chunk), "r"(su32(&full[s]))
                     : "memory");
    }
    for (int i = iters; i < iters + stages; ++i) {
        const int s = i % stages;
        const uint32_t ph = (uint32_t)((i / stages) - 1) & 1u;
        asm volatile(
            "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra WAIT_%=;\n\t}" ::"r"(su32(&full[s])), "r"(ph) : "memory");
    }
    if (w == 0) clk[blockIdx.x] = clock64() - c0;
}

// One producer warp whose first `lanes` lanes each issue one chunk of every stage (stage = lanes
// chunks, one barrier); tests whether TMA issue serialises per thread or per warp.
__global__ void __launch_bounds__(32, 1) ingest_lanes(const uint8_t* buf, size_t buf_bytes, int chunk, int stages,
                                                       int iters, int lanes, unsigned long long* clk) {
    extern __shared__ __align__(1024) uint8_t ring[];
    __shared__ __align__(8) uint64_t full[16];
    const int lane = threadIdx.x;
    if (lane == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const size_t nchunks = buf_bytes / chunk;
    const size_t base = (size_t)blockIdx.x * 977;
    const uint32_t sb = (uint32_t)chunk * lanes;
    const unsigned long long c0 = clock64();
    for (int i = 0; i < iters + stages; ++i) {
        const int s = i % stages;
        if (i >= stages && lane == 0) {
            const uint32_t ph = (uint32_t)((i / stages) - 1) & 1u;
            asm volatile(
                "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                "@!p bra WAIT_%=;\n\t}" ::"r"(su32(&full[s])), "r"(ph) : "memory");
        }
        if (i >= iters) continue;
        if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(sb) : "memory");
        __syncwarp();
        if (lane < lanes) {
            const uint8_t* src = buf + ((base + (size_t)i * lanes + lane) % nchunks) * chunk;
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             su32(ring + (size_t)s * sb + (size_t)lane * chunk)),
                         "l"(src), "r"(chunk), "r"(su32(&full[s]))
                         : "memory");
        }
        __syncwarp();
    }
    if (lane == 0) clk[blockIdx.x] = clock64() - c0;
}

int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t buf_bytes = 48ull << 20;  // L2-resident
    uint8_t* buf;
    cudaMalloc(&buf, buf_bytes);
    cudaMemset(buf, 1, buf_bytes);
    unsigned long long* clk;
    cudaMalloc(&clk, sizeof(unsigned long long) * 1024);
    cudaFuncSetAttribute(ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct Cfg { int ctas, chunk, stages, mode, prod; };
    const Cfg cfgs[] = {{sms, 4096, 12, 0, 1},  {sms, 8192, 12, 0, 1},  {sms, 16384, 6, 0, 1}, {sms, 16384, 12, 0, 1},
                        {sms, 32768, 6, 0, 1},  {sms, 65536, 3, 0, 1},  {sms, 16384, 6, 0, 2}, {sms, 16384, 3, 0, 4},
                        {sms, 8192, 6, 0, 4},   {sms, 32768, 3, 0, 2},  {sms, 16384, 6, 1, 2}, {8, 16384, 6, 0, 2}};
    for (const Cfg& c : cfgs) {
        const int iters = 4000;
        const size_t smem = (size_t)c.chunk * c.stages * c.prod;
        ingest<<<c.ctas, 128, smem>>>(buf, buf_bytes, c.chunk, c.stages, 200, c.mode, c.prod, clk);  // warm L2
        cudaDeviceSynchronize();
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        ingest<<<c.ctas, 128, smem>>>(buf, buf_bytes, c.chunk, c.stages, iters, c.mode, c.prod, clk);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long h[1024];
        cudaMemcpy(h, clk, sizeof(unsigned long long) * c.ctas, cudaMemcpyDeviceToHost);
        double cyc = 0;
        for (int i = 0; i < c.ctas; ++i) cyc += (double)h[i];
        cyc /= c.ctas;
        const double bytes = (double)c.ctas * iters * c.chunk * c.prod;
        printf("ctas %3d chunk %5d stages %2d mode %d producers %d: %8.1f GB/s total, %6.1f GB/s per CTA, %5.1f B/clk per CTA (%.0f MHz) %s\n",
               c.ctas, c.chunk, c.stages, c.mode, c.prod, bytes / ms / 1e6, bytes / c.ctas / ms / 1e6, (double)iters * c.chunk * c.prod / cyc,
               cyc / ms / 1e3, cudaGetErrorString(cudaGetLastError()));
    }
    cudaFuncSetAttribute(ingest_lanes, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct LCfg { int chunk, stages, lanes; };
    const LCfg lc[] = {{16384, 6, 1}, {16384, 3, 2}, {16384, 3, 4}, {8192, 3, 4}, {8192, 3, 8}, {4096, 3, 16}};
    for (const LCfg& c : lc) {
        const int iters = 2000;
        const size_t smem = (size_t)c.chunk * c.stages * c.lanes;
        ingest_lanes<<<sms, 32, smem>>>(buf, buf_bytes, c.chunk, c.stages, 100, c.lanes, clk);
        cudaDeviceSynchronize();
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        ingest_lanes<<<sms, 32, smem>>>(buf, buf_bytes, c.chunk, c.stages, iters, c.lanes, clk);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = (double)sms * iters * c.chunk * c.lanes;
        printf("lanes %2d chunk %5d stages %d: %8.1f GB/s total, %6.1f GB/s per CTA %s\n", c.lanes, c.chunk, c.stages,
               bytes / ms / 1e6, bytes / sms / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
