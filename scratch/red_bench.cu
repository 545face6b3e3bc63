// Throughput of fp32 vector reductions into L2 (red.global.add.v4.f32) vs plain stores,
// 148 CTAs x 128 threads, each CTA adding a 128x64 fp32 tile (32 KB) into one of `tiles` slots.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void red_kernel(float* acc, int tiles, int mode) {
    const int tile = blockIdx.x % tiles;
    float* dst = acc + (size_t)tile * 128 * 64 + threadIdx.x * 64;
    float v[64];
    for (int i = 0; i < 64; ++i) v[i] = threadIdx.x * 0.001f + i;
    if (mode == 0) {
        for (int q = 0; q < 16; ++q)
            asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(dst + 4 * q), "f"(v[4 * q]), "f"(v[4 * q + 1]),
                         "f"(v[4 * q + 2]), "f"(v[4 * q + 3]) : "memory");
    } else if (mode == 1) {
        for (int q = 0; q < 16; ++q) atomicAdd(reinterpret_cast<float4*>(dst) + q, make_float4(v[4*q], v[4*q+1], v[4*q+2], v[4*q+3]));
    } else {
        float* mine = acc + (size_t)(1024 + blockIdx.x) * 128 * 64 + threadIdx.x * 64;
        for (int q = 0; q < 16; ++q) __stcg(reinterpret_cast<float4*>(mine) + q, make_float4(v[4*q], v[4*q+1], v[4*q+2], v[4*q+3]));
    }
}
int main() {
    float* acc; cudaMalloc(&acc, sizeof(float) * 2048 * 128 * 64);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const char* names[] = {"red.v4", "atomicAdd(float4)", "store"};
    for (int mode = 0; mode < 3; ++mode)
        for (int tiles : {16, 32, 148}) {
            red_kernel<<<148, 128>>>(acc, tiles, mode);
            cudaDeviceSynchronize();
            cudaEventRecord(a);
            for (int i = 0; i < 20; ++i) red_kernel<<<148, 128>>>(acc, tiles, mode);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("%-18s tiles=%3d: %.2f us per launch (%.0f GB/s)\n", names[mode], tiles, ms * 1000 / 20,
                   148.0 * 32768 / (ms / 20 * 1e-3) / 1e9);
        }
    // empty kernel launch cost
    cudaEventRecord(a);
    for (int i = 0; i < 20; ++i) red_kernel<<<148, 128>>>(acc, 1, 9);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("empty: %.2f us\n", ms * 1000 / 20);
    return 0;
}
