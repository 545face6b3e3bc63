// kernels.cuh -- non-GEMM kernels of the decode step: synthetic init, slot patches,
// embedding gather (+ first RMSNorm input), paged-KV GQA decode attention (split-KV +
// merge), and the SIMT fp32 GEMM used by the fp32 parity path.
#pragma once
#include "common.cuh"
#include "epilogue.cuh"
#include "step_params.h"

namespace cvy {

// ------------------------------------------------------------------ synthetic init
// w[i] = a*(2U-1) rounded to fp32 then to the storage dtype; rows of tensor `tid` are
// written at dst_row0 + row (optionally with the gate/up 64-row interleave).
template <typename T>
__global__ void init_hash_kernel(T* dst, uint64_t seed, uint64_t tid, int64_t rows, int64_t cols, double a,
                                 int interleave, int which /*0 gate 1 up*/) {
    int64_t n = rows * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float v = hash_uniform_f32(seed, tid, (uint64_t)i, a);
        int64_t r = i / cols, c = i % cols;
        int64_t rr = r;
        if (interleave) rr = (r / 64) * 128 + which * 64 + (r % 64);
        dst[rr * cols + c] = DT<T>::from_f(v);
    }
}

__global__ void fill_f32_kernel(float* dst, int64_t n, float v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = v;
}

// Synthetic KV prefix: post-RoPE K/V from the counter hash (std 1), DESIGN.md "Input recipe".
template <typename T>
__global__ void synth_prefix_kernel(T* kv_pool, const int32_t* pages, int n_pages_total, int L, int Hkv,
                                    int hd, int prefix_len, uint64_t synth_seed) {
    // one thread per element of [L][prefix][2][Hkv][hd]
    int64_t per_layer = (int64_t)prefix_len * 2 * Hkv * hd;
    int64_t n = per_layer * L;
    const double a = 1.7320508075688772;  // sqrt(3)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int l = (int)(i / per_layer);
        int64_t idx = i % per_layer;  // ((pos*2 + c)*Hkv + g)*hd + e
        int e = (int)(idx % hd);
        int64_t t = idx / hd;
        int g = (int)(t % Hkv);
        t /= Hkv;
        int c = (int)(t % 2);
        int pos = (int)(t / 2);
        uint64_t tid = (1ULL << 62) ^ (synth_seed * (uint64_t)L + (uint64_t)l);
        float v = hash_uniform_f32(0, tid, (uint64_t)idx, a);
        int page = pages[pos / kPageTokens];
        size_t off = ((((size_t)l * n_pages_total + page) * Hkv + g) * 2 + c) * (size_t)(kPageTokens * hd) +
                     (size_t)(pos % kPageTokens) * hd + e;
        kv_pool[off] = DT<T>::from_f(v);
    }
}

// ------------------------------------------------------------------ slot patches
__global__ void apply_patches_kernel(SlotDev* slots, const Patch* patches, int n, SlotStatus* status) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int i = 0; i < n; ++i) {
        const Patch& p = patches[i];
        SlotDev& s = slots[p.slot];
        switch (p.kind) {
            case PATCH_SUBMIT:
                s.req_id = p.req_id;
                s.active = 1;
                s.tool = p.tool;
                s.pos = p.pos;
                s.cur_tok = p.cur_tok;
                s.in_idx = p.in_idx;
                s.in_len = p.in_len;
                s.gen = 0;
                s.max_new = p.max_new;
                s.force_len = p.force_len;
                s.round = 0;
                s.seq = 0;
                s.stream_len = s.seg_start = 0;
                s.win = 0;
                s.depth = s.in_str = s.esc = 0;
                s.cancel = 0;
                s.max_pos = p.max_pos;
                s.tool_set = p.tool_set;
                s.set_max_seg = p.set_max_seg;
                s.region = -1;
                status[p.slot].state = 0;
                status[p.slot].round = 0;
                status[p.slot].gen = 0;
                break;
            case PATCH_INJECT:
                if (p.set_pos) {  // observation prefilled (NEXT-1): resume at its last token
                    s.pos = p.pos;
                    s.cur_tok = p.cur_tok;
                }
                s.active = 1;
                s.in_idx = 0;
                s.in_len = p.in_len;
                s.gen = 0;
                s.max_new = p.max_new;
                s.force_len = p.force_len;
                s.round += 1;
                s.stream_len = s.seg_start = 0;
                s.win = 0;
                s.depth = s.in_str = s.esc = 0;
                s.cancel = 0;
                s.max_pos = p.max_pos;
                s.region = -1;
                status[p.slot].state = 0;
                status[p.slot].round = s.round;
                status[p.slot].gen = 0;
                break;
            case PATCH_CANCEL:
                if (s.active) s.cancel = 1;
                break;
            case PATCH_RELEASE:
                s.active = 0;
                s.cancel = 0;
                status[p.slot].state = 3;
                break;
        }
    }
}

// ------------------------------------------------------------------ embedding gather
// x_b = E[cur_tok_b] (fp32 residual); act_b = x_b * w_attn[0] in the model dtype; ssq
// partial sums of x_b^2 per 128-wide block (the RMS scale is applied in the QKV epilogue).
template <typename T>
__global__ void __launch_bounds__(128) embed_kernel(const __grid_constant__ StepParams P) {
    pdl_launch_dependents();
    pdl_wait();
    if (threadIdx.x == 0) span_begin(P.spans, P.span_base);
    const int b = blockIdx.x;
    int tok;
    if (P.row_tok) {
        tok = P.row_pos[b] >= 0 ? P.row_tok[b] : 0;
    } else {
        const SlotDev& s = P.slots[b];
        tok = s.active ? s.cur_tok : 0;
    }
    const T* E = reinterpret_cast<const T*>(P.embed) + (size_t)tok * P.d;
    T* act = reinterpret_cast<T*>(P.act) + (size_t)b * P.act_ld;
    const float* nw = P.L > 0 ? P.attn_norm : P.final_norm;  // L == 0: straight to the LM head
    // thread t owns element blk * 128 + t of every 128-block; the embedding row is read with all
    // loads in flight (it comes from HBM: a dependent load per block made this a latency chain),
    // and the per-block sums of squares keep their reduction tree (warp xor, then 4 warps)
    constexpr int kMaxBlk = 64;  // d <= 8192
    __shared__ float red[kMaxBlk][4];
    const int nblk = P.d / 128;
    for (int blk0 = 0; blk0 < nblk; blk0 += 16) {
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
            v[j] = blk0 + j < nblk ? DT<T>::to_f(E[(blk0 + j) * 128 + threadIdx.x]) : 0.f;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int blk = blk0 + j;
            if (blk >= nblk) break;
            const int i = blk * 128 + threadIdx.x;
            P.x[(size_t)b * P.d + i] = v[j];
            DT<T>::store_act(act + i, (size_t)P.act_plane, v[j] * nw[i]);
            float sq = v[j] * v[j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
            if ((threadIdx.x & 31) == 0 && blk < kMaxBlk) red[blk][threadIdx.x >> 5] = sq;
        }
    }
    __syncthreads();
    for (int blk = threadIdx.x; blk < nblk && blk < kMaxBlk; blk += blockDim.x)
        P.ssq[(size_t)blk * P.Bmax + b] = (red[blk][0] + red[blk][1]) + (red[blk][2] + red[blk][3]);
    if (threadIdx.x == 0) span_end(P.spans, kSpanSlots, P.span_base);
}

// ------------------------------------------------------------------ paged GQA decode attention
// One CTA per (kv head g, slot b, split): the G = H/Hkv query heads of group g attend over
// keys [0, pos_b] (the current token's K/V were appended by the QKV epilogue).  Phase 1:
// one thread per key computes the G scores (K row read once, reused by the G heads).
// Phase 2: online-softmax update.  Phase 3: thread t accumulates dims (t, t+128, ...) of
// the G heads from V (each V element read once, reused by the G heads).
constexpr int kAttnThreads = 128;
constexpr int kAttnMaxG = 8;

template <typename T>
__global__ void __launch_bounds__(kAttnThreads) attention_kernel(const __grid_constant__ StepParams P, int layer) {
    pdl_launch_dependents();
    const int g = blockIdx.x, b = blockIdx.y, split = blockIdx.z;
    const int G = P.H / P.Hkv, hd = P.hd;
    extern __shared__ float asmem[];
    float* qs = asmem;                          // [G][hd]
    float* sc = qs + G * hd;                    // [G][128]
    float* mrow = sc + G * kAttnThreads;        // [G] running max
    float* lrow = mrow + kAttnMaxG;             // [G] running sum
    float* alpha = lrow + kAttnMaxG;            // [G] rescale of this chunk
    float* red = alpha + kAttnMaxG;             // [4][G]
    pdl_wait();
    const int nsplit = P.attn_splits;
    const int tid = threadIdx.x;
    const int nkeys = row_nkeys(P, b);
    const int per = ((nkeys + nsplit - 1) / nsplit + kAttnThreads - 1) / kAttnThreads * kAttnThreads;
    const int k_begin = split * per, k_end = min(nkeys, k_begin + per);
    const float qscale = rsqrtf((float)hd) * 1.4426950408889634f;  // log2(e)/sqrt(hd)
    for (int i = tid; i < G * hd; i += kAttnThreads)
        qs[i] = P.q[(size_t)b * (P.H * hd) + (size_t)(g * G) * hd + i] * qscale;
    if (tid < G) {
        mrow[tid] = -INFINITY;
        lrow[tid] = 0.f;
    }
    __syncthreads();
    const T* kv = reinterpret_cast<const T*>(P.kv_pool);
    const int32_t* pt = P.page_table + (size_t)row_slot_of(P, b) * P.max_pages;
    const size_t page_stride = (size_t)2 * P.Hkv * kPageTokens * hd;
    const size_t layer_base = (size_t)layer * P.n_pages * page_stride;
    const int nout = (G * hd + kAttnThreads - 1) / kAttnThreads;  // outputs per thread (<= 8)
    float acc[kAttnMaxG];
#pragma unroll
    for (int j = 0; j < kAttnMaxG; ++j) acc[j] = 0.f;
    for (int k0 = k_begin; k0 < k_end; k0 += kAttnThreads) {
        // phase 1: scores
        const int key = k0 + tid;
        float sv[kAttnMaxG];
        if (key < k_end) {
            const int page = pt[key / kPageTokens];
            const T* krow = kv + layer_base + (size_t)page * page_stride + ((size_t)g * 2 + 0) * kPageTokens * hd +
                            (size_t)(key % kPageTokens) * hd;
#pragma unroll
            for (int j = 0; j < kAttnMaxG; ++j) sv[j] = 0.f;
            for (int e = 0; e < hd; e += 8) {
                float kf[8];
                if constexpr (sizeof(T) == 2) {
                    uint4 raw = *reinterpret_cast<const uint4*>(krow + e);
                    const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        float2 f = __bfloat1622float2(p2[u]);
                        kf[2 * u] = f.x;
                        kf[2 * u + 1] = f.y;
                    }
                } else {
                    float4 r0 = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(krow) + e);
                    float4 r1 = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(krow) + e + 4);
                    kf[0] = r0.x; kf[1] = r0.y; kf[2] = r0.z; kf[3] = r0.w;
                    kf[4] = r1.x; kf[5] = r1.y; kf[6] = r1.z; kf[7] = r1.w;
                }
#pragma unroll
                for (int j = 0; j < kAttnMaxG; ++j) {
                    if (j < G) {
#pragma unroll
                        for (int u = 0; u < 8; ++u) sv[j] += qs[j * hd + e + u] * kf[u];
                    }
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < kAttnMaxG; ++j) sv[j] = -INFINITY;
        }
        // phase 2: chunk max per head, online-softmax rescale
        const int lane = tid & 31, warp = tid >> 5;
        for (int j = 0; j < G; ++j) {
            float m = sv[j];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) red[warp * kAttnMaxG + j] = m;
        }
        __syncthreads();
        if (tid < G) {
            float m = fmaxf(fmaxf(red[tid], red[kAttnMaxG + tid]), fmaxf(red[2 * kAttnMaxG + tid], red[3 * kAttnMaxG + tid]));
            float mnew = fmaxf(mrow[tid], m);
            alpha[tid] = exp2f(mrow[tid] - mnew);  // mrow=-inf first time -> 0
            mrow[tid] = mnew;
        }
        __syncthreads();
        for (int j = 0; j < G; ++j) {
            float p = (key < k_end) ? exp2f(sv[j] - mrow[j]) : 0.f;
            sc[j * kAttnThreads + tid] = p;
            float ps = p;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
            if (lane == 0) red[warp * kAttnMaxG + j] = ps;
        }
        __syncthreads();
        if (tid < G) {
            float ps = (red[tid] + red[kAttnMaxG + tid]) + (red[2 * kAttnMaxG + tid] + red[3 * kAttnMaxG + tid]);
            lrow[tid] = lrow[tid] * alpha[tid] + ps;
        }
        // phase 3: P V
        const int kn = min(kAttnThreads, k_end - k0);
        for (int u = 0; u < nout; ++u) {
            const int idx = tid + u * kAttnThreads;
            if (idx >= G * hd) break;
            const int j = idx / hd, e = idx % hd;
            float a = acc[u] * alpha[j];
            for (int kk = 0; kk < kn; ++kk) {
                const int kkey = k0 + kk;
                const int page = pt[kkey / kPageTokens];
                const T* vrow = kv + layer_base + (size_t)page * page_stride + ((size_t)g * 2 + 1) * kPageTokens * hd +
                                (size_t)(kkey % kPageTokens) * hd;
                a += sc[j * kAttnThreads + kk] * DT<T>::to_f(vrow[e]);
            }
            acc[u] = a;
        }
        __syncthreads();
    }
    // write: nsplit == 1 -> normalised output; else partial (acc, m, l)
    if (nsplit == 1) {
        T* o = reinterpret_cast<T*>(P.o) + (size_t)b * P.act_ld + (size_t)g * G * hd;
        for (int u = 0; u < nout; ++u) {
            const int idx = tid + u * kAttnThreads;
            if (idx >= G * hd) break;
            const int j = idx / hd;
            float l = lrow[j];
            DT<T>::store_act(o + idx, (size_t)P.act_plane, l > 0.f ? acc[u] / l : 0.f);
        }
    } else {
        float* part = P.attn_part + (((size_t)b * P.Hkv + g) * nsplit + split) * (size_t)(G * (hd + 2));
        for (int u = 0; u < nout; ++u) {
            const int idx = tid + u * kAttnThreads;
            if (idx >= G * hd) break;
            part[idx] = acc[u];
        }
        if (tid < G) {
            part[G * hd + tid] = mrow[tid];
            part[G * hd + G + tid] = lrow[tid];
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(128) attention_merge_kernel(const __grid_constant__ StepParams P) {
    pdl_launch_dependents();
    pdl_wait();
    const int g = blockIdx.x, b = blockIdx.y;
    const int G = P.H / P.Hkv, hd = P.hd, nsplit = P.attn_splits;
    const float* part = P.attn_part + ((size_t)b * P.Hkv + g) * nsplit * (size_t)(G * (hd + 2));
    T* o = reinterpret_cast<T*>(P.o) + (size_t)b * P.act_ld + (size_t)g * G * hd;
    for (int idx = threadIdx.x; idx < G * hd; idx += blockDim.x) {
        const int j = idx / hd;
        float m = -INFINITY;
        for (int s = 0; s < nsplit; ++s) m = fmaxf(m, part[(size_t)s * G * (hd + 2) + G * hd + j]);
        float num = 0.f, den = 0.f;
        for (int s = 0; s < nsplit; ++s) {
            const float* ps = part + (size_t)s * G * (hd + 2);
            float ms = ps[G * hd + j];
            if (ms == -INFINITY) continue;
            float w = exp2f(ms - m);
            num += w * ps[idx];
            den += w * ps[G * hd + G + j];
        }
        DT<T>::store_act(o + idx, (size_t)P.act_plane, den > 0.f ? num / den : 0.f);
    }
}

// ------------------------------------------------------------------ SIMT GEMM (fp32 path)
// One CTA per 128*nsub-row tile; thread et owns row n = tile*128*nsub + s*128 + et and
// computes all Bp columns (fp32 FMA, no TF32), then runs the shared epilogue.
template <typename T>
__global__ void __launch_bounds__(128) gemm_simt_kernel(const __grid_constant__ StepParams P, const T* W,
                                                        int64_t w_row0, const T* X, int K, int nsub, int tiles,
                                                        EpiArgs E) {
    pdl_launch_dependents();
    extern __shared__ float gsm[];
    float* esm = gsm;                          // [128][33]
    EpiMeta meta;
    meta.kvoff = reinterpret_cast<long long*>(esm + 128 * kEsmLd + 4);
    meta.scale = reinterpret_cast<float*>(meta.kvoff + P.Bp);
    meta.pos = reinterpret_cast<int*>(meta.scale + P.Bp);
    float* xs = reinterpret_cast<float*>(meta.pos + P.Bp);  // [32][K]
    __shared__ int flag;
    pdl_wait();
    const int et = threadIdx.x;
    epilogue_prepare(P, E, meta, et);
    __syncthreads();
    const int tile = blockIdx.x;
    for (int s = 0; s < nsub; ++s) {
        const int n0 = (tile * nsub + s) * 128;
        const int n = n0 + et;
        for (int cb = 0; cb < P.Bp; cb += 32) {
            __syncthreads();
            for (int i = et; i < 32 * K; i += 128) {
                int c = i / K, k = i % K;
                xs[i] = DT<T>::to_f(X[(size_t)(cb + c) * P.act_ld + k]);
            }
            __syncthreads();
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
            const T* wr = W + (size_t)(w_row0 + n) * K;
            if (n < E.N) {
                for (int k = 0; k < K; ++k) {
                    float w = DT<T>::to_f(wr[k]);
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = fmaf(w, xs[i * K + k], v[i]);
                }
            }
            epilogue_chunk<T>(P, E, n0, cb, v, esm, meta, et);
        }
    }
    if (E.kind == EPI_LMHEAD) {
        __threadfence();
        __syncthreads();
        if (et == 0) flag = (atomicAdd(P.lm_done, 1) == tiles - 1);
        __syncthreads();
        if (flag) sample_scan_publish(P, et, reinterpret_cast<int*>(esm));
    }
}

}  // namespace cvy
