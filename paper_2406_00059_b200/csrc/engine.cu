// engine.cu -- host engine of libconveyor: device buffers, slot table, page allocator,
// pinned segment ring, step-graph cache per batch bucket, and the C ABI of conveyor.h.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/conveyor.h"
#include "common.cuh"
#include "epilogue.cuh"
#include "gemm_sm100.cuh"
#include "kernels.cuh"
#include "attention_tc.cuh"
#include "step_params.h"

using namespace cvy;

namespace {

thread_local std::string g_last_error;

cvy_status fail(cvy_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}

#define CUDA_TRY(expr)                                                                          \
    do {                                                                                        \
        cudaError_t _e = (expr);                                                                \
        if (_e != cudaSuccess) {                                                                \
            return fail(CVY_E_CUDA, std::string(#expr ": ") + cudaGetErrorString(_e));          \
        }                                                                                       \
    } while (0)

size_t dtype_size(cvy_dtype d) { return d == CVY_DTYPE_BF16 ? 2 : 4; }

uint32_t pow2_at_least(uint32_t v) {
    uint32_t p = 32;
    while (p < v) p <<= 1;
    return p;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 2D bf16 tensor map: [rows][cols] row-major, box {box_cols, box_rows}; box_cols 64 -> 128B
// swizzle, 32 -> 64B swizzle (matches the UMMA shared-memory descriptors).
bool make_tmap(CUtensorMap* out, const void* base, uint64_t rows, uint64_t cols, uint64_t row_stride_elems,
               uint32_t box_rows, uint32_t box_cols = 64) {
    auto fn = get_encode_fn();
    if (!fn) return false;
    cuuint64_t gdim[2] = {cols, rows};
    cuuint64_t gstride[1] = {row_stride_elems * 2};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estride[2] = {1, 1};
    CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstride, box, estride,
                    CU_TENSOR_MAP_INTERLEAVE_NONE,
                    box_cols == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// 3D view of a [rows][128] bf16 KV pool: dims (64 elements, rows, 2 halves), strides 256 B
// (row) and 128 B (half); box (64, 16, 2) = one 4 KB block, 128B swizzle per 128-byte row,
// landing in shared memory as [half][16 rows][64] (the layout of two 16 x 64 2D boxes).
bool make_tmap_kv3(CUtensorMap* out, const void* base, uint64_t rows) {
    auto fn = get_encode_fn();
    if (!fn) return false;
    cuuint64_t gdim[3] = {64, rows, 2};
    cuuint64_t gstride[2] = {256, 128};
    cuuint32_t box[3] = {64, 32, 2};  // one (page, kv-head) K+V block: 32 rows x 2 halves
    cuuint32_t estride[3] = {1, 1, 1};
    CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), gdim, gstride, box, estride,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// CTA-pair GEMMs (cta_group::2) for the epilogue kinds in the bit mask CVY_GEMM_PAIR (1 << EpiKind).
// Default on batch tiles (Bp > 128): QKV (whole 256-row tiles left 52 SMs idle; stream-K over 144
// pair CTAs) and gate/up (a single-CTA 256-row tile fills all 512 TMEM columns, so its epilogue
// stalled the MMAs; a pair CTA's 128 rows double-buffer the accumulator): C4 QKV 2.22 -> 2.03,
// gate/up 6.8 -> 5.9 ms/step; O / down as whole pair tiles instead of the 2-CTA cluster split-K:
// 1.40 -> 1.30 and 3.23 -> 3.13 ms/step (as stream-K pairs they lose, so they pair only when whole
// tiles fill the GPU). DESIGN.md §7.3. The LM head never pairs (its sampling CTA counts whole tiles).
bool gemm_pair_ok(int epi_kind) {
    if (epi_kind == EPI_LMHEAD) return false;
    const char* v = getenv("CVY_GEMM_PAIR");
    const int mask = v ? atoi(v) : ((1 << EPI_QKV) | (1 << EPI_RESID) | (1 << EPI_SWIGLU));
    return ((mask >> epi_kind) & 1) != 0;
}

// Tile/pipeline configuration of the tcgen05 GEMM for a padded batch Bp.
//   Bp <= 128: 2 sub-tiles (256 weight rows) per tile, hi/lo planes merged (MMA N = 2*Bp)
//   Bp 160..256: 1 sub-tile, planes as two MMAs into one accumulator (N = Bp)
//   Bp 512: 1 sub-tile, 2 batch halves of N = 256, 32-element K stages (64B swizzle)
bool gemm_config(GemmTC& g, int N, int K, int Bp, int num_sms, int* grid, size_t* smem, std::string* why,
                 bool allow_kernel_split = true, bool streamk = false, int nsub_override = 0, int epi_groups = 1,
                 bool pair_ok = false, bool pair_sk_ok = true) {
    g.N = N;
    g.K = K;
    g.pair = 0;
    // batches above 128 columns run as nbt tiles of 128 on grid.y, each with the merged
    // (hi, lo) N = 256 pipeline (measured: the unmerged Bp = 256 layout, 4x more activation
    // than weight bytes per stage and 2 stages, ran gate/up at 1.7 TB/s)
    int bq_max = 128;
    if (const char* v = getenv("CVY_GEMM_BQ")) bq_max = std::max(32, std::min(256, atoi(v)));  // A/B knob
    g.nbt = Bp > bq_max ? Bp / bq_max : 1;
    g.bq = Bp / g.nbt;
    if (getenv("CVY_GEMM_NO_BATCH_TILES")) {
        g.nbt = 1;
        g.bq = Bp;
    }
    const int Bq = g.bq;
    g.merge = Bq <= 128;
    g.bk = Bq >= 512 ? 32 : 64;
    // CTA pairs (cta_group::2) for batch-tiled GEMMs: a 256-row tile per pair, each CTA streams
    // its 128 weight rows and ONE activation plane, the leader issues M = 256 MMAs -- per SM half
    // the activation bytes through shared memory of a 128-row tile, no split-K reduction
    const bool pair_small = getenv("CVY_GEMM_PAIR_SMALL") && atoi(getenv("CVY_GEMM_PAIR_SMALL")) != 0;  // A/B knob
    const bool force_sk = getenv("CVY_PAIR_STREAMK") && atoi(getenv("CVY_PAIR_STREAMK")) != 0;  // A/B knob
    const int pair_tiles = N / 256, pairs_per_bt = std::max(1, num_sms / std::max(1, g.nbt) / 2);
    // whole pair tiles when they fill >= 3/4 of the SMs in one wave, else stream-K over the pairs
    const bool pair_whole = !force_sk && pair_tiles <= pairs_per_bt && 4 * 2 * pair_tiles * g.nbt >= 3 * num_sms;
    if (pair_ok && (pair_whole || pair_sk_ok) && g.merge && (g.nbt > 1 || pair_small) && N % 256 == 0 &&
        K % 128 == 0 && K / 128 >= 2) {
        g.pair = 1;
        g.nsub = 1;
        g.mma_n = 2 * Bq;
        g.nbh = 1;
        g.cols_per_sub = 2 * Bq;
        g.acc_stages = 2;
        g.tmem_cols = pow2_at_least((uint32_t)(2 * g.cols_per_sub));
        g.tiles = N / 256;
        g.kblocks = K / 128;  // pipeline stages of two 64-column k-blocks (gemm_sm100.cuh KB2)
        g.l2_prefetch = 0;
        const uint32_t stage = 2 * GemmSmem::stage_bytes(1, Bq, 1, 64);
        const uint32_t fixed = GemmSmem::fixed_bytes(Bp) + 1024;
        g.stages = std::min(12, (int)((232448 - fixed) / stage));
        *smem = (size_t)g.stages * stage + fixed;
        if (pair_whole) {
            g.split = 1;  // whole tiles: one pair per (tile, batch tile)
            *grid = 2 * g.tiles;
        } else {
            g.split = 0;  // stream-K over the pairs of a batch tile
            *grid = 2 * (int)std::min<long long>(pairs_per_bt, (long long)g.tiles * g.kblocks);
        }
        return true;
    }
    if (const char* v = getenv("CVY_GEMM_BK")) g.bk = (atoi(v) == 32 && !g.merge) ? 32 : 64;  // A/B knob
    // wide GEMMs (gate/up, LM head): 256-row tiles, one per CTA, no reduction; narrow ones
    // (QKV, O, down): 128-row tiles with K split over a 2..4-CTA cluster (DSMEM reduction)
    // 256-row tiles halve the activation bytes per weight byte; worth it down to the QKV
    // width (6144 rows: 24 tiles x 4-CTA clusters; measured QKV 0.896 -> 0.836 ms/step at B=64),
    // not for the 4096-row O / down GEMMs (16 tiles: too few CTAs)
    g.nsub = (g.merge && N >= 6144) ? 2 : 1;
    // batch tiles (Bp > 128): the narrow GEMMs (O, down) also take 256-row tiles, K split over a
    // 2-CTA cluster per (tile, batch tile) -- half the shared-memory traffic per MMA of 128-row
    // tiles, which cap the tensor pipe at ~2/3 there (measured at B = 512: down 97 -> 81 us)
    bool bt_split = g.merge && g.nbt > 1 && allow_kernel_split && !streamk &&
                    ((N + 255) / 256) * g.nbt * 2 <= num_sms && K / 64 >= 2;
    if (const char* v = getenv("CVY_GEMM_BT_SPLIT")) bt_split = bt_split && atoi(v) != 0;  // A/B knob
    if (bt_split) g.nsub = 2;
    if (const char* ns = getenv("CVY_GEMM_NSUB")) g.nsub = std::max(1, std::min(2, atoi(ns)));
    if (nsub_override > 0) g.nsub = nsub_override;
    if (g.merge) {
        g.mma_n = 2 * Bq;
        g.nbh = 1;
        g.cols_per_sub = 2 * Bq;
    } else {
        g.mma_n = std::min(Bq, 256);
        g.nbh = Bq / g.mma_n;
        g.cols_per_sub = Bq;
    }
    // unmerged (Bq > 128): hi and lo accumulate into the same TMEM columns; two 128-row
    // sub-tiles fill all 512 columns at Bq = 256 (one accumulator stage)
    if (!g.merge && !(nsub_override == 2 || getenv("CVY_GEMM_NSUB"))) g.nsub = 1;
    if (g.nsub * g.cols_per_sub > 512) {
        *why = "accumulator exceeds TMEM";
        return false;
    }
    g.acc_stages = (2 * g.nsub * g.cols_per_sub <= 512) ? 2 : 1;
    g.tmem_cols = pow2_at_least((uint32_t)(g.acc_stages * g.nsub * g.cols_per_sub));
    g.tiles = (N + 128 * g.nsub - 1) / (128 * g.nsub);
    g.kblocks = K / g.bk;
    const uint32_t stage = GemmSmem::stage_bytes(g.nsub, Bq, 2, g.bk);
    const uint32_t fixed = GemmSmem::fixed_bytes(Bp) + 1024;
    (void)epi_groups;  // the second epilogue group borrows the idle ring (gemm_sm100.cuh)
    // shared-memory budget per CTA (A/B knob CVY_GEMM_SMEM: a smaller ring lets the next
    // kernel's CTA co-reside and start its weight stream under this kernel's epilogue tail)
    uint32_t budget = 232448;
    if (const char* v = getenv("CVY_GEMM_SMEM")) budget = std::max(fixed + 2 * stage, std::min<uint32_t>(232448, atoi(v)));
    int stages = std::min(12, (int)((budget - fixed) / stage));
    if (stages < 2) {
        *why = "not enough shared memory for 2 stages";
        return false;
    }
    g.stages = stages;
    *smem = (size_t)stages * stage + fixed;
    // split mode: tiles <= SMs (one tile, or one cluster of S CTAs per tile)
    g.split = 0;
    if (g.merge && !getenv("CVY_GEMM_STREAMK") && !streamk && (g.nbt == 1 || !allow_kernel_split || bt_split)) {
        int S = 1;
        // the LM head counts completed tiles to elect the sampling CTA: whole tiles only
        int smax = kMaxSplit;
        if (const char* v = getenv("CVY_GEMM_MAXSPLIT")) smax = std::max(1, std::min(kMaxSplit, atoi(v)));  // A/B knob
        while (allow_kernel_split && S < smax && g.tiles * g.nbt * (S + 1) <= num_sms && S + 1 <= g.kblocks) ++S;
        if (S == 3 && !getenv("CVY_GEMM_ALLOW_S3")) S = 2;  // clusters of 3 do not pack onto the GPCs (measured: second wave)
        if ((bt_split ? g.tiles * g.nbt : g.tiles) <= num_sms) g.split = S;
        // the DSMEM staging of the partial must fit in the pipeline smem
        if (g.split > 1 && (size_t)g.nsub * Bq * 512 > (size_t)stages * stage) g.split = 0;
        // the kernel's reduce-scatter sums at most kMaxSplit ranks (gemm_sm100.cuh, t4[kMaxSplit])
        if (g.split > kMaxSplit) {
            *why = "cluster split-K wider than the kernel's reduce-scatter";
            return false;
        }
    }
    // L2 look-ahead: ~256 KB of weights per CTA beyond the smem ring (bounded by L2 capacity)
    g.l2_prefetch = 0;  // measured: no gain (mainloops already stream at 5.6-6.8 TB/s once unblocked)
    if (const char* pf = getenv("CVY_GEMM_L2PF")) g.l2_prefetch = atoi(pf);
    if (g.split > 0) {
        *grid = g.tiles * g.split;
    } else {
        // stream-K: the nbt batch tiles share the SMs (each streams 1/grid of the weights).
        // When every (tile, batch tile) fits one wave, whole tiles instead: no shared tile, so no
        // L2 partial fix-up in the kernel's tail (measured at B = 512)
        const long long T = (long long)g.tiles * g.kblocks;
        *grid = (int)std::min<long long>(std::max(1, num_sms / g.nbt), T);
        int whole = 1;
        if (const char* v = getenv("CVY_GEMM_WHOLE")) whole = atoi(v);
        if (whole && g.nbt > 1 && g.tiles * g.nbt <= num_sms) *grid = g.tiles;
        // A/B knob: exactly k whole tiles per CTA (no shared tile): tile i's epilogue overlaps
        // tile i+1's main loop through the double-buffered TMEM accumulator
        if (const char* v = getenv(streamk ? "CVY_GU_TPC" : "CVY_GEMM_TPC"))
            if (atoi(v) > 0 && g.tiles % atoi(v) == 0) *grid = g.tiles / atoi(v);
    }
    return true;
}

void set_gemm_smem_attrs() {
    static bool done = false;
    if (done) return;
    done = true;
    for (int epi = 0; epi <= EPI_STORE; ++epi)
        for (int nsub = 1; nsub <= 2; ++nsub)
            for (int merge = 0; merge <= 1; ++merge)
                for (int bk : {32, 64})
                    cudaFuncSetAttribute(gemm_tc_kernel_ptr<__nv_bfloat16>(nsub, merge != 0, bk, epi),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    for (int epi = 0; epi <= EPI_STORE; ++epi)
        cudaFuncSetAttribute(gemm_tc_kernel_ptr<__nv_bfloat16>(1, true, 64, epi, true),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
}

struct SlotHost {
    bool used = false;
    uint64_t req_id = 0;
    int state = 3;  // 0 running, 1 parked (FINAL polled), 2 cancelled, 3 free
    std::vector<int32_t> pages;
    int32_t reserved = 0;  // KV positions reserved (pages * 16)
    int32_t next_pos = 0;  // host's view of the position after the last fed/forced token
    bool final_seen = false;
    bool final_pending = false;  // round running (a FINAL will come)
    int32_t round_pos0 = 0;      // device pos of the round's first input token
    int32_t round_inputs = 0;    // input tokens the round feeds before generating (incl. cur_tok)
    bool cancel_pending = false; // a CANCEL patch is queued for the running round (de-duplication)
};

// A synthetic KV prefix to write before the slot's first step (queued by submit, run by
// cvy_step on the engine stream after the page-table uploads, never during a graph capture).
struct SynthJob {
    int slot;
    uint32_t len;
    uint64_t seed;
};

// A chunked-prefill job (NEXT-1): tokens fed at positions pos0, pos0+1, ... of a slot.
struct PrefillJob {
    int slot;
    int32_t pos0;
    std::vector<int32_t> toks;
};
constexpr int kPrefillRows = 512;  // rows per prefill pass (activation buffer capacity)

struct Upload {
    void* dst;
    std::vector<uint8_t> data;
};

struct GemmPlan {
    CUtensorMap tmW, tmX;
    CUtensorMap tmN;  // weights of the next GEMM in the step (L2 prefetch in the epilogue tail)
    GemmTC g;
    int grid;
    size_t smem;
    // SIMT path
    const void* W;
    const void* X;
    int64_t w_row0;
};

struct Bucket {
    int Bp = 0;
    StepParams P;
    int nsub = 2;
    std::vector<GemmPlan> plans;  // per launch in order
    cudaGraphExec_t graph = nullptr;
    cudaGraphExec_t graph_timed = nullptr;  // event pair around every kernel, no PDL
    cudaGraphExec_t graph_spans = nullptr;  // the production graph + in-graph kernel spans
    std::vector<cudaEvent_t> kev;
    std::vector<std::pair<int, int>> kinfo;  // (kind, layer) per launch
    uint32_t launches = 0;
};

}  // namespace

struct cvy_engine;
int m_d(const cvy_engine* e);
struct cvy_engine {
    cvy_model_config m{};
    cvy_engine_config c{};
    cvy_weights w{};
    int dev = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t cur = nullptr;        // stream launch_k enqueues on
    bool dead = false;
    bool bf16 = true;
    int act_ld = 0;
    // device buffers
    SlotDev* d_slots = nullptr;
    int32_t* d_page_table = nullptr;
    int32_t* d_in_buf = nullptr;
    int32_t* d_force_buf = nullptr;
    float2* d_rope = nullptr;
    int max_rope_pos = 0;
    float* d_x = nullptr;
    void* d_act = nullptr;
    float* d_q = nullptr;
    void* d_o = nullptr;
    void* d_h = nullptr;
    float* d_ssq = nullptr;
    unsigned long long* d_am = nullptr;
    float* d_dbg = nullptr;
    int32_t* d_lm_done = nullptr;
    float* d_attn_part = nullptr;
    int attn_splits_max = 16;
    uint8_t* d_vtab = nullptr;
    uint8_t* d_vlen = nullptr;
    ToolDev* d_tools = nullptr;
    unsigned long long* d_ring_tail = nullptr;
    unsigned long long* d_step = nullptr;
    float* d_gemm_acc = nullptr;
    int32_t* d_tile_cnt = nullptr;
    Patch* d_patches = nullptr;
    int max_patches = 0;
    // pinned mapped host buffers
    cvy_segment* h_ring = nullptr;
    unsigned long long* h_ring_tail = nullptr;
    uint8_t* h_byte_log = nullptr;
    int32_t* h_tok_log = nullptr;
    SlotStatus* h_status = nullptr;
    StepStats* h_stats = nullptr;
    void* dm_ring = nullptr;
    void* dm_ring_tail = nullptr;
    void* dm_byte_log = nullptr;
    void* dm_tok_log = nullptr;
    void* dm_status = nullptr;
    void* dm_stats = nullptr;
    // host state
    std::mutex mu;
    std::vector<Patch> pending;
    std::vector<Upload> uploads;
    std::vector<SynthJob> synth_pending;
    std::vector<SlotHost> slots;
    std::vector<int32_t> free_pages;
    std::vector<ToolDev> tools;
    std::vector<std::string> tool_names;
    std::vector<uint32_t> tool_max_seg;
    bool submitted_any = false;
    uint64_t next_req = 1;
    std::unordered_map<uint64_t, int> req_slot;
    std::map<int, Bucket> buckets;
    std::deque<std::pair<cudaEvent_t, cudaEvent_t>> inflight;  // (start, end)
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> event_pool;
    uint64_t steps_launched = 0;
    uint64_t ring_head = 0;  // consumer position
    float last_step_ms = 0.f;
    int last_bucket = 0;
    uint32_t last_launches = 0;
    std::vector<uint8_t> vlen_host;
    bool attn_tc = false;       // bf16 KV, head_dim 64/128, G <= 4: TMA + mma.sync attention
    int attn_stages = 2;
    int attn_pps = 2;           // KV pages per attention stage: 2 x 2 stages = 32 KB of ring per CTA,
                                // 6 CTAs per SM, so the decode grid (Hkv x B) runs in one wave
                                // (measured at B=64: attention -3..6% vs 4 pages x 3 stages)
    CUtensorMap tm_kv;          // 2D view of the KV pool: [L*pages*2*Hkv*16 rows][hd] (3D when kv_tma3d)
    bool kv_tma3d = false;
    // chunked prefill (NEXT-1): row tables and activation buffers of a prefill pass
    float* d_px = nullptr;
    void* d_pact = nullptr;
    float* d_pq = nullptr;
    void* d_po = nullptr;
    void* d_ph = nullptr;
    float* d_pssq = nullptr;
    float* d_pattn_part = nullptr;
    int32_t* d_prow = nullptr;      // [3][kPrefillRows]: slot, pos, token
    std::vector<PrefillJob> prefill_pending;
    std::map<int, Bucket> prefill_buckets;
    uint64_t prefill_rows_total = 0;
    bool w_tiled = false;           // projection weights packed tile-major (CVY_ENGINE_TILED_WEIGHTS)
    unsigned long long* d_trace = nullptr;  // test hook: GEMM CTA timestamps of one layer
    int trace_layer = -1;
    bool timing = false;        // launch the timed graph variant
    bool spans_on = false;      // launch the span-recording graph variant
    bool capturing_spans = false;
    unsigned long long* d_spans = nullptr;  // [2][kSpanSlots] (StepParams::spans)
    Bucket* last_spans = nullptr;
    bool capturing_timed = false;
    Bucket* last_timed = nullptr;
};

int m_d(const cvy_engine* e) { return e->m.d_model; }

namespace {

cvy_status check_cuda(cvy_engine* e, cudaError_t err, const char* what) {
    if (err != cudaSuccess) {
        e->dead = true;
        std::string msg = std::string(what) + ": " + cudaGetErrorString(err);
        return fail(CVY_E_CUDA, msg);
    }
    return CVY_OK;
}

bool model_ok(const cvy_model_config* m, std::string* why) {
    if (!m) { *why = "null model config"; return false; }
    if (m->n_layers < 0 || m->d_model <= 0 || m->n_heads <= 0 || m->n_kv_heads <= 0 || m->vocab <= 0 || m->d_ff <= 0) {
        *why = "non-positive model dimension";
        return false;
    }
    if (m->head_dim != 32 && m->head_dim != 64 && m->head_dim != 128) { *why = "head_dim must be 32, 64 or 128"; return false; }
    if (m->d_model % 128 || (m->n_heads * m->head_dim) % 128 || m->d_ff % 64) { *why = "d_model, H*hd must be multiples of 128, d_ff of 64"; return false; }
    if (m->n_heads % m->n_kv_heads || m->n_heads / m->n_kv_heads > kAttnMaxG) { *why = "n_heads / n_kv_heads must be an integer <= 8"; return false; }
    if (m->d_model > 8192) { *why = "d_model must be <= 8192 (embedding kernel's per-block sums)"; return false; }
    if (m->dtype != CVY_DTYPE_BF16 && m->dtype != CVY_DTYPE_FP32) { *why = "bad dtype"; return false; }
    if (m->dtype == CVY_DTYPE_FP32 && std::max(m->d_model, std::max(m->d_ff, m->n_heads * m->head_dim)) > 1024) {
        *why = "fp32 parity path supports K <= 1024 only";
        return false;
    }
    return true;
}

}  // namespace

// the native runtime (runtime.cpp) reports its errors through the same thread-local message
cvy_status cvy_internal_fail(cvy_status st, const std::string& msg) { return fail(st, msg); }

// ============================================================================ C ABI
extern "C" {

int32_t cvy_abi_version(void) { return CVY_ABI_VERSION; }
const char* cvy_last_error(void) { return g_last_error.c_str(); }

cvy_status cvy_weight_sizes_for(const cvy_model_config* m, uint32_t n_pages, cvy_weight_sizes* out) {
    std::string why;
    if (!model_ok(m, &why) || !out) return fail(CVY_E_INVAL, why.empty() ? "null output" : why);
    const size_t es = dtype_size(m->dtype);
    const size_t L = m->n_layers, d = m->d_model, H = m->n_heads, Hkv = m->n_kv_heads, hd = m->head_dim,
                 dff = m->d_ff, V = m->vocab;
    out->embed = V * d * es;
    out->lm_head = V * d * es;
    out->final_norm = d * 4;
    out->attn_norm = L * d * 4;
    out->mlp_norm = L * d * 4;
    out->wqkv = L * (H + 2 * Hkv) * hd * d * es;
    out->wo = L * d * H * hd * es;
    out->wgu = L * 2 * dff * d * es;
    out->wd = L * d * dff * es;
    out->kv_pool = L * (size_t)n_pages * 2 * Hkv * kPageTokens * hd * es;
    return CVY_OK;
}

cvy_status cvy_init_synthetic_weights(const cvy_model_config* m, const cvy_weights* w, uint64_t seed, int32_t device) {
    std::string why;
    if (!model_ok(m, &why) || !w) return fail(CVY_E_INVAL, why.empty() ? "null weights" : why);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(CVY_E_CUDA, "no CUDA device");
    CUDA_TRY(cudaSetDevice(device));
    const double a = 0.02 * std::sqrt(3.0);
    const int64_t L = m->n_layers, d = m->d_model, H = m->n_heads, Hkv = m->n_kv_heads, hd = m->head_dim,
                  dff = m->d_ff, V = m->vocab;
    const bool bf = m->dtype == CVY_DTYPE_BF16;
    const size_t es = dtype_size(m->dtype);
    auto launch = [&](const void* dst, uint64_t tid, int64_t rows, int64_t cols, int inter, int which) {
        dim3 grid(2048), block(256);
        if (bf)
            init_hash_kernel<__nv_bfloat16><<<grid, block>>>((__nv_bfloat16*)dst, seed, tid, rows, cols, a, inter, which);
        else
            init_hash_kernel<float><<<grid, block>>>((float*)dst, seed, tid, rows, cols, a, inter, which);
    };
    launch(w->embed, 0, V, d, 0, 0);
    launch(w->lm_head, (uint64_t)(1 + 8 * L), V, d, 0, 0);
    for (int64_t l = 0; l < L; ++l) {
        const uint8_t* qkv = (const uint8_t*)w->wqkv + (size_t)l * (H + 2 * Hkv) * hd * d * es;
        launch(qkv, 1 + 8 * l + 0, H * hd, d, 0, 0);
        launch(qkv + (size_t)H * hd * d * es, 1 + 8 * l + 1, Hkv * hd, d, 0, 0);
        launch(qkv + (size_t)(H + Hkv) * hd * d * es, 1 + 8 * l + 2, Hkv * hd, d, 0, 0);
        launch((const uint8_t*)w->wo + (size_t)l * d * H * hd * es, 1 + 8 * l + 3, d, H * hd, 0, 0);
        const uint8_t* gu = (const uint8_t*)w->wgu + (size_t)l * 2 * dff * d * es;
        launch(gu, 1 + 8 * l + 4, dff, d, 1, 0);
        launch(gu, 1 + 8 * l + 5, dff, d, 1, 1);
        launch((const uint8_t*)w->wd + (size_t)l * d * dff * es, 1 + 8 * l + 6, d, dff, 0, 0);
    }
    fill_f32_kernel<<<64, 256>>>((float*)w->final_norm, d, 1.f);
    fill_f32_kernel<<<256, 256>>>((float*)w->attn_norm, L * d, 1.f);
    fill_f32_kernel<<<256, 256>>>((float*)w->mlp_norm, L * d, 1.f);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    return CVY_OK;
}

// Tile-major packing of the projection weights (DESIGN.md §7.2 "Weight layout").
bool tiled_shape_ok(const cvy_model_config* m, std::string* why) {
    const int64_t d = m->d_model, H = m->n_heads, Hkv = m->n_kv_heads, hd = m->head_dim, dff = m->d_ff;
    if (m->dtype != CVY_DTYPE_BF16) {
        *why = "tile-major weights are bf16 only";
        return false;
    }
    if (((H + 2 * Hkv) * hd) % 128 || d % 128 || (2 * dff) % 128 || d % 64 || (H * hd) % 64 || dff % 64) {
        *why = "tile-major weights need every projection's rows % 128 == 0 and columns % 64 == 0";
        return false;
    }
    return true;
}

// The LM head joins the tile-major packing when its rows split into 128-row tiles.
bool lm_head_tiled(const cvy_model_config* m) { return m->vocab % 128 == 0 && m->d_model % 64 == 0; }

// dst[((r / 128) * (K / 64) + k / 64) * 8192 + (r % 128) * 64 + k % 64] = src[r * K + k] for one
// [R][K] bf16 block (R % 128 == 0); 16 bytes per thread step.
__global__ void pack_tiled_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, int64_t R, int64_t K) {
    const int64_t n = R * K / 8, kc = K / 8, KB = K / 64;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / kc, k = (i % kc) * 8;
        dst[(((r / 128) * KB + k / 64) * 8192 + (r % 128) * 64 + k % 64) / 8] = src[i];
    }
}

cvy_status cvy_pack_weights_tiled(const cvy_model_config* m, const cvy_weights* w, int32_t device) {
    std::string why;
    if (!model_ok(m, &why) || !w) return fail(CVY_E_INVAL, why.empty() ? "null weights" : why);
    if (!w->wqkv || !w->wo || !w->wgu || !w->wd) return fail(CVY_E_INVAL, "null weight pointer");
    if (!tiled_shape_ok(m, &why)) return fail(CVY_E_INVAL, why);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(CVY_E_CUDA, "no CUDA device");
    CUDA_TRY(cudaSetDevice(device));
    const int64_t L = m->n_layers, d = m->d_model, H = m->n_heads, Hkv = m->n_kv_heads, hd = m->head_dim,
                  dff = m->d_ff;
    // the LM head [V][d] is packed too when V % 128 == 0 (lm_head_tiled(); one "layer")
    const int nq = lm_head_tiled(m) ? 5 : 4;
    const int64_t R[5] = {(H + 2 * Hkv) * hd, d, 2 * dff, d, (int64_t)m->vocab}, K[5] = {d, H * hd, d, dff, d};
    const int64_t Lq[5] = {L, L, L, L, 1};
    // the pack rewrites the caller's buffers (documented in conveyor.h); cvy_weights holds them const
    void* base[5] = {const_cast<void*>(w->wqkv), const_cast<void*>(w->wo), const_cast<void*>(w->wgu),
                     const_cast<void*>(w->wd), const_cast<void*>(w->lm_head)};
    if (nq == 5 && !w->lm_head) return fail(CVY_E_INVAL, "null weight pointer");
    size_t tmp_bytes = 0;
    for (int q = 0; q < nq; ++q) tmp_bytes = std::max(tmp_bytes, (size_t)(R[q] * K[q] * 2));
    void* tmp = nullptr;
    CUDA_TRY(cudaMalloc(&tmp, tmp_bytes));
    cudaError_t err = cudaSuccess;
    // one layer at a time through a scratch copy: a layer's tiles occupy exactly its own bytes
    for (int q = 0; q < nq && err == cudaSuccess; ++q)
        for (int64_t l = 0; l < Lq[q] && err == cudaSuccess; ++l) {
            uint8_t* blk = (uint8_t*)base[q] + (size_t)l * R[q] * K[q] * 2;
            err = cudaMemcpy(tmp, blk, (size_t)R[q] * K[q] * 2, cudaMemcpyDeviceToDevice);
            if (err == cudaSuccess) {
                pack_tiled_kernel<<<1184, 256>>>((uint4*)blk, (const uint4*)tmp, R[q], K[q]);
                err = cudaGetLastError();
            }
        }
    if (err == cudaSuccess) err = cudaDeviceSynchronize();
    cudaFree(tmp);
    if (err != cudaSuccess) return fail(CVY_E_CUDA, cudaGetErrorString(err));
    return CVY_OK;
}

void cvy_engine_destroy(cvy_engine* e);

cvy_status cvy_engine_create(const cvy_model_config* m, const cvy_engine_config* ec, const cvy_weights* w,
                             const uint8_t* vocab_bytes, const uint8_t* vocab_lens, cvy_engine** out) {
    std::string why;
    if (!out) return fail(CVY_E_INVAL, "null out");
    *out = nullptr;
    if (!model_ok(m, &why)) return fail(CVY_E_INVAL, why);
    if (!ec || !w || !vocab_bytes || !vocab_lens) return fail(CVY_E_INVAL, "null argument");
    if (ec->max_slots < 1 || ec->max_slots > (uint32_t)kMaxSlots) return fail(CVY_E_INVAL, "max_slots out of range");
    if (ec->ring_records < 32u * ec->max_slots || (ec->ring_records & (ec->ring_records - 1)))
        return fail(CVY_E_INVAL, "ring_records must be a power of two >= 32*max_slots");
    if (ec->n_pages < 1 || ec->max_pages_per_slot < 1 || ec->round_bytes < 16 || ec->round_tokens < 1 ||
        ec->input_cap < 1 || ec->forced_cap < 1)
        return fail(CVY_E_INVAL, "capacity fields must be positive");
    if (!w->embed || !w->lm_head || !w->final_norm || !w->attn_norm || !w->mlp_norm || !w->wqkv || !w->wo || !w->wgu ||
        !w->wd || !w->kv_pool)
        return fail(CVY_E_INVAL, "null weight pointer");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(CVY_E_CUDA, "no CUDA device");
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, ec->device));
    if (prop.major != 10) return fail(CVY_E_CUDA, "libconveyor is built for sm_100a (B200) only");
    CUDA_TRY(cudaSetDevice(ec->device));

    if ((ec->flags & CVY_ENGINE_TILED_WEIGHTS) && !tiled_shape_ok(m, &why)) return fail(CVY_E_INVAL, why);

    cvy_engine* e = new cvy_engine();
    e->w_tiled = (ec->flags & CVY_ENGINE_TILED_WEIGHTS) != 0;
    e->m = *m;
    e->c = *ec;
    e->w = *w;
    e->dev = ec->device;
    e->num_sms = prop.multiProcessorCount;
    e->bf16 = m->dtype == CVY_DTYPE_BF16;
    int Bmax = (int)((ec->max_slots + 31) / 32 * 32);
    if (Bmax > 256) Bmax = 512 * ((Bmax + 511) / 512);
    else if (Bmax > 128) Bmax = 256;
    const int d = m->d_model, H = m->n_heads, Hkv = m->n_kv_heads, hd = m->head_dim, dff = m->d_ff, V = m->vocab;
    e->act_ld = std::max(d, std::max(H * hd, dff));
    const size_t es = dtype_size(m->dtype);
    auto dmalloc = [&](void** p, size_t bytes) -> cvy_status {
        if (cudaMalloc(p, bytes) != cudaSuccess) return fail(CVY_E_NOMEM, "cudaMalloc failed");
        if (cudaMemset(*p, 0, bytes) != cudaSuccess) return fail(CVY_E_CUDA, "cudaMemset failed");
        return CVY_OK;
    };
    auto hmalloc = [&](void** hp, void** dp, size_t bytes) -> cvy_status {
        if (cudaHostAlloc(hp, bytes, cudaHostAllocMapped) != cudaSuccess) return fail(CVY_E_NOMEM, "cudaHostAlloc failed");
        std::memset(*hp, 0, bytes);
        if (cudaHostGetDevicePointer(dp, *hp, 0) != cudaSuccess) return fail(CVY_E_CUDA, "cudaHostGetDevicePointer");
        return CVY_OK;
    };
    cvy_status st = CVY_OK;
#define ALLOC(ptr, bytes)                                          \
    if ((st = dmalloc((void**)&(ptr), (bytes))) != CVY_OK) {       \
        cvy_engine_destroy(e);                                     \
        return st;                                                 \
    }
#define HALLOC(hptr, dptr, bytes)                                               \
    if ((st = hmalloc((void**)&(hptr), (void**)&(dptr), (bytes))) != CVY_OK) {  \
        cvy_engine_destroy(e);                                                  \
        return st;                                                              \
    }
    ALLOC(e->d_slots, sizeof(SlotDev) * Bmax);
    ALLOC(e->d_page_table, sizeof(int32_t) * Bmax * ec->max_pages_per_slot);
    ALLOC(e->d_in_buf, sizeof(int32_t) * (size_t)Bmax * ec->input_cap);
    ALLOC(e->d_force_buf, sizeof(int32_t) * (size_t)Bmax * ec->forced_cap);
    e->max_rope_pos = (int)(ec->max_pages_per_slot * kPageTokens);
    ALLOC(e->d_rope, sizeof(float2) * (size_t)e->max_rope_pos * (hd / 2));
    ALLOC(e->d_x, sizeof(float) * (size_t)Bmax * d);
    const size_t planes = e->bf16 ? 2 : 1;  // bf16: (hi, lo) activation pair
    ALLOC(e->d_act, planes * es * (size_t)Bmax * e->act_ld);
    ALLOC(e->d_q, sizeof(float) * (size_t)Bmax * H * hd);
    ALLOC(e->d_o, planes * es * (size_t)Bmax * e->act_ld);
    ALLOC(e->d_h, planes * es * (size_t)Bmax * e->act_ld);
    ALLOC(e->d_ssq, sizeof(float) * (size_t)(d / 128) * Bmax);
    ALLOC(e->d_am, sizeof(unsigned long long) * Bmax);
    if (ec->flags & CVY_ENGINE_DEBUG_LOGITS) ALLOC(e->d_dbg, sizeof(float) * (size_t)Bmax * V);
    ALLOC(e->d_lm_done, sizeof(int32_t) * 4);
    const int G = H / Hkv;
    ALLOC(e->d_attn_part, sizeof(float) * (size_t)Bmax * Hkv * e->attn_splits_max * G * (hd + 2));
    ALLOC(e->d_vtab, (size_t)V * kMaxTokenBytes);
    ALLOC(e->d_vlen, (size_t)V);
    ALLOC(e->d_tools, sizeof(ToolDev) * kMaxTools);
    ALLOC(e->d_ring_tail, sizeof(unsigned long long) * 2);
    ALLOC(e->d_step, sizeof(unsigned long long) * 2);
    // stream-K accumulators of shared tiles: rows padded to 256 per GEMM, Bmax columns
    const size_t max_rows = (size_t)std::max({(size_t)V, (size_t)2 * dff, (size_t)(H + 2 * Hkv) * hd, (size_t)d}) + 256;
    // (a chunked-prefill pass runs the same GEMMs over up to kPrefillRows rows)
    const size_t acc_cols = (ec->flags & CVY_ENGINE_CHUNKED_PREFILL) ? std::max(Bmax, kPrefillRows) : (size_t)Bmax;
    ALLOC(e->d_gemm_acc, sizeof(float) * max_rows * acc_cols);
    ALLOC(e->d_tile_cnt, sizeof(int32_t) * 8192);
    ALLOC(e->d_spans, sizeof(unsigned long long) * 2 * kSpanSlots);
    if ((ec->flags & CVY_ENGINE_CHUNKED_PREFILL) && e->bf16) {
        const size_t R = kPrefillRows;
        ALLOC(e->d_px, sizeof(float) * R * d);
        ALLOC(e->d_pact, 2 * es * R * e->act_ld);
        ALLOC(e->d_pq, sizeof(float) * R * H * hd);
        ALLOC(e->d_po, 2 * es * R * e->act_ld);
        ALLOC(e->d_ph, 2 * es * R * e->act_ld);
        ALLOC(e->d_pssq, sizeof(float) * (size_t)(d / 128) * R);
        ALLOC(e->d_pattn_part, sizeof(float) * R * Hkv * e->attn_splits_max * (H / Hkv) * (hd + 2));
        ALLOC(e->d_prow, sizeof(int32_t) * 3 * R);
    }
    e->max_patches = 4 * Bmax + 64;
    ALLOC(e->d_patches, sizeof(Patch) * e->max_patches);
    HALLOC(e->h_ring, e->dm_ring, sizeof(cvy_segment) * ec->ring_records);
    HALLOC(e->h_ring_tail, e->dm_ring_tail, sizeof(unsigned long long) * 8);
    HALLOC(e->h_byte_log, e->dm_byte_log, (size_t)Bmax * ec->round_bytes);
    HALLOC(e->h_tok_log, e->dm_tok_log, sizeof(int32_t) * (size_t)Bmax * ec->round_tokens);
    HALLOC(e->h_status, e->dm_status, sizeof(SlotStatus) * Bmax);
    HALLOC(e->h_stats, e->dm_stats, sizeof(StepStats) * 16);
#undef ALLOC
#undef HALLOC
    for (int b = 0; b < Bmax; ++b) e->h_status[b].state = 3;
    // RoPE table (fp64 angles -> fp32 cos/sin), theta_i = base^(-2i/hd)
    {
        std::vector<float2> rope((size_t)e->max_rope_pos * (hd / 2));
        for (int p = 0; p < e->max_rope_pos; ++p)
            for (int i = 0; i < hd / 2; ++i) {
                double th = std::pow(m->rope_base, -2.0 * i / hd);
                double ang = (double)p * th;
                rope[(size_t)p * (hd / 2) + i] = make_float2((float)std::cos(ang), (float)std::sin(ang));
            }
        if (cudaMemcpy(e->d_rope, rope.data(), rope.size() * sizeof(float2), cudaMemcpyHostToDevice) != cudaSuccess) {
            cvy_engine_destroy(e);
            return fail(CVY_E_CUDA, "rope upload");
        }
    }
    if (cudaMemcpy(e->d_vtab, vocab_bytes, (size_t)V * kMaxTokenBytes, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(e->d_vlen, vocab_lens, (size_t)V, cudaMemcpyHostToDevice) != cudaSuccess) {
        cvy_engine_destroy(e);
        return fail(CVY_E_CUDA, "vocab upload");
    }
    e->vlen_host.assign(vocab_lens, vocab_lens + V);
    for (int i = 0; i < V; ++i)
        if (vocab_lens[i] > kMaxTokenBytes) {
            cvy_engine_destroy(e);
            return fail(CVY_E_INVAL, "vocab entry longer than 16 bytes");
        }
    if (cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking) != cudaSuccess) {
        cvy_engine_destroy(e);
        return fail(CVY_E_CUDA, "stream create");
    }
    e->cur = e->stream;
    e->slots.resize(Bmax);
    for (int p = (int)ec->n_pages - 1; p >= 0; --p) e->free_pages.push_back(p);
    if (const char* tl = getenv("CVY_GEMM_TRACE_LAYER")) {
        e->trace_layer = atoi(tl);
        if (cudaMalloc(&e->d_trace, sizeof(unsigned long long) * kTraceStride * 4 * e->num_sms) != cudaSuccess) {
            cvy_engine_destroy(e);
            return fail(CVY_E_NOMEM, "trace buffer");
        }
        cudaMemset(e->d_trace, 0, sizeof(unsigned long long) * kTraceStride * 4 * e->num_sms);
    }
    e->attn_tc = e->bf16 && (hd == 64 || hd == 128) && (H / Hkv) <= 4;
    if (e->attn_tc) {
        const uint64_t rows = (uint64_t)m->n_layers * ec->n_pages * 2 * Hkv * kPageTokens;
        // hd 128: a 3D view (64 dims, rows, 2 halves; strides 256 B and 128 B) so one TMA box
        // moves a whole 4 KB (page, K/V, kv-head) block (CVY_KV_TMA3D=0: two 2D boxes)
        e->kv_tma3d = hd == 128;
        if (const char* v = getenv("CVY_KV_TMA3D")) e->kv_tma3d = e->kv_tma3d && atoi(v) != 0;
        if (e->kv_tma3d && !make_tmap_kv3(&e->tm_kv, w->kv_pool, rows)) e->kv_tma3d = false;
        if (!e->kv_tma3d && !make_tmap(&e->tm_kv, w->kv_pool, rows, (uint64_t)hd, (uint64_t)hd, 32, 64)) {
            cvy_engine_destroy(e);
            return fail(CVY_E_CUDA, "KV tensor map encode failed");
        }
        e->attn_stages = 2;
        if (const char* as = getenv("CVY_ATTN_STAGES")) e->attn_stages = std::max(2, std::min(6, atoi(as)));
        if (const char* ap = getenv("CVY_ATTN_PPS")) e->attn_pps = atoi(ap) == 2 ? 2 : 4;
        for (const void* f : {(const void*)attention_tc_kernel<128, 2>, (const void*)attention_tc_kernel<128, 3>,
                              (const void*)attention_tc_kernel<128, 4>, (const void*)attention_tc_kernel<64, 2>,
                              (const void*)attention_tc_kernel<64, 3>, (const void*)attention_tc_kernel<64, 4>,
                              (const void*)attention_tc_kernel<128, 2, 2>, (const void*)attention_tc_kernel<128, 4, 2>,
                              (const void*)attention_tc_kernel<128, 6, 2>, (const void*)attention_tc_kernel<64, 2, 2>,
                              (const void*)attention_tc_kernel<64, 4, 2>, (const void*)attention_tc_kernel<64, 6, 2>})
            cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    }
    // kernel attributes
    set_gemm_smem_attrs();
    cudaFuncSetAttribute(gemm_simt_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(gemm_simt_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (cudaDeviceSynchronize() != cudaSuccess) {
        cvy_engine_destroy(e);
        return fail(CVY_E_CUDA, "init sync");
    }
    *out = e;
    return CVY_OK;
}

void cvy_engine_destroy(cvy_engine* e) {
    if (!e) return;
    cudaSetDevice(e->dev);
    if (e->stream) cudaStreamSynchronize(e->stream);
    for (auto& kv : e->buckets) {
        if (kv.second.graph) cudaGraphExecDestroy(kv.second.graph);
        if (kv.second.graph_timed) cudaGraphExecDestroy(kv.second.graph_timed);
        if (kv.second.graph_spans) cudaGraphExecDestroy(kv.second.graph_spans);
        for (cudaEvent_t ev : kv.second.kev) cudaEventDestroy(ev);
    }
    for (auto& pr : e->inflight) {
        cudaEventDestroy(pr.first);
        cudaEventDestroy(pr.second);
    }
    for (auto& pr : e->event_pool) {
        cudaEventDestroy(pr.first);
        cudaEventDestroy(pr.second);
    }
    void* dptrs[] = {e->d_trace, e->d_slots, e->d_page_table, e->d_in_buf, e->d_force_buf, e->d_rope, e->d_x, e->d_act, e->d_q,
                     e->d_o, e->d_h, e->d_ssq, e->d_am, e->d_dbg, e->d_lm_done, e->d_attn_part, e->d_vtab, e->d_vlen,
                     e->d_tools, e->d_ring_tail, e->d_step, e->d_gemm_acc, e->d_tile_cnt, e->d_patches,
                     e->d_px, e->d_pact, e->d_pq, e->d_po, e->d_ph, e->d_pssq, e->d_pattn_part, e->d_prow,
                     e->d_spans};
    for (void* p : dptrs)
        if (p) cudaFree(p);
    void* hptrs[] = {e->h_ring, e->h_ring_tail, e->h_byte_log, e->h_tok_log, e->h_status, e->h_stats};
    for (void* p : hptrs)
        if (p) cudaFreeHost(p);
    if (e->stream) cudaStreamDestroy(e->stream);
    delete e;
}

cvy_status cvy_register_tool(cvy_engine* e, const cvy_tool_desc* t, int32_t* tool_id) {
    if (!e || !t || !tool_id) return fail(CVY_E_INVAL, "null argument");
    if (e->dead) return fail(CVY_E_CUDA, "engine is dead");
    std::lock_guard<std::mutex> lk(e->mu);
    if (e->submitted_any) return fail(CVY_E_STATE, "tools must be registered before the first submit");
    std::string name = t->name ? t->name : "";
    if (name.empty()) return fail(CVY_E_INVAL, "empty tool name");
    for (auto& n : e->tool_names)
        if (n == name) return fail(CVY_E_DUP, "duplicate tool name: " + name);
    if ((int)e->tools.size() >= kMaxTools) return fail(CVY_E_FULL, "too many tools");
    ToolDev td;
    std::memset(&td, 0, sizeof(td));
    td.kind = (int32_t)t->parser;
    td.max_seg = t->max_segment_bytes ? (int32_t)t->max_segment_bytes : 4096;
    if (t->parser == CVY_PARSER_LITERAL) {
        if (t->n_delims < 1 || t->n_delims > 8 || !t->delims || !t->delim_lens)
            return fail(CVY_E_INVAL, "LITERAL needs 1..8 delimiters");
        for (uint32_t i = 0; i < t->n_delims; ++i) {
            uint32_t L = t->delim_lens[i];
            if (L < 1 || L > 8 || !t->delims[i]) return fail(CVY_E_INVAL, "delimiter length must be 1..8");
            uint64_t pack = 0;
            for (uint32_t j = 0; j < L; ++j) pack = (pack << 8) | t->delims[i][j];
            for (uint32_t k = 0; k < i; ++k)
                if ((uint32_t)td.dlen[k] == L && td.dpack[k] == pack) return fail(CVY_E_INVAL, "duplicate delimiter");
            td.dpack[i] = pack;
            td.dmask[i] = L == 8 ? ~0ULL : ((1ULL << (8 * L)) - 1);
            td.dlen[i] = (int32_t)L;
        }
        td.n_delims = (int32_t)t->n_delims;
    } else if (t->parser == CVY_PARSER_JSON_MEMBER || t->parser == CVY_PARSER_JSON_OBJECT) {
        if (t->n_delims != 0) return fail(CVY_E_INVAL, "JSON parsers take no delimiters");
    } else if (t->parser == CVY_PARSER_FENCE || t->parser == CVY_PARSER_CALL) {
        // the open marker ("```" TAG "\n" / "@call " TAG " ") packed little-endian into dpack[0..1]
        const bool fence = t->parser == CVY_PARSER_FENCE;
        if (t->n_delims != 1 || !t->delims || !t->delim_lens || !t->delims[0])
            return fail(CVY_E_INVAL, "FENCE / CALL take exactly one delimiter: the tag");
        const uint32_t L = t->delim_lens[0];
        if (L < 1 || L > 8) return fail(CVY_E_INVAL, "tag length must be 1..8");
        uint8_t marker[16];
        const char* pre = fence ? "```" : "@call ";
        const uint32_t np = fence ? 3 : 6;
        for (uint32_t j = 0; j < np; ++j) marker[j] = (uint8_t)pre[j];
        for (uint32_t j = 0; j < L; ++j) {
            if (t->delims[0][j] == '\n') return fail(CVY_E_INVAL, "tag must not contain a newline");
            marker[np + j] = t->delims[0][j];
        }
        marker[np + L] = fence ? '\n' : ' ';
        const int mlen = (int)(np + L + 1);
        if (td.max_seg < mlen) return fail(CVY_E_INVAL, "max_segment_bytes shorter than the open marker");
        for (int k = 0; k < mlen; ++k) td.dpack[k >> 3] |= (uint64_t)marker[k] << (8 * (k & 7));
        td.dlen[0] = mlen;
        td.n_delims = 1;
    } else if (t->parser == CVY_PARSER_PLAN) {
        if (t->n_delims != 0) return fail(CVY_E_INVAL, "PLAN takes no delimiters");
    } else {
        return fail(CVY_E_INVAL, "unknown parser kind");
    }
    int id = (int)e->tools.size();
    if (cudaMemcpy(e->d_tools + id, &td, sizeof(td), cudaMemcpyHostToDevice) != cudaSuccess)
        return check_cuda(e, cudaErrorUnknown, "tool upload");
    e->tools.push_back(td);
    e->tool_names.push_back(name);
    *tool_id = id;
    return CVY_OK;
}

static bool reserve_pages(cvy_engine* e, SlotHost& sh, int32_t tokens_needed, int slot, std::vector<Upload>& ups) {
    int need_pages = (tokens_needed + kPageTokens - 1) / kPageTokens;
    if (need_pages > (int)e->c.max_pages_per_slot) return false;
    int have = (int)sh.pages.size();
    if (need_pages <= have) return true;
    if ((int)e->free_pages.size() < need_pages - have) return false;
    std::vector<int32_t> added;
    for (int i = have; i < need_pages; ++i) {
        sh.pages.push_back(e->free_pages.back());
        added.push_back(e->free_pages.back());
        e->free_pages.pop_back();
    }
    Upload u;
    u.dst = e->d_page_table + (size_t)slot * e->c.max_pages_per_slot + have;
    u.data.resize(added.size() * sizeof(int32_t));
    std::memcpy(u.data.data(), added.data(), u.data.size());
    ups.push_back(std::move(u));
    sh.reserved = (int32_t)sh.pages.size() * kPageTokens;
    return true;
}

cvy_status cvy_submit_request(cvy_engine* e, const cvy_request_desc* r, uint64_t* req_id) {
    if (!e || !r || !req_id) return fail(CVY_E_INVAL, "null argument");
    if (e->dead) return fail(CVY_E_CUDA, "engine is dead");
    if (r->prompt_len < 1 || !r->prompt) return fail(CVY_E_INVAL, "prompt_len must be >= 1");
    if (r->prompt_len - 1 > e->c.input_cap) return fail(CVY_E_INVAL, "prompt longer than input_cap + 1");
    if (r->forced_len > e->c.forced_cap || (r->forced_len && !r->forced)) return fail(CVY_E_INVAL, "bad forced stream");
    if (r->max_new_tokens < 1) return fail(CVY_E_INVAL, "max_new_tokens must be >= 1");
    for (uint32_t i = 0; i < r->prompt_len; ++i)
        if (r->prompt[i] < 0 || r->prompt[i] >= e->m.vocab) return fail(CVY_E_INVAL, "prompt token out of range");
    for (uint32_t i = 0; i < r->forced_len; ++i)
        if (r->forced[i] < 0 || r->forced[i] >= e->m.vocab) return fail(CVY_E_INVAL, "forced token out of range");
    std::lock_guard<std::mutex> lk(e->mu);
    if (r->tool_id < -1 || r->tool_id >= (int)e->tools.size()) return fail(CVY_E_NOTFOUND, "unknown tool id");
    // region tool set (NEXT-2, R24); a single FENCE / CALL tool is the set of one
    uint64_t tool_set = 0;
    int32_t set_max_seg = 0;
    int32_t tool_primary = r->tool_id;
    {
        std::vector<int32_t> ids;
        if (r->n_tool_set > 0) {
            if (!r->tool_set || r->n_tool_set > 64) return fail(CVY_E_INVAL, "tool_set: 1..64 tool ids");
            ids.assign(r->tool_set, r->tool_set + r->n_tool_set);
        } else if (r->tool_id >= 0 && (e->tools[r->tool_id].kind == CVY_PARSER_FENCE ||
                                       e->tools[r->tool_id].kind == CVY_PARSER_CALL)) {
            ids.push_back(r->tool_id);
        }
        int32_t max_marker = 0;
        set_max_seg = 1 << 30;
        for (int32_t id : ids) {
            if (id < 0 || id >= (int)e->tools.size() || id >= 64) return fail(CVY_E_NOTFOUND, "tool_set: unknown tool id");
            const ToolDev& t = e->tools[id];
            if (t.kind != CVY_PARSER_FENCE && t.kind != CVY_PARSER_CALL)
                return fail(CVY_E_INVAL, "tool_set: only FENCE and CALL tools select themselves by marker");
            if (tool_set & (1ull << id)) return fail(CVY_E_INVAL, "tool_set: duplicate tool id");
            tool_set |= 1ull << id;
            set_max_seg = std::min(set_max_seg, t.max_seg);
            max_marker = std::max(max_marker, t.dlen[0]);
        }
        if (!ids.empty()) {
            if (set_max_seg < max_marker) return fail(CVY_E_INVAL, "tool_set: a marker is longer than the smallest max_segment_bytes");
            if (r->n_tool_set > 0 && r->tool_id >= 0 && !(tool_set & (1ull << r->tool_id)))
                return fail(CVY_E_INVAL, "tool_id is not a member of tool_set");
            if (tool_primary < 0) tool_primary = ids[0];
        }
    }
    int slot = -1;
    for (int b = 0; b < (int)e->c.max_slots; ++b)
        if (!e->slots[b].used) {
            slot = b;
            break;
        }
    if (slot < 0) return fail(CVY_E_FULL, "no free slot");
    SlotHost sh;
    const uint32_t gen = r->forced_len ? std::min(r->forced_len, r->max_new_tokens) : r->max_new_tokens;
    const int32_t need = (int32_t)(r->synth_prefix_len + r->prompt_len + gen + 1 + r->reserve_tokens);
    std::vector<Upload> ups;
    if (!reserve_pages(e, sh, need, slot, ups)) {
        for (int32_t p : sh.pages) e->free_pages.push_back(p);
        return fail(CVY_E_FULL, "not enough KV pages");
    }
    // the synthetic prefix is written by cvy_step (after this slot's page-table upload, before
    // its first step), so submit never touches the stream a step graph may be capturing on
    if (r->synth_prefix_len) e->synth_pending.push_back(SynthJob{slot, r->synth_prefix_len, r->synth_seed});
    for (auto& u : ups) e->uploads.push_back(std::move(u));
    // chunked prefill (NEXT-1): all prompt tokens but the last run as one batched pass at the
    // next step boundary; the slot then starts at the last prompt token
    const bool prefill = (e->c.flags & CVY_ENGINE_CHUNKED_PREFILL) && e->d_prow && r->prompt_len > 1;
    if (prefill) {
        PrefillJob j;
        j.slot = slot;
        j.pos0 = (int32_t)r->synth_prefix_len;
        j.toks.assign(r->prompt, r->prompt + r->prompt_len - 1);
        e->prefill_pending.push_back(std::move(j));
    } else if (r->prompt_len > 1) {
        Upload u;
        u.dst = e->d_in_buf + (size_t)slot * e->c.input_cap;
        u.data.resize((r->prompt_len - 1) * sizeof(int32_t));
        std::memcpy(u.data.data(), r->prompt + 1, u.data.size());
        e->uploads.push_back(std::move(u));
    }
    if (r->forced_len) {
        Upload u;
        u.dst = e->d_force_buf + (size_t)slot * e->c.forced_cap;
        u.data.resize(r->forced_len * sizeof(int32_t));
        std::memcpy(u.data.data(), r->forced, u.data.size());
        e->uploads.push_back(std::move(u));
    }
    Patch p;
    std::memset(&p, 0, sizeof(p));
    p.kind = PATCH_SUBMIT;
    p.slot = slot;
    p.req_id = e->next_req++;
    p.tool = (e->c.flags & CVY_ENGINE_SCAN_OFF) ? -1 : tool_primary;
    p.tool_set = (e->c.flags & CVY_ENGINE_SCAN_OFF) ? 0 : tool_set;
    p.set_max_seg = set_max_seg;
    p.pos = (int32_t)r->synth_prefix_len + (prefill ? (int32_t)r->prompt_len - 1 : 0);
    p.cur_tok = prefill ? r->prompt[r->prompt_len - 1] : r->prompt[0];
    p.in_idx = 0;
    p.in_len = prefill ? 0 : (int32_t)r->prompt_len - 1;
    p.max_new = (int32_t)r->max_new_tokens;
    p.force_len = (int32_t)r->forced_len;
    p.max_pos = sh.reserved;
    e->pending.push_back(p);
    sh.used = true;
    sh.req_id = p.req_id;
    sh.state = 0;
    sh.final_pending = true;
    sh.next_pos = (int32_t)(r->synth_prefix_len + r->prompt_len + gen);
    sh.round_pos0 = p.pos;
    sh.round_inputs = 1 + p.in_len;
    e->slots[slot] = std::move(sh);
    e->req_slot[p.req_id] = slot;
    e->submitted_any = true;
    *req_id = p.req_id;
    return CVY_OK;
}

cvy_status cvy_inject_observation(cvy_engine* e, uint64_t req_id, const int32_t* tokens, uint32_t n,
                                  uint32_t max_new_tokens, const int32_t* forced, uint32_t forced_len) {
    if (!e || (n && !tokens) || (forced_len && !forced)) return fail(CVY_E_INVAL, "null argument");
    if (e->dead) return fail(CVY_E_CUDA, "engine is dead");
    if (n > e->c.input_cap || forced_len > e->c.forced_cap) return fail(CVY_E_INVAL, "observation too long");
    if (max_new_tokens < 1) return fail(CVY_E_INVAL, "max_new_tokens must be >= 1");
    for (uint32_t i = 0; i < n; ++i)
        if (tokens[i] < 0 || tokens[i] >= e->m.vocab) return fail(CVY_E_INVAL, "token out of range");
    for (uint32_t i = 0; i < forced_len; ++i)
        if (forced[i] < 0 || forced[i] >= e->m.vocab) return fail(CVY_E_INVAL, "forced token out of range");
    std::lock_guard<std::mutex> lk(e->mu);
    auto it = e->req_slot.find(req_id);
    if (it == e->req_slot.end()) return fail(CVY_E_NOTFOUND, "unknown request");
    const int slot = it->second;
    SlotHost& sh = e->slots[slot];
    if (sh.state != 1) return fail(CVY_E_STATE, "request is not parked after a polled FINAL");
    const uint32_t gen = forced_len ? std::min(forced_len, max_new_tokens) : max_new_tokens;
    std::vector<Upload> ups;
    const int32_t need = sh.next_pos + 1 + (int32_t)n + (int32_t)gen + 1;
    if (!reserve_pages(e, sh, need, slot, ups)) return fail(CVY_E_FULL, "not enough KV pages for the next round");
    for (auto& u : ups) e->uploads.push_back(std::move(u));
    // the round just parked: its last generated token is the next input (R19) at
    // pos_end = round_pos0 + round_inputs + gen - 1
    const uint32_t gen_done = e->h_status[slot].gen;
    const bool prefill = (e->c.flags & CVY_ENGINE_CHUNKED_PREFILL) && e->d_prow && n >= 1 && gen_done >= 1 &&
                         gen_done <= e->c.round_tokens;
    int32_t pos_end = 0;
    if (prefill) {
        // prefill [last generated token, obs[0..n-2]]; the slot resumes at obs[n-1]
        pos_end = sh.round_pos0 + sh.round_inputs + (int32_t)gen_done - 1;
        PrefillJob j;
        j.slot = slot;
        j.pos0 = pos_end;
        j.toks.push_back(e->h_tok_log[(size_t)slot * e->c.round_tokens + gen_done - 1]);
        j.toks.insert(j.toks.end(), tokens, tokens + n - 1);
        e->prefill_pending.push_back(std::move(j));
    } else if (n) {
        Upload u;
        u.dst = e->d_in_buf + (size_t)slot * e->c.input_cap;
        u.data.resize(n * sizeof(int32_t));
        std::memcpy(u.data.data(), tokens, u.data.size());
        e->uploads.push_back(std::move(u));
    }
    if (forced_len) {
        Upload u;
        u.dst = e->d_force_buf + (size_t)slot * e->c.forced_cap;
        u.data.resize(forced_len * sizeof(int32_t));
        std::memcpy(u.data.data(), forced, u.data.size());
        e->uploads.push_back(std::move(u));
    }
    Patch p;
    std::memset(&p, 0, sizeof(p));
    p.kind = PATCH_INJECT;
    p.slot = slot;
    p.req_id = req_id;
    p.in_len = prefill ? 0 : (int32_t)n;
    if (prefill) {
        p.set_pos = 1;
        p.pos = pos_end + (int32_t)n;
        p.cur_tok = tokens[n - 1];
    }
    p.max_new = (int32_t)max_new_tokens;
    p.force_len = (int32_t)forced_len;
    p.max_pos = sh.reserved;
    e->pending.push_back(p);
    sh.state = 0;
    sh.final_seen = false;
    sh.final_pending = true;
    sh.cancel_pending = false;
    sh.next_pos = sh.next_pos + 1 + (int32_t)n + (int32_t)gen;
    if (prefill) {
        sh.round_pos0 = pos_end + (int32_t)n;
        sh.round_inputs = 1;
    } else {
        sh.round_pos0 = sh.round_pos0 + sh.round_inputs + (int32_t)gen_done - 1;
        sh.round_inputs = 1 + (int32_t)n;
    }
    return CVY_OK;
}

cvy_status cvy_cancel_request(cvy_engine* e, uint64_t req_id) {
    if (!e) return fail(CVY_E_INVAL, "null engine");
    std::lock_guard<std::mutex> lk(e->mu);
    auto it = e->req_slot.find(req_id);
    if (it == e->req_slot.end()) return fail(CVY_E_NOTFOUND, "unknown request");
    SlotHost& sh = e->slots[it->second];
    if (sh.state != 0 || sh.cancel_pending) return CVY_OK;  // idempotent: parked, cancelled or queued
    sh.cancel_pending = true;
    Patch p;
    std::memset(&p, 0, sizeof(p));
    p.kind = PATCH_CANCEL;
    p.slot = it->second;
    p.req_id = req_id;
    e->pending.push_back(p);
    return CVY_OK;
}

cvy_status cvy_release_request(cvy_engine* e, uint64_t req_id) {
    if (!e) return fail(CVY_E_INVAL, "null engine");
    std::lock_guard<std::mutex> lk(e->mu);
    auto it = e->req_slot.find(req_id);
    if (it == e->req_slot.end()) return fail(CVY_E_NOTFOUND, "unknown request");
    const int slot = it->second;
    SlotHost& sh = e->slots[slot];
    if (sh.state == 0) return fail(CVY_E_STATE, "request still running (cancel it or wait for FINAL)");
    Patch p;
    std::memset(&p, 0, sizeof(p));
    p.kind = PATCH_RELEASE;
    p.slot = slot;
    p.req_id = req_id;
    e->pending.push_back(p);
    for (int32_t pg : sh.pages) e->free_pages.push_back(pg);
    e->req_slot.erase(it);
    e->slots[slot] = SlotHost();
    return CVY_OK;
}

int32_t cvy_request_state(cvy_engine* e, uint64_t req_id) {
    if (!e) return -1;
    std::lock_guard<std::mutex> lk(e->mu);
    auto it = e->req_slot.find(req_id);
    if (it == e->req_slot.end()) return -1;
    return e->slots[it->second].state;
}

}  // extern "C"

// ============================================================================ step graph
namespace {

cvy_status launch_k(cvy_engine* e, const void* func, dim3 grid, dim3 block, size_t smem, void** args, bool pdl,
                    int cluster = 1) {
    cudaLaunchConfig_t cfg;
    std::memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = e->cur ? e->cur : e->stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (pdl && !(e->c.flags & CVY_ENGINE_NO_PDL) && !e->capturing_timed) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (cluster > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = (unsigned)cluster;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaError_t err = cudaLaunchKernelExC(&cfg, func, args);
    if (err != cudaSuccess) return fail(CVY_E_CUDA, std::string("launch: ") + cudaGetErrorString(err));
    return CVY_OK;
}

StepParams base_params(cvy_engine* e, int Bp) {
    StepParams P;
    std::memset(&P, 0, sizeof(P));
    const cvy_model_config& m = e->m;
    P.L = m.n_layers;
    P.d = m.d_model;
    P.H = m.n_heads;
    P.Hkv = m.n_kv_heads;
    P.hd = m.head_dim;
    P.dff = m.d_ff;
    P.V = m.vocab;
    P.eos = m.eos_id;
    P.eps = m.rms_eps;
    P.Bp = Bp;
    P.Bmax = (int)e->slots.size();
    P.n_pages = (int)e->c.n_pages;
    P.max_pages = (int)e->c.max_pages_per_slot;
    P.act_ld = e->act_ld;
    P.act_plane = e->bf16 ? (int64_t)e->slots.size() * e->act_ld : 0;
    P.slots = e->d_slots;
    P.page_table = e->d_page_table;
    P.in_buf = e->d_in_buf;
    P.input_cap = (int)e->c.input_cap;
    P.force_buf = e->d_force_buf;
    P.forced_cap = (int)e->c.forced_cap;
    P.rope = e->d_rope;
    P.max_rope_pos = e->max_rope_pos;
    P.embed = e->w.embed;
    P.attn_norm = e->w.attn_norm;
    P.mlp_norm = e->w.mlp_norm;
    P.final_norm = e->w.final_norm;
    P.kv_pool = e->w.kv_pool;
    P.x = e->d_x;
    P.act = e->d_act;
    P.q = e->d_q;
    P.o = e->d_o;
    P.h = e->d_h;
    P.ssq = e->d_ssq;
    P.am_keys = e->d_am;
    P.dbg_logits = e->d_dbg;
    P.lm_done = e->d_lm_done;
    P.attn_part = e->d_attn_part;
    // split-KV only when the (head, row) grid cannot cover the SMs: measured at B=64 / ctx 372
    // on 7B, splits=1 beats 2 by 0.4 ms/step (the merge pass costs more than the extra waves).
    const int cells = m.n_kv_heads * Bp;
    const int want = cells >= e->num_sms ? 1 : (2 * e->num_sms + cells - 1) / cells;
    P.attn_splits = std::max(1, std::min(e->attn_splits_max, want));
    if (const char* as = getenv("CVY_ATTN_SPLITS")) P.attn_splits = std::max(1, std::min(e->attn_splits_max, atoi(as)));
    P.kv_tma3d = e->kv_tma3d ? 1 : 0;
    P.attn_early = 0;  // measured neutral; off keeps the in-graph spans clean
    if (const char* v = getenv("CVY_ATTN_EARLY")) P.attn_early = atoi(v);  // A/B knob
    P.vtab = e->d_vtab;
    P.vlen = e->d_vlen;
    P.tools = e->d_tools;
    P.ring = e->dm_ring;
    P.ring_mask = e->c.ring_records - 1;
    P.ring_tail_dev = e->d_ring_tail;
    P.ring_tail_host = reinterpret_cast<unsigned long long*>(e->dm_ring_tail);
    P.byte_log = reinterpret_cast<uint8_t*>(e->dm_byte_log);
    P.round_bytes = e->c.round_bytes;
    P.tok_log = reinterpret_cast<int32_t*>(e->dm_tok_log);
    P.round_tokens = e->c.round_tokens;
    P.status = reinterpret_cast<SlotStatus*>(e->dm_status);
    P.stats = reinterpret_cast<StepStats*>(e->dm_stats);
    P.step_ctr = e->d_step;
    P.scan_off = (e->c.flags & CVY_ENGINE_SCAN_OFF) ? 1 : 0;
    return P;
}


// plan one GEMM: W rows N per layer, K, epilogue
bool plan_gemm(cvy_engine* e, Bucket& bk, const void* Wbase, int N, int K, int layer, int L_rows_total, const void* X,
               EpiArgs epi, GemmPlan* out, std::string* why, int xcap = 0) {
    if (xcap <= 0) xcap = (int)e->slots.size();  // activation buffer rows (planes are xcap rows apart)
    GemmPlan gp;
    std::memset(&gp, 0, sizeof(gp));
    const int Bp = bk.Bp;
    const int sms = e->num_sms;
    gp.W = Wbase;
    gp.X = X;
    gp.w_row0 = (int64_t)layer * N;
    GemmTC& g = gp.g;
    g.N = N;
    g.K = K;
    g.epi = epi;
    if (e->bf16) {
        // gate/up: optionally stream-K over every SM instead of 112 whole 256-row tiles (A/B knob)
        bool gu_sk = epi.kind == EPI_SWIGLU && getenv("CVY_GU_STREAMK") && atoi(getenv("CVY_GU_STREAMK")) != 0;
        int gu_nsub = (epi.kind == EPI_SWIGLU && getenv("CVY_GU_NSUB")) ? atoi(getenv("CVY_GU_NSUB")) : 0;
        // A/B knob: stream-K for the epilogue kinds in the bit mask CVY_SK_KINDS (1 << EpiKind),
        // with CVY_SK_NSUB 128-row sub-tiles per tile
        if (const char* v = getenv("CVY_SK_KINDS"))
            if (Bp > 128 && ((atoi(v) >> epi.kind) & 1) &&
                K <= (getenv("CVY_SK_MAXK") ? atoi(getenv("CVY_SK_MAXK")) : 1 << 30)) {
                gu_sk = true;
                if (const char* ns = getenv("CVY_SK_NSUB")) gu_nsub = atoi(ns);
            }
        if (!gemm_config(g, N, K, Bp, sms, &gp.grid, &gp.smem, why, epi.kind != EPI_LMHEAD, gu_sk, gu_nsub,
                         gemm_epi_groups(epi.kind), gemm_pair_ok(epi.kind), epi.kind != EPI_RESID))
            return false;
        g.w_row0 = layer * N;
        if (e->d_trace && layer == e->trace_layer && epi.kind != EPI_LMHEAD && xcap == (int)e->slots.size()) {
            const int k = epi.kind == EPI_QKV ? 0 : epi.kind == EPI_SWIGLU ? 2 : (K == ::m_d(e) ? 1 : 3);
            g.trace = e->d_trace + (size_t)k * kTraceStride * e->num_sms;
        }
        g.part = e->d_gemm_acc;
        g.tile_cnt = e->d_tile_cnt;
        // measurement knob (wrong results): the gate/up epilogue's debug bits (GemmTC::dbg)
        if (const char* dg = getenv("CVY_GEMM_DBG_GU"))
            if (epi.kind == EPI_SWIGLU) g.dbg = atoi(dg);
        if (const char* dg = getenv("CVY_GEMM_DBG_ALL"))  // every projection but the LM head
            if (epi.kind != EPI_LMHEAD) g.dbg = atoi(dg);
        g.x_plane_rows = (int32_t)xcap;
        g.wtiled = e->w_tiled && (Wbase == e->w.wqkv || Wbase == e->w.wo || Wbase == e->w.wgu || Wbase == e->w.wd ||
                                  (Wbase == e->w.lm_head && lm_head_tiled(&e->m)));
        if (g.wtiled && g.bk != 64) {
            *why = "tile-major weights need 64-element k-blocks (batch tiles of <= 128 columns)";
            return false;
        }
        // tile-major: a [rows * K / 64][64] view, box = one 128-row x 64-column tile (16 KB)
        if (!(g.wtiled ? make_tmap(&gp.tmW, Wbase, (uint64_t)L_rows_total * K / 64, 64, 64, 128, 64)
                       : make_tmap(&gp.tmW, Wbase, (uint64_t)L_rows_total, (uint64_t)K, (uint64_t)K,
                                   (uint32_t)(128 * g.nsub), (uint32_t)g.bk))) {
            *why = "cuTensorMapEncodeTiled (weights) failed";
            return false;
        }
        const uint32_t xrows = g.merge ? (uint32_t)g.bq : (uint32_t)g.mma_n;
        if (!make_tmap(&gp.tmX, X, (uint64_t)(2 * xcap), (uint64_t)K, (uint64_t)e->act_ld, xrows,
                       (uint32_t)g.bk)) {
            *why = "cuTensorMapEncodeTiled (activations) failed";
            return false;
        }
    } else {
        g.nsub = (epi.kind == EPI_SWIGLU) ? 2 : 1;
        g.tiles = (N + 128 * g.nsub - 1) / (128 * g.nsub);
        gp.grid = g.tiles;
        gp.smem = (size_t)(128 * kEsmLd + 4 + 4 * Bp + 32 * K) * sizeof(float);
    }
    *out = gp;
    return true;
}

cvy_status build_bucket(cvy_engine* e, int Bp, Bucket** out) {
    auto it = e->buckets.find(Bp);
    if (it != e->buckets.end()) {
        *out = &it->second;
        return CVY_OK;
    }
    Bucket bk;
    bk.Bp = Bp;
    bk.nsub = Bp <= 128 ? 2 : 1;
    bk.P = base_params(e, Bp);
    const cvy_model_config& m = e->m;
    const int L = m.n_layers, d = m.d_model, H = m.n_heads, Hkv = m.n_kv_heads, hd = m.head_dim, dff = m.d_ff,
              V = m.vocab;
    const int Nqkv = (H + 2 * Hkv) * hd;
    std::string why;
    for (int l = 0; l < L; ++l) {
        GemmPlan gp;
        EpiArgs eq{EPI_QKV, l, Nqkv, nullptr, nullptr, 1};
        if (!plan_gemm(e, bk, e->w.wqkv, Nqkv, d, l, L * Nqkv, e->d_act, eq, &gp, &why)) return fail(CVY_E_INVAL, why);
        bk.plans.push_back(gp);
        EpiArgs eo{EPI_RESID, l, d, e->w.mlp_norm + (size_t)l * d, nullptr, 4};
        if (!plan_gemm(e, bk, e->w.wo, d, H * hd, l, L * d, e->d_o, eo, &gp, &why)) return fail(CVY_E_INVAL, why);
        bk.plans.push_back(gp);
        EpiArgs eg{EPI_SWIGLU, l, 2 * dff, nullptr, nullptr, 5};
        if (!plan_gemm(e, bk, e->w.wgu, 2 * dff, d, l, L * 2 * dff, e->d_act, eg, &gp, &why)) return fail(CVY_E_INVAL, why);
        bk.plans.push_back(gp);
        EpiArgs ed{EPI_RESID, l, d, (l + 1 < L) ? e->w.attn_norm + (size_t)(l + 1) * d : e->w.final_norm, nullptr, 6};
        if (!plan_gemm(e, bk, e->w.wd, d, dff, l, L * d, e->d_h, ed, &gp, &why)) return fail(CVY_E_INVAL, why);
        bk.plans.push_back(gp);
    }
    {
        GemmPlan gp;
        EpiArgs el{EPI_LMHEAD, 0, V, nullptr, nullptr, 7};
        if (!plan_gemm(e, bk, e->w.lm_head, V, d, 0, V, e->d_act, el, &gp, &why)) return fail(CVY_E_INVAL, why);
        bk.plans.push_back(gp);
    }
    // cross-kernel weight prefetch: GEMM i warms L2 with the first k-blocks of GEMM i+1 (the LM
    // head warms the next step's layer-0 QKV) while its own epilogue drains
    if (e->bf16) {
        int pf_kb = 0;  // measured at B=64: 128 KB -1%, 256 KB -2% (the prefetch competes, nothing idles)
        if (const char* pk = getenv("CVY_GEMM_PF_KB")) pf_kb = atoi(pk);
        const size_t n = bk.plans.size();
        for (size_t i = 0; i < n; ++i) {
            GemmPlan& a = bk.plans[i];
            const GemmPlan& b = bk.plans[(i + 1) % n];
            GemmNext& nx = a.g.nx;
            nx.tiles = b.g.tiles;
            nx.kblocks = b.g.kblocks;
            nx.split = b.g.split;
            nx.rows_per_tile = 128 * b.g.nsub;
            nx.w_row0 = b.g.w_row0;
            nx.grid = b.grid;
            nx.bk = b.g.bk;
            nx.blocks = b.g.wtiled ? 0 : std::max(0, pf_kb * 1024 / (nx.rows_per_tile * nx.bk * 2));
            a.tmN = b.tmW;
        }
    }
    auto res = e->buckets.emplace(Bp, std::move(bk));
    *out = &res.first->second;
    return CVY_OK;
}

cvy_status launch_gemm(cvy_engine* e, Bucket& bk, GemmPlan& gp, StepParams* Pq = nullptr) {
    if (e->bf16) {
        void* args[] = {&gp.tmW, &gp.tmX, Pq ? Pq : &bk.P, &gp.g, &gp.tmN};
        return launch_k(e, gemm_tc_kernel_ptr<__nv_bfloat16>(gp.g.nsub, gp.g.merge != 0, gp.g.bk, gp.g.epi.kind, gp.g.pair != 0),
                        dim3(gp.grid, gp.g.nbt), dim3(gemm_launch_threads(gp.g.epi.kind, gp.g.split)), gp.smem, args, true,
                        gp.g.pair ? 2 : (gp.g.split > 1 ? gp.g.split : 1));
    }
    const float* W = (const float*)gp.W;
    const float* X = (const float*)gp.X;
    int64_t w_row0 = gp.w_row0;
    int K = gp.g.K, nsub = gp.g.nsub, tiles = gp.g.tiles;
    EpiArgs E = gp.g.epi;
    void* args[] = {&bk.P, &W, &w_row0, &X, &K, &nsub, &tiles, &E};
    return launch_k(e, (const void*)gemm_simt_kernel<float>, dim3(gp.grid), dim3(128), gp.smem, args, true);
}

// Event pair around a launch when building the timed graph variant.
struct KTimer {
    cvy_engine* e;
    Bucket& bk;
    size_t i = 0;
    KTimer(cvy_engine* e_, Bucket& b) : e(e_), bk(b) {}
    void begin(int kind, int layer) {
        if (!e->capturing_timed) return;
        if (bk.kev.size() < 2 * (i + 1)) {
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            bk.kev.push_back(a);
            bk.kev.push_back(b);
            bk.kinfo.push_back({kind, layer});
        }
        cudaEventRecordWithFlags(bk.kev[2 * i], e->cur ? e->cur : e->stream, cudaEventRecordExternal);
    }
    void end() {
        if (!e->capturing_timed) return;
        cudaEventRecordWithFlags(bk.kev[2 * i + 1], e->cur ? e->cur : e->stream, cudaEventRecordExternal);
        ++i;
    }
};

// Paged attention of one layer for every row of the bucket (+ the split-KV merge).
cvy_status launch_attention(cvy_engine* e, Bucket& bk, int l, KTimer* kt, StepParams* Pq = nullptr) {
    StepParams& P = Pq ? *Pq : bk.P;
    cvy_status st;
    const cvy_model_config& m = e->m;
    const int Bp = P.Bp;
    const int G = m.n_heads / m.n_kv_heads;
    const size_t attn_smem = sizeof(float) * (G * m.head_dim + G * kAttnThreads + 3 * kAttnMaxG + 4 * kAttnMaxG);
    int layer = l;
    void* aargs[] = {&P, &layer};
    if (e->attn_tc) {
        void* targs[] = {&e->tm_kv, &P, &layer};
        const int pps = e->attn_pps;
        const int nst = pps == 2 ? (e->attn_stages <= 2 ? 2 : e->attn_stages >= 6 ? 6 : 4) : e->attn_stages;
        const void* tf;
        if (pps == 2)
            tf = m.head_dim == 128 ? (nst <= 2 ? (const void*)attention_tc_kernel<128, 2, 2>
                                                : nst >= 6 ? (const void*)attention_tc_kernel<128, 6, 2>
                                                           : (const void*)attention_tc_kernel<128, 4, 2>)
                                    : (nst <= 2 ? (const void*)attention_tc_kernel<64, 2, 2>
                                                : nst >= 6 ? (const void*)attention_tc_kernel<64, 6, 2>
                                                           : (const void*)attention_tc_kernel<64, 4, 2>);
        else
            tf = m.head_dim == 128 ? (nst == 2 ? (const void*)attention_tc_kernel<128, 2>
                                                : nst == 4 ? (const void*)attention_tc_kernel<128, 4>
                                                           : (const void*)attention_tc_kernel<128, 3>)
                                    : (nst == 2 ? (const void*)attention_tc_kernel<64, 2>
                                                : nst == 4 ? (const void*)attention_tc_kernel<64, 4>
                                                           : (const void*)attention_tc_kernel<64, 3>);
        const int blk = kPageTokens * m.head_dim * 2;
        const size_t tsmem = 1024 + (size_t)nst * pps * 2 * blk + kAtcWarps * 8 * 16 * 2 +
                             (size_t)kAtcWarps * (8 + 4 * m.head_dim) * 4 + 2 * nst * 8;
        if ((st = launch_k(e, tf, dim3(m.n_kv_heads, Bp, P.attn_splits), dim3(kAtcThreads), tsmem, targs, true)) !=
            CVY_OK)
            return st;
    } else {
        const void* af = e->bf16 ? (const void*)attention_kernel<__nv_bfloat16> : (const void*)attention_kernel<float>;
        if ((st = launch_k(e, af, dim3(m.n_kv_heads, Bp, P.attn_splits), dim3(kAttnThreads), attn_smem, aargs,
                           true)) != CVY_OK)
            return st;
    }
    if (kt) kt->end();
    if (P.attn_splits > 1) {
        void* margs[] = {&P};
        const void* mf =
            e->bf16 ? (const void*)attention_merge_kernel<__nv_bfloat16> : (const void*)attention_merge_kernel<float>;
        if (kt) kt->begin(3, l);
        if ((st = launch_k(e, mf, dim3(m.n_kv_heads, Bp), dim3(128), 0, margs, true)) != CVY_OK) return st;
        if (kt) kt->end();
    }
    return CVY_OK;
}

// ------------------------------------------------------------------ chunked prefill (NEXT-1)
// A prefill bucket: the per-layer projection plans over the prefill activation buffers
// (kPrefillRows rows) and a StepParams whose rows map to (slot, position, token).
cvy_status build_prefill_bucket(cvy_engine* e, int Bp, Bucket** out) {
    auto it = e->prefill_buckets.find(Bp);
    if (it != e->prefill_buckets.end()) {
        *out = &it->second;
        return CVY_OK;
    }
    Bucket bk;
    bk.Bp = Bp;
    bk.P = base_params(e, Bp);
    StepParams& P = bk.P;
    P.Bmax = kPrefillRows;
    P.act_plane = (int64_t)kPrefillRows * e->act_ld;
    P.x = e->d_px;
    P.act = e->d_pact;
    P.q = e->d_pq;
    P.o = e->d_po;
    P.h = e->d_ph;
    P.ssq = e->d_pssq;
    P.attn_part = e->d_pattn_part;
    P.dbg_logits = nullptr;
    P.row_slot = e->d_prow;
    P.row_pos = e->d_prow + kPrefillRows;
    P.row_tok = e->d_prow + 2 * kPrefillRows;
    const cvy_model_config& m = e->m;
    const int L = m.n_layers, d = m.d_model, H = m.n_heads, Hkv = m.n_kv_heads, hd = m.head_dim, dff = m.d_ff;
    const int Nqkv = (H + 2 * Hkv) * hd;
    std::string why;
    for (int l = 0; l < L; ++l) {
        GemmPlan gp;
        EpiArgs eq{EPI_QKV, l, Nqkv, nullptr};
        if (!plan_gemm(e, bk, e->w.wqkv, Nqkv, d, l, L * Nqkv, e->d_pact, eq, &gp, &why, kPrefillRows))
            return fail(CVY_E_INVAL, why);
        bk.plans.push_back(gp);
        EpiArgs eo{EPI_RESID, l, d, e->w.mlp_norm + (size_t)l * d};
        if (!plan_gemm(e, bk, e->w.wo, d, H * hd, l, L * d, e->d_po, eo, &gp, &why, kPrefillRows))
            return fail(CVY_E_INVAL, why);
        bk.plans.push_back(gp);
        EpiArgs eg{EPI_SWIGLU, l, 2 * dff, nullptr};
        if (!plan_gemm(e, bk, e->w.wgu, 2 * dff, d, l, L * 2 * dff, e->d_pact, eg, &gp, &why, kPrefillRows))
            return fail(CVY_E_INVAL, why);
        bk.plans.push_back(gp);
        EpiArgs ed{EPI_RESID, l, d, (l + 1 < L) ? e->w.attn_norm + (size_t)(l + 1) * d : e->w.final_norm};
        if (!plan_gemm(e, bk, e->w.wd, d, dff, l, L * d, e->d_ph, ed, &gp, &why, kPrefillRows))
            return fail(CVY_E_INVAL, why);
        bk.plans.push_back(gp);
    }
    auto res = e->prefill_buckets.emplace(Bp, std::move(bk));
    *out = &res.first->second;
    return CVY_OK;
}

// Run the queued prefill jobs: rows (slot, pos, token) in passes of <= kPrefillRows, each
// pass = embed + L x (QKV + RoPE + KV append, attention over keys [0, pos], O, gate/up, down);
// no LM head (the slot resumes at its last prompt token in the next decode step).
cvy_status enqueue_prefill(cvy_engine* e, const std::vector<PrefillJob>& jobs) {
    std::vector<int32_t> rs, rp, rt;
    for (const auto& j : jobs)
        for (size_t i = 0; i < j.toks.size(); ++i) {
            rs.push_back(j.slot);
            rp.push_back(j.pos0 + (int32_t)i);
            rt.push_back(j.toks[i]);
        }
    cvy_status st;
    for (size_t r0 = 0; r0 < rs.size(); r0 += kPrefillRows) {
        const int n = (int)std::min<size_t>(kPrefillRows, rs.size() - r0);
        int Bp = 32;
        while (Bp < n) Bp *= 2;
        Bucket* bk = nullptr;
        if ((st = build_prefill_bucket(e, Bp, &bk)) != CVY_OK) return st;
        std::vector<int32_t> tab(3 * (size_t)kPrefillRows, 0);
        for (int i = 0; i < kPrefillRows; ++i) tab[kPrefillRows + i] = -1;  // padding rows
        for (int i = 0; i < n; ++i) {
            tab[i] = rs[r0 + i];
            tab[kPrefillRows + i] = rp[r0 + i];
            tab[2 * kPrefillRows + i] = rt[r0 + i];
        }
        if ((st = check_cuda(e, cudaMemcpyAsync(e->d_prow, tab.data(), tab.size() * sizeof(int32_t),
                                                cudaMemcpyHostToDevice, e->stream),
                             "prefill rows")) != CVY_OK)
            return st;
        // (pageable source: cudaMemcpyAsync stages it before returning, as for the uploads)
        void* args[] = {&bk->P};
        if ((st = launch_k(e, (const void*)embed_kernel<__nv_bfloat16>, dim3(Bp), dim3(128), 0, args, true)) != CVY_OK)
            return st;
        size_t pi = 0;
        for (int l = 0; l < e->m.n_layers; ++l) {
            if ((st = launch_gemm(e, *bk, bk->plans[pi++])) != CVY_OK) return st;
            if ((st = launch_attention(e, *bk, l, nullptr)) != CVY_OK) return st;
            for (int k = 0; k < 3; ++k)
                if ((st = launch_gemm(e, *bk, bk->plans[pi++])) != CVY_OK) return st;
        }
        e->prefill_rows_total += (uint64_t)n;
    }
    return CVY_OK;
}

cvy_status enqueue_step_kernels(cvy_engine* e, Bucket& bk) {
    cvy_status st;
    uint32_t launches = 0;
    KTimer kt(e, bk);
    const int Bp = bk.Bp;
    const cvy_model_config& m = e->m;
    if (e->capturing_spans) {
        if ((st = check_cuda(e, cudaMemsetAsync(e->d_spans, 0xFF, sizeof(unsigned long long) * kSpanSlots, e->stream),
                             "span reset")) != CVY_OK ||
            (st = check_cuda(e, cudaMemsetAsync(e->d_spans + kSpanSlots, 0, sizeof(unsigned long long) * kSpanSlots,
                                                e->stream), "span reset")) != CVY_OK)
            return st;
    }
    {
        void* args[] = {&bk.P};
        const void* f = e->bf16 ? (const void*)embed_kernel<__nv_bfloat16> : (const void*)embed_kernel<float>;
        kt.begin(0, 0);
        if ((st = launch_k(e, f, dim3(Bp), dim3(128), 0, args, true)) != CVY_OK) return st;
        kt.end();
        launches++;
    }
    size_t pi = 0;
    for (int l = 0; l < m.n_layers; ++l) {
        kt.begin(1, l);
        if ((st = launch_gemm(e, bk, bk.plans[pi++])) != CVY_OK) return st;
        kt.end();
        kt.begin(2, l);
        if ((st = launch_attention(e, bk, l, &kt)) != CVY_OK) return st;
        launches += bk.P.attn_splits > 1 ? 3 : 2;  // QKV + attention (+ merge)
        for (int k = 0; k < 3; ++k) {
            kt.begin(4 + k, l);
            if ((st = launch_gemm(e, bk, bk.plans[pi++])) != CVY_OK) return st;
            kt.end();
            launches++;
        }
    }
    kt.begin(7, 0);
    if ((st = launch_gemm(e, bk, bk.plans[pi++])) != CVY_OK) return st;
    kt.end();
    launches++;
    bk.launches = launches;
    return CVY_OK;
}

// Wait for the oldest step in flight and return its events to the pool.
cvy_status retire_oldest(cvy_engine* e) {
    auto ev = e->inflight.front();
    cvy_status st = check_cuda(e, cudaEventSynchronize(ev.second), "event sync");
    if (st != CVY_OK) return st;
    cudaEventElapsedTime(&e->last_step_ms, ev.first, ev.second);
    e->inflight.pop_front();
    e->event_pool.push_back(ev);
    return CVY_OK;
}

}  // namespace

extern "C" {

cvy_status cvy_step(cvy_engine* e, cvy_step_info* last_completed) {
    if (!e) return fail(CVY_E_INVAL, "null engine");
    if (e->dead) return fail(CVY_E_CUDA, "engine is dead");
    cudaSetDevice(e->dev);
    // at most 2 steps in flight
    while (e->inflight.size() >= 2) {
        cvy_status st = retire_oldest(e);
        if (st != CVY_OK) return st;
    }
    // Ring back-pressure, checked BEFORE the queued host updates are taken (a non-fatal
    // E_FULL leaves them queued): the steps in flight plus this one may each publish up to
    // kMaxRecPerSlot records per slot in use.  While steps are in flight, retire the oldest
    // (its records are then in the ring and the bound shrinks); only with none in flight
    // wait for the poller.
    std::vector<Patch> patches;
    std::vector<Upload> uploads;
    std::vector<PrefillJob> prefills;
    std::vector<SynthJob> synths;
    int max_used = -1;
    {
        auto t0 = std::chrono::steady_clock::now();
        while (true) {
            int mu_now = -1;
            {
                std::lock_guard<std::mutex> lk(e->mu);
                for (int b = 0; b < (int)e->slots.size(); ++b)
                    if (e->slots[b].used) mu_now = b;
            }
            const uint64_t worst = (uint64_t)(e->inflight.size() + 1) * (uint64_t)(mu_now + 1) * kMaxRecPerSlot;
            const uint64_t tail = __atomic_load_n(e->h_ring_tail, __ATOMIC_ACQUIRE);
            const uint64_t head = __atomic_load_n(&e->ring_head, __ATOMIC_ACQUIRE);
            if (tail - head + worst <= e->c.ring_records) {
                std::lock_guard<std::mutex> lk(e->mu);
                for (int b = 0; b < (int)e->slots.size(); ++b)
                    if (e->slots[b].used) max_used = b;
                if (max_used > mu_now) continue;  // a submit raced in: re-check with its slot
                patches.swap(e->pending);
                uploads.swap(e->uploads);
                prefills.swap(e->prefill_pending);
                synths.swap(e->synth_pending);
                break;
            }
            if (!e->inflight.empty()) {
                cvy_status st = retire_oldest(e);
                if (st != CVY_OK) return st;
                continue;
            }
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30))
                return fail(CVY_E_FULL, "segment ring full: poll_segments is not draining it");
            std::this_thread::yield();
        }
    }
    // released slots still need their patch applied even if nothing is in use
    // batch bucket: multiple of 32 (epilogue chunk), 256 and 512 above 128/256
    int Bp = std::max(32, (max_used + 1 + 31) / 32 * 32);
    if (Bp > 256) Bp = 512;
    else if (Bp > 128) Bp = 256;
    if (Bp > (int)e->slots.size()) Bp = (int)e->slots.size();
    // from here on the queues are consumed: any failure is a CUDA error (sticky, engine dead)
    for (auto& u : uploads) {
        cvy_status st = check_cuda(e, cudaMemcpyAsync(u.dst, u.data.data(), u.data.size(), cudaMemcpyHostToDevice, e->stream),
                                   "upload");
        if (st != CVY_OK) return st;
    }
    for (const SynthJob& j : synths) {
        int32_t* d_pages = e->d_page_table + (size_t)j.slot * e->c.max_pages_per_slot;
        const int64_t n = (int64_t)e->m.n_layers * j.len * 2 * e->m.n_kv_heads * e->m.head_dim;
        const int blocks = (int)std::min<int64_t>(4096, (n + 255) / 256);
        if (e->bf16)
            synth_prefix_kernel<__nv_bfloat16><<<blocks, 256, 0, e->stream>>>(
                (__nv_bfloat16*)e->w.kv_pool, d_pages, (int)e->c.n_pages, e->m.n_layers, e->m.n_kv_heads,
                e->m.head_dim, (int)j.len, j.seed);
        else
            synth_prefix_kernel<float><<<blocks, 256, 0, e->stream>>>(
                (float*)e->w.kv_pool, d_pages, (int)e->c.n_pages, e->m.n_layers, e->m.n_kv_heads, e->m.head_dim,
                (int)j.len, j.seed);
        cvy_status cs = check_cuda(e, cudaGetLastError(), "synth prefix");
        if (cs != CVY_OK) return cs;
    }
    // patches in chunks of the device patch buffer (stream order keeps them sequential)
    for (size_t p0 = 0; p0 < patches.size(); p0 += (size_t)e->max_patches) {
        const int np = (int)std::min<size_t>((size_t)e->max_patches, patches.size() - p0);
        cvy_status st = check_cuda(e,
                                   cudaMemcpyAsync(e->d_patches, patches.data() + p0, np * sizeof(Patch),
                                                   cudaMemcpyHostToDevice, e->stream),
                                   "patch upload");
        if (st != CVY_OK) return st;
        apply_patches_kernel<<<1, 1, 0, e->stream>>>(e->d_slots, e->d_patches, np,
                                                     reinterpret_cast<SlotStatus*>(e->dm_status));
        st = check_cuda(e, cudaGetLastError(), "apply patches");
        if (st != CVY_OK) return st;
    }
    if (!prefills.empty()) {
        // page tables are uploaded above; the pass writes the jobs' KV before this step reads it
        cvy_status st = enqueue_prefill(e, prefills);
        if (st != CVY_OK) {
            e->dead = true;
            return st;
        }
    }
    Bucket* bk = nullptr;
    cvy_status st = build_bucket(e, Bp, &bk);
    if (st != CVY_OK) return st;
    std::pair<cudaEvent_t, cudaEvent_t> ev;
    if (!e->event_pool.empty()) {
        ev = e->event_pool.back();
        e->event_pool.pop_back();
    } else {
        cudaEventCreate(&ev.first);
        cudaEventCreate(&ev.second);
    }
    cudaEventRecord(ev.first, e->stream);
    if (e->c.flags & CVY_ENGINE_NO_GRAPH) {
        if ((st = enqueue_step_kernels(e, *bk)) != CVY_OK) {
            e->dead = true;
            return st;
        }
    } else {
        cudaGraphExec_t* target = e->timing ? &bk->graph_timed : e->spans_on ? &bk->graph_spans : &bk->graph;
        if (!*target) {
            cudaGraph_t g;
            e->capturing_timed = e->timing;
            e->capturing_spans = !e->timing && e->spans_on;
            if (e->capturing_spans) {  // kernel parameters are copied at capture: spans only in this variant
                bk->P.spans = e->d_spans;
            }
            st = check_cuda(e, cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal), "begin capture");
            if (st != CVY_OK) return st;
            cvy_status st2 = enqueue_step_kernels(e, *bk);
            cudaError_t ce = cudaStreamEndCapture(e->stream, &g);
            e->capturing_timed = false;
            e->capturing_spans = false;
            bk->P.spans = nullptr;
            if (st2 != CVY_OK) {
                e->dead = true;
                return st2;
            }
            if ((st = check_cuda(e, ce, "end capture")) != CVY_OK) return st;
            if ((st = check_cuda(e, cudaGraphInstantiate(target, g, 0), "graph instantiate")) != CVY_OK) return st;
            cudaGraphDestroy(g);
        }
        if ((st = check_cuda(e, cudaGraphLaunch(*target, e->stream), "graph launch")) != CVY_OK) return st;
        if (e->timing) e->last_timed = bk;
        else if (e->spans_on) e->last_spans = bk;
    }
    cudaEventRecord(ev.second, e->stream);
    if ((st = check_cuda(e, cudaGetLastError(), "step launch")) != CVY_OK) return st;
    e->inflight.push_back(ev);
    e->steps_launched++;
    e->last_bucket = Bp;
    e->last_launches = bk->launches;
    if (last_completed) {
        std::memset(last_completed, 0, sizeof(*last_completed));
        const uint64_t done = e->steps_launched - e->inflight.size();
        if (done > 0) {
            StepStats ss = e->h_stats[(done - 1) & 15];
            last_completed->step = ss.step;
            last_completed->n_active = ss.n_active;
            last_completed->n_generated = ss.n_generated;
            last_completed->n_segments = ss.n_segments;
            last_completed->n_finished = ss.n_finished;
            last_completed->step_ms = e->last_step_ms;
        }
    }
    return CVY_OK;
}

cvy_status cvy_sync(cvy_engine* e) {
    if (!e) return fail(CVY_E_INVAL, "null engine");
    if (e->dead) return fail(CVY_E_CUDA, "engine is dead");
    cudaSetDevice(e->dev);
    cvy_status st = check_cuda(e, cudaStreamSynchronize(e->stream), "stream sync");
    if (st != CVY_OK) return st;
    while (!e->inflight.empty()) {
        auto ev = e->inflight.front();
        cudaEventElapsedTime(&e->last_step_ms, ev.first, ev.second);
        e->inflight.pop_front();
        e->event_pool.push_back(ev);
    }
    return CVY_OK;
}

cvy_status cvy_poll_segments(cvy_engine* e, cvy_segment* out, uint32_t cap, uint32_t* n, uint8_t* bytes,
                             size_t bytes_cap, size_t* bytes_used) {
    if (!e || !out || !n) return fail(CVY_E_INVAL, "null argument");
    *n = 0;
    if (bytes_used) *bytes_used = 0;
    const uint64_t tail = __atomic_load_n(e->h_ring_tail, __ATOMIC_ACQUIRE);
    uint64_t head = e->ring_head;
    if (tail == head) return CVY_E_AGAIN;
    size_t used = 0;
    uint32_t k = 0;
    std::vector<std::pair<uint32_t, uint64_t>> finals;
    while (head < tail && k < cap) {
        const cvy_segment& r = e->h_ring[head & (e->c.ring_records - 1)];
        cvy_segment rec;
        std::memcpy(&rec, (const void*)&r, sizeof(rec));
        if (bytes) {
            if (used + rec.byte_len > bytes_cap) break;
            const uint32_t off = std::min(rec.byte_offset, e->c.round_bytes);
            const uint32_t len = std::min(rec.byte_len, e->c.round_bytes - off);
            std::memcpy(bytes + used, e->h_byte_log + (size_t)rec.slot * e->c.round_bytes + off, len);
            if (len < rec.byte_len) std::memset(bytes + used + len, 0, rec.byte_len - len);
            used += rec.byte_len;
        }
        out[k++] = rec;
        if (rec.flags & CVY_SEG_FINAL) finals.push_back({rec.slot, rec.req_id});
        ++head;
    }
    __atomic_store_n(&e->ring_head, head, __ATOMIC_RELEASE);
    *n = k;
    if (bytes_used) *bytes_used = used;
    if (!finals.empty()) {
        std::lock_guard<std::mutex> lk(e->mu);
        for (auto& f : finals) {
            SlotHost& sh = e->slots[f.first];
            if (sh.used && sh.req_id == f.second) {
                sh.final_seen = true;
                sh.final_pending = false;
                const cvy_segment* last = nullptr;
                for (uint32_t i = 0; i < k; ++i)
                    if (out[i].req_id == f.second && (out[i].flags & CVY_SEG_FINAL)) last = &out[i];
                sh.state = (last && (last->flags & CVY_SEG_CANCELLED)) ? 2 : 1;
            }
        }
    }
    return k ? CVY_OK : CVY_E_AGAIN;
}

cvy_status cvy_round_tokens(cvy_engine* e, uint64_t req_id, int32_t* out, uint32_t cap, uint32_t* n) {
    if (!e || !out || !n) return fail(CVY_E_INVAL, "null argument");
    int slot;
    {
        std::lock_guard<std::mutex> lk(e->mu);
        auto it = e->req_slot.find(req_id);
        if (it == e->req_slot.end()) return fail(CVY_E_NOTFOUND, "unknown request");
        slot = it->second;
    }
    const uint32_t gen_raw = ((volatile SlotStatus*)e->h_status)[slot].gen;
    const uint32_t gen = std::min(gen_raw, e->c.round_tokens);
    const uint32_t m = std::min(gen, cap);
    std::memcpy(out, e->h_tok_log + (size_t)slot * e->c.round_tokens, m * sizeof(int32_t));
    *n = m;
    return CVY_OK;
}

cvy_status cvy_debug_logits(cvy_engine* e, uint64_t req_id, float* out, uint32_t cap) {
    if (!e || !out) return fail(CVY_E_INVAL, "null argument");
    if (!e->d_dbg) return fail(CVY_E_STATE, "engine created without CVY_ENGINE_DEBUG_LOGITS");
    if (cap < (uint32_t)e->m.vocab) return fail(CVY_E_INVAL, "cap < vocab");
    int slot;
    {
        std::lock_guard<std::mutex> lk(e->mu);
        auto it = e->req_slot.find(req_id);
        if (it == e->req_slot.end()) return fail(CVY_E_NOTFOUND, "unknown request");
        slot = it->second;
    }
    cvy_status st = cvy_sync(e);
    if (st != CVY_OK) return st;
    return check_cuda(e,
                      cudaMemcpy(out, e->d_dbg + (size_t)slot * e->m.vocab, sizeof(float) * e->m.vocab,
                                 cudaMemcpyDeviceToHost),
                      "logits copy");
}

cvy_status cvy_perf(cvy_engine* e, cvy_perf_info* out) {
    if (!e || !out) return fail(CVY_E_INVAL, "null argument");
    out->last_step_ms = e->last_step_ms;
    out->launches_per_step = e->last_launches;
    out->slots_bucket = (uint32_t)e->last_bucket;
    return CVY_OK;
}

void* cvy_stream(cvy_engine* e) { return e ? (void*)e->stream : nullptr; }

cvy_status cvy_set_kernel_timing(cvy_engine* e, int32_t on) {
    if (!e) return fail(CVY_E_INVAL, "null engine");
    if (e->c.flags & CVY_ENGINE_NO_GRAPH) return fail(CVY_E_STATE, "kernel timing needs the graph path");
    e->timing = on != 0;
    return CVY_OK;
}

cvy_status cvy_set_kernel_spans(cvy_engine* e, int32_t on) {
    if (!e) return fail(CVY_E_INVAL, "null engine");
    if (e->c.flags & CVY_ENGINE_NO_GRAPH) return fail(CVY_E_STATE, "kernel spans need the graph path");
    e->spans_on = on != 0;
    return CVY_OK;
}

cvy_status cvy_kernel_spans(cvy_engine* e, cvy_kernel_span* out, uint32_t cap, uint32_t* n) {
    if (!e || !out || !n) return fail(CVY_E_INVAL, "null argument");
    *n = 0;
    if (!e->last_spans) return fail(CVY_E_STATE, "no span-recording step has run");
    cvy_status st = cvy_sync(e);
    if (st != CVY_OK) return st;
    std::vector<unsigned long long> h(2 * (size_t)kSpanSlots);
    if ((st = check_cuda(e, cudaMemcpy(h.data(), e->d_spans, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost),
                         "span copy")) != CVY_OK)
        return st;
    uint32_t k = 0;
    for (int i = 0; i < kSpanSlots && k < cap; ++i) {
        if (h[i] == ~0ull || h[kSpanSlots + i] == 0) continue;
        const int half = kSpanSlots / 2;
        out[k].chain = i / half;
        out[k].layer = (i % half) / 8;
        out[k].kind = (i % half) % 8;
        out[k].t0_ns = h[i];
        out[k].t1_ns = h[kSpanSlots + i];
        ++k;
    }
    *n = k;
    return CVY_OK;
}

cvy_status cvy_kernel_times(cvy_engine* e, cvy_kernel_time* out, uint32_t cap, uint32_t* n) {
    if (!e || !out || !n) return fail(CVY_E_INVAL, "null argument");
    *n = 0;
    if (!e->last_timed) return fail(CVY_E_STATE, "no timed step has run");
    cvy_status st = cvy_sync(e);
    if (st != CVY_OK) return st;
    Bucket& bk = *e->last_timed;
    const uint32_t m = std::min<uint32_t>(cap, (uint32_t)bk.kinfo.size());
    for (uint32_t i = 0; i < m; ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, bk.kev[2 * i], bk.kev[2 * i + 1]);
        out[i].kind = bk.kinfo[i].first;
        out[i].layer = bk.kinfo[i].second;
        out[i].ms = ms;
    }
    *n = m;
    return CVY_OK;
}

cvy_status cvy_debug_buffer(cvy_engine* e, int32_t which, void* dst, size_t cap, size_t* bytes) {
    if (!e || !bytes) return fail(CVY_E_INVAL, "null argument");
    const size_t B = e->slots.size(), es = dtype_size(e->m.dtype);
    const void* src = nullptr;
    size_t n = 0;
    switch (which) {
        case 0: src = e->d_x; n = B * e->m.d_model * 4; break;
        case 1: src = e->d_act; n = (e->bf16 ? 2 : 1) * B * e->act_ld * es; break;
        case 2: src = e->d_q; n = B * e->m.n_heads * e->m.head_dim * 4; break;
        case 3: src = e->d_o; n = (e->bf16 ? 2 : 1) * B * e->act_ld * es; break;
        case 4: src = e->d_h; n = (e->bf16 ? 2 : 1) * B * e->act_ld * es; break;
        case 5: src = e->d_ssq; n = (size_t)(e->m.d_model / 128) * B * 4; break;
        case 6: src = e->d_page_table; n = B * e->c.max_pages_per_slot * 4; break;
        case 7:
            if (!e->d_prow) return fail(CVY_E_STATE, "no chunked prefill");
            src = e->d_prow;
            n = (size_t)3 * kPrefillRows * 4;
            break;
        case 8: case 9: case 12 + 8: case 13 + 8: case 14 + 8:  // last prefill pass: x, q, o, h, act
            if (!e->d_px) return fail(CVY_E_STATE, "no chunked prefill");
            if (which == 8) { src = e->d_px; n = sizeof(float) * kPrefillRows * e->m.d_model; }
            else if (which == 9) { src = e->d_pq; n = sizeof(float) * kPrefillRows * e->m.n_heads * e->m.head_dim; }
            else {
                src = which == 20 ? e->d_po : which == 21 ? e->d_ph : e->d_pact;
                n = 2 * es * kPrefillRows * e->act_ld;
            }
            break;
        case 10: case 11: case 12: case 13:
            if (!e->d_trace) return fail(CVY_E_STATE, "set CVY_GEMM_TRACE_LAYER before engine create");
            src = e->d_trace + (size_t)(which - 10) * kTraceStride * e->num_sms;
            n = sizeof(unsigned long long) * kTraceStride * e->num_sms;
            break;
        default: return fail(CVY_E_INVAL, "unknown buffer");
    }
    *bytes = n;
    if (!dst) return CVY_OK;
    if (cap < n) return fail(CVY_E_INVAL, "buffer too small");
    cvy_status st = cvy_sync(e);
    if (st != CVY_OK) return st;
    return check_cuda(e, cudaMemcpy(dst, src, n, cudaMemcpyDeviceToHost), "debug copy");
}

}  // extern "C"

// ============================================================================ multi-GPU stats
// One decode replica per GPU (requests shard across replicas); the
// only GPU<->GPU traffic is this all-gather of a 64-byte per-engine stats record over
// NVLink / NVSwitch, on a side stream so it never sits on the decode critical path.
#include <dlfcn.h>
#include <nccl.h>

namespace {
// NCCL is resolved lazily (dlopen at first use) so that loading libconveyor never pins an
// NCCL build ahead of the one PyTorch ships (same soname, different versions).
struct NcclApi {
    decltype(&ncclCommInitAll) CommInitAll = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclAllGather) AllGather = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    bool ok = false;
};
NcclApi& nccl() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW);
        if (h) {
            api.CommInitAll = (decltype(api.CommInitAll))dlsym(h, "ncclCommInitAll");
            api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
            api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
            api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
            api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
            api.ok = api.CommInitAll && api.CommDestroy && api.AllGather && api.GroupStart && api.GroupEnd;
        }
    }
    return api;
}
struct StatsComm {
    std::vector<int> devs;
    std::vector<ncclComm_t> comms;
    std::vector<cudaStream_t> streams;
    std::vector<uint64_t*> bufs;  // [n][8] recv + [8] send per device
};
std::mutex g_stats_mu;
StatsComm g_stats;
}  // namespace

extern "C" cvy_status cvy_stats_allgather(cvy_engine* const* engines, int32_t n, uint64_t* out) {
    if (!engines || n < 1 || !out) return fail(CVY_E_INVAL, "bad arguments");
    std::lock_guard<std::mutex> lk(g_stats_mu);
    NcclApi& N = nccl();
    if (!N.ok) return fail(CVY_E_NCCL, "libnccl.so.2 not found");
    std::vector<int> devs(n);
    for (int i = 0; i < n; ++i) {
        if (!engines[i]) return fail(CVY_E_INVAL, "null engine");
        devs[i] = engines[i]->dev;
    }
    if (g_stats.devs != devs) {
        for (size_t i = 0; i < g_stats.comms.size(); ++i) {
            N.CommDestroy(g_stats.comms[i]);
            cudaSetDevice(g_stats.devs[i]);
            cudaStreamDestroy(g_stats.streams[i]);
            cudaFree(g_stats.bufs[i]);
        }
        g_stats = StatsComm();
        g_stats.devs = devs;
        g_stats.comms.resize(n);
        if (N.CommInitAll(g_stats.comms.data(), n, devs.data()) != ncclSuccess) {
            g_stats = StatsComm();
            return fail(CVY_E_NCCL, "ncclCommInitAll failed");
        }
        for (int i = 0; i < n; ++i) {
            cudaSetDevice(devs[i]);
            cudaStream_t s;
            cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
            g_stats.streams.push_back(s);
            uint64_t* b = nullptr;
            CUDA_TRY(cudaMalloc(&b, sizeof(uint64_t) * 8 * (n + 1)));
            g_stats.bufs.push_back(b);
        }
    }
    std::vector<std::vector<uint64_t>> send(n, std::vector<uint64_t>(8, 0));
    for (int i = 0; i < n; ++i) {
        cvy_engine* e = engines[i];
        const uint64_t done = e->steps_launched - e->inflight.size();
        StepStats ss{};
        if (done > 0) ss = e->h_stats[(done - 1) & 15];
        send[i][0] = ss.step;
        send[i][1] = ss.n_active;
        send[i][2] = ss.n_generated;
        send[i][3] = ss.n_segments;
        send[i][4] = ss.n_finished;
        uint32_t ms_bits;
        std::memcpy(&ms_bits, &e->last_step_ms, 4);
        send[i][5] = ms_bits;
        send[i][6] = (uint64_t)e->dev;
        send[i][7] = e->steps_launched;
        cudaSetDevice(devs[i]);
        CUDA_TRY(cudaMemcpyAsync(g_stats.bufs[i] + 8 * n, send[i].data(), 64, cudaMemcpyHostToDevice, g_stats.streams[i]));
    }
    if (N.GroupStart() != ncclSuccess) return fail(CVY_E_NCCL, "ncclGroupStart");
    for (int i = 0; i < n; ++i) {
        if (N.AllGather(g_stats.bufs[i] + 8 * n, g_stats.bufs[i], 8, ncclUint64, g_stats.comms[i], g_stats.streams[i]) !=
            ncclSuccess) {
            N.GroupEnd();
            return fail(CVY_E_NCCL, "ncclAllGather");
        }
    }
    if (N.GroupEnd() != ncclSuccess) return fail(CVY_E_NCCL, "ncclGroupEnd");
    cudaSetDevice(devs[0]);
    CUDA_TRY(cudaMemcpyAsync(out, g_stats.bufs[0], sizeof(uint64_t) * 8 * n, cudaMemcpyDeviceToHost, g_stats.streams[0]));
    for (int i = 0; i < n; ++i) {
        cudaSetDevice(devs[i]);
        CUDA_TRY(cudaStreamSynchronize(g_stats.streams[i]));
    }
    return CVY_OK;
}

// ============================================================================ test hook
extern "C" cvy_status cvy_debug_gemm(const void* W, const void* X, float* Y, int32_t N, int32_t K, int32_t B,
                                     int32_t iters, int32_t device, float* ms) {
    if (!W || !X || !Y || N < 1 || K < 64 || K % 64 || B < 1 || B > 512 || iters < 1)
        return fail(CVY_E_INVAL, "bad GEMM arguments");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(CVY_E_CUDA, "no CUDA device");
    CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return fail(CVY_E_CUDA, "sm_100a only");
    set_gemm_smem_attrs();
    const int Bp0 = (B + 31) / 32 * 32;
    const int Bp = Bp0 > 256 ? 512 : (Bp0 > 128 ? 256 : Bp0);
    StepParams P;
    std::memset(&P, 0, sizeof(P));
    P.Bp = Bp;
    P.Bmax = Bp;
    P.act_ld = K;
    GemmTC g;
    std::memset(&g, 0, sizeof(g));
    int grid = 0;
    size_t smem = 0;
    std::string why;
    if (!gemm_config(g, N, K, Bp, prop.multiProcessorCount, &grid, &smem, &why, true, false, 0, 1, gemm_pair_ok(EPI_STORE)))
        return fail(CVY_E_INVAL, why);
    g.w_row0 = 0;
    g.x_plane_rows = Bp;
    g.epi.kind = EPI_STORE;
    g.epi.N = N;
    if (const char* dbg = getenv("CVY_GEMM_DEBUG")) g.dbg = atoi(dbg);
    float* Ytmp = nullptr;
    CUDA_TRY(cudaMalloc(&Ytmp, sizeof(float) * (size_t)Bp * N));
    g.epi.store_out = Ytmp;
    const size_t tile_rows = (size_t)(g.pair ? 256 : 128 * g.nsub);
    CUDA_TRY(cudaMalloc(&g.part, sizeof(float) * (size_t)g.tiles * tile_rows * Bp));
    CUDA_TRY(cudaMemset(g.part, 0, sizeof(float) * (size_t)g.tiles * tile_rows * Bp));
    CUDA_TRY(cudaMalloc(&g.tile_cnt, sizeof(int32_t) * (2 * g.tiles * g.nbt + 1)));
    CUDA_TRY(cudaMemset(g.tile_cnt, 0, sizeof(int32_t) * (2 * g.tiles * g.nbt + 1)));
    // X as the (hi, lo) pair the engine uses: hi = X (exact bf16), lo = 0, padded to Bp rows
    void* Xp = nullptr;
    CUDA_TRY(cudaMalloc(&Xp, (size_t)2 * Bp * K * 2));
    CUDA_TRY(cudaMemset(Xp, 0, (size_t)2 * Bp * K * 2));
    CUDA_TRY(cudaMemcpy(Xp, X, (size_t)B * K * 2, cudaMemcpyDeviceToDevice));
    // test hook: X holds 2*B rows, [hi][lo] (the kernel computes W (hi + lo))
    if (getenv("CVY_DEBUG_GEMM_LO") && atoi(getenv("CVY_DEBUG_GEMM_LO")) != 0)
        CUDA_TRY(cudaMemcpy(static_cast<uint8_t*>(Xp) + (size_t)Bp * K * 2, static_cast<const uint8_t*>(X) + (size_t)B * K * 2,
                            (size_t)B * K * 2, cudaMemcpyDeviceToDevice));
    CUtensorMap tmW, tmX;
    const uint32_t xrows = g.merge ? (uint32_t)g.bq : (uint32_t)g.mma_n;
    if (!make_tmap(&tmW, W, (uint64_t)N, (uint64_t)K, (uint64_t)K, (uint32_t)(128 * g.nsub), (uint32_t)g.bk) ||
        !make_tmap(&tmX, Xp, (uint64_t)(2 * Bp), (uint64_t)K, (uint64_t)K, xrows, (uint32_t)g.bk))
        return fail(CVY_E_CUDA, "tensor map encode failed");
    const void* kfn = gemm_tc_kernel_ptr<__nv_bfloat16>(g.nsub, g.merge != 0, g.bk, EPI_STORE, g.pair != 0);
    void* args[] = {&tmW, &tmX, &P, &g, &tmW};
    cudaLaunchConfig_t lc;
    std::memset(&lc, 0, sizeof(lc));
    lc.gridDim = dim3(grid, g.nbt);
    lc.blockDim = dim3(kGemmThreads);
    lc.dynamicSmemBytes = smem;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeClusterDimension;
    la[0].val.clusterDim.x = (unsigned)(g.pair ? 2 : (g.split > 1 ? g.split : 1));
    la[0].val.clusterDim.y = 1;
    la[0].val.clusterDim.z = 1;
    lc.attrs = la;
    lc.numAttrs = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    CUDA_TRY(cudaLaunchKernelExC(&lc, kfn, args));  // warm-up
    CUDA_TRY(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    for (int i = 0; i < iters; ++i) cudaLaunchKernelExC(&lc, kfn, args);
    cudaEventRecord(e1);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventSynchronize(e1));
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    if (ms) *ms = t / iters;
    if (getenv("CVY_GEMM_TRACE")) {
        // one traced launch: per-CTA globaltimer stamps relative to the earliest CTA start
        unsigned long long* tr = nullptr;
        CUDA_TRY(cudaMalloc(&tr, sizeof(unsigned long long) * kTraceStride * grid));
        CUDA_TRY(cudaMemset(tr, 0, sizeof(unsigned long long) * kTraceStride * grid));
        g.trace = tr;
        void* targs[] = {&tmW, &tmX, &P, &g, &tmW};
        CUDA_TRY(cudaLaunchKernelExC(&lc, kfn, targs));
        CUDA_TRY(cudaDeviceSynchronize());
        std::vector<unsigned long long> h(kTraceStride * (size_t)grid);
        CUDA_TRY(cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost));
        cudaFree(tr);
        g.trace = nullptr;
        unsigned long long t0 = ~0ull;
        for (int c = 0; c < grid; ++c) t0 = std::min(t0, h[kTraceStride * c]);
        double mx[6] = {0}, mn[6], sum[6] = {0};
        for (int k = 0; k < 6; ++k) mn[k] = 1e30;
        for (int c = 0; c < grid; ++c)
            for (int k = 0; k < 6; ++k) {
                double v = h[kTraceStride * c + k] ? (h[kTraceStride * c + k] - t0) * 1e-3 : -1;
                mx[k] = std::max(mx[k], v);
                mn[k] = std::min(mn[k], v);
                sum[k] += v;
            }
        const char* names[6] = {"start", "producer done", "first seg MMA done", "last seg MMA done", "epilogue done",
                                "exit"};
        for (int k = 0; k < 6; ++k)
            fprintf(stderr, "trace %-20s min %8.2f avg %8.2f max %8.2f us\n", names[k], mn[k], sum[k] / grid, mx[k]);
    }
    CUDA_TRY(cudaMemcpy2D(Y, sizeof(float) * N, Ytmp, sizeof(float) * N, sizeof(float) * N, B, cudaMemcpyDeviceToDevice));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(Ytmp);
    cudaFree(g.part);
    cudaFree(g.tile_cnt);
    cudaFree(Xp);
    return CVY_OK;
}
