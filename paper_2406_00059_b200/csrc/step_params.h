// step_params.h -- plain structs shared by the engine's host code and its kernels.
#pragma once
#include <stdint.h>

#include "../../include/conveyor.h"

namespace cvy {

constexpr int kPageTokens = 16;
constexpr int kMaxTokenBytes = 16;
constexpr int kMaxRecPerSlot = kMaxTokenBytes + 1;  // cuts of one token + FINAL
constexpr int kMaxTools = 64;
constexpr int kMaxSlots = 512;

// Per-slot device state (one continuous-batching slot = one in-flight request).
struct SlotDev {
    uint64_t req_id;
    int32_t active;     // 1: in the batch (feeding or generating); 0: idle / parked
    int32_t tool;       // registered tool id, -1: scan off
    int32_t pos;        // position of cur_tok in the sequence (= KV length before this step)
    int32_t cur_tok;    // input token of the next step
    int32_t in_idx;     // forced inputs still to feed: in_buf[slot][in_idx .. in_len)
    int32_t in_len;
    int32_t gen;        // generated tokens in the current round
    int32_t max_new;
    int32_t force_len;  // teacher forcing of the round's generated tokens
    uint32_t round, seq;
    uint32_t stream_len, seg_start;  // round byte stream length / current segment start
    uint64_t win;       // last <= 8 bytes since seg_start, newest in the low byte
    int32_t depth, in_str, esc;      // JSON automaton
    int32_t cancel;
    int32_t max_pos;    // reserved KV positions (exclusive bound on pos)
    int32_t region;     // tool set: tool whose region is open (-1: outside)
    uint64_t tool_set;  // region-tool set (bit i = tool i; 0: the single tool `tool`)
    int32_t set_max_seg;  // tool set: cut of a line outside a region (smallest max_seg)
    int32_t pad_;
};

struct ToolDev {
    int32_t kind;       // cvy_parser_kind
    int32_t n_delims;
    int32_t max_seg;
    int32_t pad_;
    uint64_t dpack[8];  // delimiter bytes packed newest-low (last byte in bits 0..7)
    uint64_t dmask[8];
    int32_t dlen[8];
};

// Host-visible per-slot status (pinned, mapped).
struct SlotStatus {
    uint32_t round, gen, state, last_step;  // state: 0 running, 1 parked, 2 cancelled, 3 idle
};

// Host-visible per-step statistics (pinned, mapped ring of 16).
struct StepStats {
    uint64_t step;
    uint32_t n_active, n_generated, n_segments, n_finished;
};

enum PatchKind : int32_t { PATCH_SUBMIT = 0, PATCH_INJECT = 1, PATCH_CANCEL = 2, PATCH_RELEASE = 3 };

struct Patch {
    int32_t kind, slot;
    uint64_t req_id;
    int32_t tool, pos, cur_tok, in_len, in_idx, max_new, force_len, max_pos;
    uint32_t round, seq;
    int32_t set_pos;   // INJECT: 1 = also set pos / cur_tok (the observation was prefilled)
    int32_t set_max_seg;  // SUBMIT: tool set's outside-line cut
    uint64_t tool_set;    // SUBMIT: region-tool set (0: single tool)
};

enum EpiKind : int32_t { EPI_QKV = 0, EPI_RESID = 1, EPI_SWIGLU = 2, EPI_LMHEAD = 3, EPI_STORE = 4 };

// Everything a step's kernels need (passed by value as a __grid_constant__ parameter).
struct StepParams {
    // model
    int32_t L, d, H, Hkv, hd, dff, V, eos;
    float eps;
    int32_t Bp;        // padded batch of this launch (multiple of 16)
    int32_t Bmax;      // leading dimension of per-slot buffers
    int32_t n_pages, max_pages;
    int32_t act_ld;    // row stride (elements) of act / o / h buffers = max(d, H*hd, dff)
    int64_t act_plane; // elements between the hi and lo planes of act / o / h (bf16 model)
    // state
    SlotDev* slots;
    const int32_t* page_table;  // [Bmax][max_pages]
    const int32_t* in_buf;      // [Bmax][input_cap]
    int32_t input_cap;
    const int32_t* force_buf;   // [Bmax][forced_cap]
    int32_t forced_cap;
    const float2* rope;         // [max_rope_pos][hd/2] (cos, sin)
    int32_t max_rope_pos;
    // weights (model dtype) and norms (fp32)
    const void* embed;
    const float* attn_norm;
    const float* mlp_norm;
    const float* final_norm;
    void* kv_pool;
    // activations
    float* x;                   // [Bmax][d] fp32 residual
    void* act;                  // [planes][Bmax][act_ld] model dtype: GEMM input after RMSNorm
    float* q;                   // [Bmax][H*hd] fp32 (RoPE applied)
    void* o;                    // [planes][Bmax][act_ld] attention output
    void* h;                    // [planes][Bmax][act_ld] SwiGLU output
    float* ssq;                 // [d/128][Bmax] sum of squares per 128-wide block of x
    unsigned long long* am_keys;  // [Bmax] argmax keys
    float* dbg_logits;          // [Bmax][V] or null
    int32_t* lm_done;           // tiles-done counter of the LM head
    // attention split-KV workspace
    float* attn_part;           // [Bmax][Hkv][nsplit][G*(hd+2)]
    int32_t attn_splits;
    int32_t attn_early;         // attention_tc: issue old-page TMA loads before the PDL wait (1)
    int32_t kv_tma3d;           // attention_tc, hd 128: the KV tensor map is 3D, one box per 4 KB block
    // scan / publish
    const uint8_t* vtab;        // [V][16]
    const uint8_t* vlen;        // [V]
    const ToolDev* tools;
    void* ring;                 // cvy_segment[ring_mask+1], pinned mapped
    uint32_t ring_mask;
    unsigned long long* ring_tail_dev;
    unsigned long long* ring_tail_host;  // mapped
    uint8_t* byte_log;          // [Bmax][round_bytes], mapped
    uint32_t round_bytes;
    int32_t* tok_log;           // [Bmax][round_tokens], mapped
    uint32_t round_tokens;
    SlotStatus* status;         // [Bmax], mapped
    StepStats* stats;           // [16], mapped
    unsigned long long* step_ctr;  // device
    int32_t scan_off;
    // Chunked prefill (NEXT-1): a prefill pass maps launch row r to (slot row_slot[r], position
    // row_pos[r], input token row_tok[r]); row_pos < 0 marks a padding row.  Null in decode
    // steps, where row r is slot r at its current position.
    const int32_t* row_slot;
    const int32_t* row_pos;
    const int32_t* row_tok;
    // In-graph kernel spans (measurement variant of the step graph; null otherwise):
    // spans[i] = earliest %globaltimer at which a CTA of launch i passed its grid-dependency
    // wait (atomicMin), spans[kSpanSlots + i] = latest CTA exit (atomicMax);
    // i = span_base + layer * 8 + kind (kind: 0 embed, 1 QKV, 2 attention, 4 O, 5 gate/up,
    // 6 down, 7 LM head).
    unsigned long long* spans;
    int32_t span_base;
};
constexpr int kSpanSlots = 2 * 8 * 65;  // two chains x 8 kinds x (<= 64 layers + the LM head row)

// keys attended by launch row r (its position + 1), 0 for idle slots / padding rows
__host__ __device__ inline int row_nkeys(const StepParams& P, int r) {
    if (P.row_slot) return P.row_pos[r] >= 0 ? P.row_pos[r] + 1 : 0;
    const SlotDev& s = P.slots[r];
    return s.active ? (s.pos < s.max_pos - 1 ? s.pos : s.max_pos - 1) + 1 : 0;
}
__host__ __device__ inline int row_slot_of(const StepParams& P, int r) { return P.row_slot ? P.row_slot[r] : r; }

struct EpiArgs {
    int32_t kind;
    int32_t layer;
    int32_t N;                  // valid output rows
    const float* norm_w;        // RESID: the next RMSNorm's weights
    float* store_out;           // STORE (test hook): out[b][n] fp32, row stride N
    int32_t span_kind;          // kind of this launch in StepParams::spans (-1: none)
};

}  // namespace cvy
