/*
 * conveyor.h -- C ABI of libconveyor, the B200-native decode hot path under Conveyor
 * (Xu, Kong, Chen, Zhuo: "Conveyor: Efficient Tool-aware LLM Serving with Tool Partial
 * Execution", arXiv 2406.00059).  One engine = one GPU = one continuous-batching decode
 * replica with a fused, device-side tool-trigger scan.
 *
 * The five calls of the paper's problem statement:
 *   cvy_register_tool      "select a parser ... register both the parser and the plugin"
 *                          (sec 3.2; workflow steps (a),(b))
 *   cvy_submit_request     a user request enters the scheduler (step (1))
 *   cvy_step               one decoding iteration for every in-flight request (step (2);
 *                          continuous batching); the trigger scan runs in
 *                          the sampling epilogue of the same launch (steps (3)-(5))
 *   cvy_poll_segments      the host "periodically polls" the completed partial-execution
 *                          pieces while decoding continues (step (8))
 *   cvy_inject_observation "concatenates the original prompt, plans, and observations ...
 *                          feeds them back" (step (g)) -- appended to the
 *                          resident KV cache of the request as forced inputs.
 *
 * Conventions
 *   - Every call returns cvy_status (0 OK, < 0 error).  Nothing throws or aborts across
 *     the ABI.  cvy_last_error() returns a thread-local message for the last failure.
 *   - CVY_E_CUDA is sticky: after a CUDA error the engine is dead; only destroy is valid.
 *   - Device pointers in cvy_weights are BORROWED (caller-owned, e.g. torch tensors) and
 *     must outlive the engine.  Every host array passed in is copied before the call
 *     returns.  Output buffers are caller-owned.
 *   - Threading: submit / inject / cancel / release may be called from any thread (queued
 *     under a mutex, applied at the next step boundary).  cvy_step is called from one
 *     driver thread; cvy_poll_segments from exactly one consumer thread.
 *   - Build: sm_100a only.  No CPU fallback: without a B200 every device call fails with
 *     CVY_E_CUDA.
 */
#ifndef CONVEYOR_H
#define CONVEYOR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CVY_ABI_VERSION 1

typedef enum {
    CVY_OK = 0,
    CVY_E_INVAL = -1,    /* bad argument                                              */
    CVY_E_NOMEM = -2,    /* host or device allocation failed                          */
    CVY_E_FULL = -3,     /* no free slot / pages / input capacity: retry later         */
    CVY_E_AGAIN = -4,    /* nothing to poll                                            */
    CVY_E_NOTFOUND = -5, /* unknown request id or tool                                 */
    CVY_E_STATE = -6,    /* call not valid in the current lifecycle state              */
    CVY_E_DUP = -7,      /* duplicate tool name                                        */
    CVY_E_CUDA = -8,     /* CUDA error or no usable sm_100 device (sticky)             */
    CVY_E_NCCL = -9      /* NCCL error                                                 */
} cvy_status;

typedef enum { CVY_DTYPE_BF16 = 0, CVY_DTYPE_FP32 = 1 } cvy_dtype;

/* Parser kinds ("Conveyor offers a set of parsers"; R5-R11).
 * LITERAL: a segment ends at the shortest prefix ending in a registered delimiter
 *          (e.g. "\n" or ";" for a code interpreter).
 * JSON_MEMBER: a ',' at depth 1 or the bracket closing depth 1 ends a segment
 *          ("field complete", validator).
 * JSON_OBJECT: the bracket returning depth to 0 ends a segment ("a complete stage of the
 *          plan").
 * FENCE:   region grammar (R21): the line "```" TAG "\n" opens the tool region and
 *          the line "```\n" closes it ("the markdown code block syntax ```python and ``` as the
 *          indicators for the start and end of the tool"); every line inside is
 *          one segment ("a complete line of Python code").  Lines outside a
 *          region are not tool input and produce no record; the open / close marker lines are
 *          records flagged CVY_SEG_OPEN / CVY_SEG_CLOSE.  TAG = the single delimiter (1..8
 *          bytes, no '\n').  A line reaching max_segment_bytes is cut (OVERFLOW inside a
 *          region, silently outside); its continuation is never a marker.
 * CALL:    (R22) a line starting with "@call " TAG " " opens a call region the
 *          moment the space after the tool name arrives ("identifies the function name of
 *          the tool") -> CVY_SEG_OPEN record; inside, the JSON
 *          argument object is cut like JSON_MEMBER (one segment per completed field) and the
 *          bracket returning depth to 0 is a CVY_SEG_CLOSE record; text outside is not input.
 *          TAG = the single delimiter (1..8 bytes, no '\n').
 * PLAN:    (R23) each line matching  #E<digits> = <Name>[<args>]  is one segment ("a
 *          complete stage of the plan"); other lines produce no
 *          record.  No delimiters. */
typedef enum {
    CVY_PARSER_LITERAL = 0,
    CVY_PARSER_JSON_MEMBER = 1,
    CVY_PARSER_JSON_OBJECT = 2,
    CVY_PARSER_FENCE = 3,
    CVY_PARSER_CALL = 4,
    CVY_PARSER_PLAN = 5
} cvy_parser_kind;

/* Host dispatch policy only; the device path is identical in both modes. */
typedef enum { CVY_MODE_PARTIAL = 0, CVY_MODE_SEQUENTIAL = 1 } cvy_exec_mode;

enum { CVY_SEG_FINAL = 1, CVY_SEG_OVERFLOW = 2, CVY_SEG_CANCELLED = 4, CVY_SEG_OPEN = 8, CVY_SEG_CLOSE = 16 };
#define CVY_DELIM_NONE 0xFFFFu
#define CVY_NO_TOKEN 0xFFFFFFFFu

/* Model shape.  Mistral/Llama family: RMSNorm, RoPE (rotate-half), GQA, SwiGLU, no bias,
 * untied LM head (R1-R3).  Requirements: head_dim in {32,64,128};
 * d_model, n_heads*head_dim, d_ff multiples of 128; n_heads % n_kv_heads == 0. */
typedef struct {
    int32_t n_layers, d_model, n_heads, n_kv_heads, head_dim, d_ff, vocab;
    float rms_eps;
    double rope_base;
    int32_t eos_id; /* -1: no EOS (rounds end at max_new_tokens) */
    cvy_dtype dtype; /* weights, activations at GEMM inputs, and KV cache */
} cvy_model_config;

enum {
    CVY_ENGINE_NO_GRAPH = 1,     /* launch kernels directly instead of a CUDA graph          */
    CVY_ENGINE_DEBUG_LOGITS = 2, /* keep the last step's fp32 logits for cvy_debug_logits   */
    CVY_ENGINE_SCAN_OFF = 4,     /* trigger scan disabled for every slot (overhead A/B)      */
    CVY_ENGINE_NO_PDL = 8,       /* no programmatic dependent launch between kernels        */
    /* 16: reserved (was the persistent all-layers kernel's opt-out; that kernel is gone) */
    CVY_ENGINE_CHUNKED_PREFILL = 32, /* prompt and observation tokens (all but the last) run
                                     as one batched prefill pass at the next step boundary
                                     instead of one token per decode step (NEXT-1)           */
    CVY_ENGINE_TILED_WEIGHTS = 64 /* wqkv / wo / wgu / wd are tile-major (packed by
                                     cvy_pack_weights_tiled); bf16 only                      */
};

typedef struct {
    uint32_t max_slots;          /* max in-flight requests, 1..512                          */
    uint32_t n_pages;            /* pages in the KV pool (16 tokens each)                  */
    uint32_t max_pages_per_slot; /* page-table width: max context = 16 * this              */
    uint32_t ring_records;       /* segment ring capacity (power of two, >= 32*max_slots)  */
    uint32_t round_bytes;        /* per-slot byte-log capacity per round                   */
    uint32_t round_tokens;       /* per-slot generated-token log capacity per round        */
    uint32_t input_cap;          /* per-slot forced-input (prompt/observation) capacity    */
    uint32_t forced_cap;         /* per-slot teacher-forcing capacity per round            */
    int32_t device;              /* CUDA device ordinal                                    */
    uint32_t flags;              /* CVY_ENGINE_*                                           */
} cvy_engine_config;

/* Weights and KV pool: BORROWED device pointers, row-major, dtype = model dtype except
 * the norm weights (fp32).  Layouts:
 *   embed      [V][d]
 *   lm_head    [V][d]
 *   final_norm [d] fp32;  attn_norm, mlp_norm [L][d] fp32
 *   wqkv       [L][(H + 2*Hkv)*hd][d]   rows: q heads, k heads, v heads
 *   wo         [L][d][H*hd]
 *   wgu        [L][2*d_ff][d]  gate/up interleaved in 64-row blocks: rows 128j..128j+63
 *                              are gate rows 64j.., rows 128j+64..128j+127 up rows 64j..
 *   wd         [L][d][d_ff]
 *   kv_pool    [L][n_pages][Hkv][2 (K,V)][16][hd]  (written by the engine)            */
typedef struct {
    const void* embed;
    const void* lm_head;
    const float* final_norm;
    const float* attn_norm;
    const float* mlp_norm;
    const void* wqkv;
    const void* wo;
    const void* wgu;
    const void* wd;
    void* kv_pool;
} cvy_weights;

typedef struct cvy_engine cvy_engine;

/* Byte sizes of every weight buffer and of the KV pool for a config (host-only helper). */
typedef struct {
    size_t embed, lm_head, final_norm, attn_norm, mlp_norm, wqkv, wo, wgu, wd, kv_pool;
} cvy_weight_sizes;
cvy_status cvy_weight_sizes_for(const cvy_model_config* m, uint32_t n_pages, cvy_weight_sizes* out);

/* Fill every weight buffer with the counter-hash random init of DESIGN.md "Input recipe"
 * (uniform, std 0.02; norms 1.0) on the given device.  Synchronous.  Zeroes nothing else. */
cvy_status cvy_init_synthetic_weights(const cvy_model_config* m, const cvy_weights* w,
                                      uint64_t seed, int32_t device);

/* Repack wqkv, wo, wgu and wd -- and lm_head when vocab % 128 == 0 -- IN PLACE from the
 * row-major layouts above into tile-major order, for an engine created with
 * CVY_ENGINE_TILED_WEIGHTS (which reads lm_head tile-major under the same vocab rule).  Each [L*R][K] matrix (R rows
 * per layer, K columns) becomes [L*R/128][K/64][128][64]: element (r, k) moves to
 *   ((r / 128) * (K / 64) + k / 64) * 8192 + (r % 128) * 64 + k % 64,
 * so every 128-row x 64-column weight tile a projection GEMM stage loads is 16 contiguous KB
 * (one DRAM-friendly TMA box instead of 128 B from each of 128 rows; DESIGN.md §7.2 "Weight
 * layout").  The weights are the same values (a permutation of their bytes); the GEMMs
 * (the projections of the decode step) compute the same products.
 * bf16 only; every R % 128 == 0 and K % 64 == 0, else CVY_E_INVAL and nothing is touched.
 * Uses a device scratch buffer of one layer's largest matrix.  Synchronous.  Not idempotent:
 * call once per weight set.  On CVY_E_CUDA the matrices may be partly packed: regenerate them
 * (cvy_init_synthetic_weights) before use. */
cvy_status cvy_pack_weights_tiled(const cvy_model_config* m, const cvy_weights* w, int32_t device);

/* Create / destroy.  vocab_bytes [V][16] and vocab_lens [V] give the byte string of every
 * token id (<= 16 bytes; specials have length 0) and are copied. */
cvy_status cvy_engine_create(const cvy_model_config* m, const cvy_engine_config* e,
                             const cvy_weights* w, const uint8_t* vocab_bytes,
                             const uint8_t* vocab_lens, cvy_engine** out);
void cvy_engine_destroy(cvy_engine* e);
const char* cvy_last_error(void);
int32_t cvy_abi_version(void);

/* Tool registration (before the first submit).  LITERAL: 1..8 distinct delimiters of
 * 1..8 bytes each.  JSON kinds take no delimiters.  FENCE: exactly one delimiter = the
 * fence tag (1..8 bytes, no '\n'); max_segment_bytes must be >= tag length + 4 (the open
 * marker line must fit one segment).  max_segment_bytes 0 => 4096.
 * Errors: E_DUP name clash, E_INVAL bad delimiters, E_STATE after the first submit,
 * E_FULL more than 64 tools. */
typedef struct {
    const char* name;
    cvy_parser_kind parser;
    uint32_t n_delims;
    const uint8_t* const* delims;
    const uint32_t* delim_lens;
    uint32_t max_segment_bytes;
} cvy_tool_desc;
cvy_status cvy_register_tool(cvy_engine* e, const cvy_tool_desc* t, int32_t* tool_id);

/* A request: prompt tokens are fed as forced inputs (scan off); then up to max_new_tokens
 * are generated (greedy argmax, lowest id on ties; "temperature to be 0").
 * forced/forced_len: teacher forcing of the generated tokens of round 0 (parity/bench);
 * when forced_len > 0 the round ends after forced_len tokens.  synth_prefix_len tokens of
 * synthetic, already-RoPE'd KV (counter hash with synth_seed) precede the prompt.
 * The engine assigns req_id.  E_FULL: no free slot or pages -- retry later. */
typedef struct {
    int32_t tool_id; /* -1: no tool; the scan is off for this request */
    cvy_exec_mode mode;
    const int32_t* prompt;
    uint32_t prompt_len; /* >= 1 */
    uint32_t synth_prefix_len;
    uint64_t synth_seed;
    uint32_t max_new_tokens;
    const int32_t* forced;
    uint32_t forced_len;
    uint32_t reserve_tokens; /* extra KV tokens to reserve for later observation rounds */
    /* Multi-tool routing (NEXT-2, R24): a SET of region tools (FENCE and / or CALL
     * kinds, ids < 64) instead of one tool.  Outside a region every line is matched against
     * each tool's open marker ("```" TAG "\n" / "@call " TAG " ") and the marker that appears
     * selects the tool: its region's records carry its id ("the indicators for the start and
     * end of the tool"; "identifies the function name of the tool").
     * Lines outside a region are cut at the smallest max_segment_bytes of the set, which must
     * be >= every marker of the set.  tool_id must then be -1 or a member.  NULL / 0: one tool. */
    const int32_t* tool_set;
    uint32_t n_tool_set;
} cvy_request_desc;
cvy_status cvy_submit_request(cvy_engine* e, const cvy_request_desc* r, uint64_t* req_id);

/* One decode step for all in-flight requests (one graph launch).  Non-blocking except
 * that at most 2 steps are in flight and the ring must have worst-case space
 * (max_slots * 17 records) -- otherwise it waits for the GPU / the poller.
 * last_completed (optional) receives the stats of the most recently completed step. */
typedef struct {
    uint64_t step;
    uint32_t n_active, n_generated, n_segments, n_finished;
    float step_ms;
} cvy_step_info;
cvy_status cvy_step(cvy_engine* e, cvy_step_info* last_completed);

/* Wait until every launched step has completed. */
cvy_status cvy_sync(cvy_engine* e);

/* A completed partial-execution piece (or a round's FINAL tail) of one request.
 * byte_offset/byte_len index the request's byte stream of that round; token_index is the
 * 0-based index (within the round's generated tokens) of the token holding the segment's
 * last byte (FINAL: the round's last token, CVY_NO_TOKEN if none). */
typedef struct {
    uint64_t req_id;
    uint32_t round, seq;       /* seq: per request, from 0, no gaps, across rounds */
    uint32_t step, token_index;
    uint32_t byte_offset, byte_len;
    uint16_t delim_id, flags;  /* delim_id: LITERAL index / JSON 0=',' 1=close / NONE  */
    uint16_t slot;             /* engine slot that produced the record (diagnostic)   */
    int16_t tool;              /* tool the record is for: the request's tool, or for a tool
                                  set (cvy_request_desc.tool_set) the tool whose region the
                                  record belongs to; FINAL outside a region: -1           */
} cvy_segment;

/* Exactly one consumer thread.  Copies up to cap records (and their bytes, concatenated
 * in record order, if bytes != NULL) and returns E_AGAIN when the ring is empty.
 * A record is only returned if its bytes fit into bytes_cap. */
cvy_status cvy_poll_segments(cvy_engine* e, cvy_segment* out, uint32_t cap, uint32_t* n,
                             uint8_t* bytes, size_t bytes_cap, size_t* bytes_used);

/* Start the next round of a request parked after FINAL: the round's last generated
 * token followed by the observation tokens are fed as forced inputs (scan off), then
 * round+1 generates (max_new_tokens; optional teacher forcing).  E_STATE if not parked. */
cvy_status cvy_inject_observation(cvy_engine* e, uint64_t req_id, const int32_t* tokens,
                                  uint32_t n, uint32_t max_new_tokens, const int32_t* forced,
                                  uint32_t forced_len);

/* Idempotent.  A running round ends with FINAL|CANCELLED at the next step. */
cvy_status cvy_cancel_request(cvy_engine* e, uint64_t req_id);

/* Frees the slot and its pages.  Only valid when the request is parked or cancelled. */
cvy_status cvy_release_request(cvy_engine* e, uint64_t req_id);

/* Generated token ids of the current/last round of a request (copied out). */
cvy_status cvy_round_tokens(cvy_engine* e, uint64_t req_id, int32_t* out, uint32_t cap,
                            uint32_t* n);

/* Request state: 0 running, 1 parked (round finished), 2 cancelled, -1 unknown. */
int32_t cvy_request_state(cvy_engine* e, uint64_t req_id);

/* Parity only (requires CVY_ENGINE_DEBUG_LOGITS): last completed step's fp32 logits of
 * the request's slot, [vocab]. */
cvy_status cvy_debug_logits(cvy_engine* e, uint64_t req_id, float* out, uint32_t cap);

/* Device-side timing of the engine's kernels for measurement: per-step CUDA-event time
 * of the last step and the number of kernel launches per step. */
typedef struct {
    float last_step_ms;
    uint32_t launches_per_step;
    uint32_t slots_bucket; /* padded batch of the last launched step */
} cvy_perf_info;
cvy_status cvy_perf(cvy_engine* e, cvy_perf_info* out);

/* Per-kernel timing (measurement only).  When on, subsequent steps run a second graph
 * variant with a CUDA event pair around every kernel launch (programmatic dependent
 * launch disabled in that variant); cvy_kernel_times then returns the device time of each
 * launch of the most recently completed timed step, in launch order.
 * kind: 0 embed, 1 QKV GEMM, 2 attention, 3 attention merge, 4 O GEMM, 5 gate/up GEMM,
 *       6 down GEMM, 7 LM-head GEMM + sampling/scan epilogue, 8 persistent all-layers kernel
 *       (QKV, attention, O, gate/up and down of every layer in one launch), 9 its counter reset. */
typedef struct {
    int32_t kind, layer;
    float ms;
} cvy_kernel_time;
cvy_status cvy_set_kernel_timing(cvy_engine* e, int32_t on);
cvy_status cvy_kernel_times(cvy_engine* e, cvy_kernel_time* out, uint32_t cap, uint32_t* n);

/* In-graph kernel spans (measurement only).  When on, subsequent steps run a variant of the
 * production step graph -- same kernels, same launch order, programmatic dependent launch kept --
 * in which every launch records, with %globaltimer, the earliest moment one of its CTAs passed
 * its grid-dependency wait (t0) and the latest CTA exit (t1).  Consecutive kernels of one chain
 * therefore have disjoint spans, and sum(t1 - t0) of a kind is its share of the step's device
 * time.  cvy_kernel_spans returns the spans of the most recently completed span-recording step
 * (kind as in cvy_kernel_time; chain 1 = the second half-batch chain of the batch-split overlap,
 * else 0).  Errors: E_STATE without a graph path or before a recorded step. */
typedef struct {
    int32_t kind, layer, chain;
    uint64_t t0_ns, t1_ns;
} cvy_kernel_span;
cvy_status cvy_set_kernel_spans(cvy_engine* e, int32_t on);
cvy_status cvy_kernel_spans(cvy_engine* e, cvy_kernel_span* out, uint32_t cap, uint32_t* n);

/* Stream the engine launches on (cudaStream_t as void*), for external event timing. */
void* cvy_stream(cvy_engine* e);

/* Multi-GPU stats gather (NCCL all-gather over NVLink/NVSwitch of a 64-byte per-engine
 * stats record; one engine per GPU, all owned by this process). out: [n][8] uint64. */
cvy_status cvy_stats_allgather(cvy_engine* const* engines, int32_t n, uint64_t* out);

/* Test hook: copy an internal device buffer of the last completed step to host memory.
 * which: 0 x (fp32 [Bmax][d]), 1 act, 2 q (fp32 [Bmax][H*hd]), 3 o, 4 h (model dtype
 * [Bmax][act_ld]), 5 ssq (fp32 [d/128][Bmax]), 6 page table (int32 [max_slots][max_pages_per_slot]),
 * 7 last chunked-prefill row table (int32 [3][512]: slot, position, token); the last chunked-prefill
 * pass's buffers (512 rows): 8 x (fp32 [512][d]), 9 q (fp32 [512][H*hd]), 20 o, 21 h, 22 act
 * (model dtype [2 planes][512][act_ld]); 10-13 GEMM trace stamps (CVY_GEMM_TRACE_LAYER).
 * CVY_E_STATE if the engine has no such buffer.  *bytes receives the buffer size; if dst is
 * NULL only the size is returned. */
cvy_status cvy_debug_buffer(cvy_engine* e, int32_t which, void* dst, size_t cap, size_t* bytes);

/* Test / measurement hook: Y[b][n] = sum_k W[n][k] X[b][k] for b < B through the same
 * tcgen05 stream-K GEMM kernel the decode step uses (bf16 W [N][K], X [B][K] device
 * pointers, fp32 Y [B][N] device pointer; K % 64 == 0, B <= 512).  iters > 1 repeats the
 * launch and returns the mean device time per launch in *ms (CUDA events). */
cvy_status cvy_debug_gemm(const void* W, const void* X, float* Y, int32_t N, int32_t K, int32_t B,
                          int32_t iters, int32_t device, float* ms);

/* ======================================================================================
 * Native host runtime: the scheduler of PAPER.md:146 (Fig. 4)
 * above the engine, in C++ threads (no interpreter lock on the path):
 *   (1) requests are submitted (cvy_submit_request), (2) the calling thread runs decoding
 *   iterations back to back (cvy_step: continuous batching), (8) a poller thread drains the
 *   pinned segment ring (cvy_poll_segments) while decoding continues, and (6)/(7) tool
 *   executors run the pieces on worker threads beside decoding;
 *   Partial mode dispatches every piece the moment it is polled ("tool partial execution",
 *   PAPER.md:39, :144); Sequential mode holds a round's pieces until its FINAL record ("tool
 *   invocation always happens after decoding to the EOS"; reading R15);
 *   when a round's FINAL is in and all its pieces have executed, the round's observation is
 *   fed back (cvy_inject_observation, step (g)) and the next round decodes;
 *   a piece whose plan says `abort` cancels its request when it completes (the validator,
 *   PAPER.md:187, :223); with max_inflight > 0 a finished / aborted request's slot is
 *   released at once and the next queued request admitted (abort-and-refill, NEXT-3).
 * Pieces of one (request, round, instance) run serially in arrival order; instances run in
 * parallel (up to n_workers at a time); a piece also waits for its dependencies (earlier
 * pieces of the round: planning DAGs).  What a tool does with a piece is the
 * plan callback's business: it maps a piece (bytes, flags) to {skip, cost, instance, deps,
 * abort}; the built-in executor then occupies a worker for `cost_ms` (a tool stub with the
 * caller's seeded cost model; a real tool would run there).  All times are seconds on the
 * host steady clock, relative to cvy_runtime_run's start.
 * ====================================================================================== */
typedef struct cvy_runtime cvy_runtime;

/* Plan of one piece (filled by the plan callback; zero-initialised before the call). */
typedef struct {
    int32_t skip;        /* 1: not tool input (e.g. a FENCE marker, a drafted code line) */
    int32_t abort;       /* 1: cancel the request when this piece completes (validator) */
    double cost_ms;      /* executor time of the piece                                   */
    int32_t instance;    /* tool instance: pieces of one instance run serially           */
    uint32_t n_deps;     /* <= 8 indices of earlier accepted pieces of the same round    */
    int32_t deps[8];
} cvy_piece_plan;

/* Called on the poller thread for every polled piece (a non-FINAL record, or a FINAL with
 * bytes) of a round bound to a tool.  piece = index among the round's accepted pieces so far
 * (a skipped piece does not consume an index).  request = index into cvy_runtime_run's array. */
typedef void (*cvy_plan_fn)(void* user, uint32_t request, uint32_t round, uint32_t piece, const uint8_t* data,
                            uint32_t len, uint16_t flags, cvy_piece_plan* out);

typedef struct {
    cvy_exec_mode mode;
    uint32_t n_workers;     /* executor threads (1..4096): size it to the concurrent tool
                               calls the workload issues, or tool capacity binds          */
    uint32_t max_inflight;  /* 0: submit every request at t = 0                         */
    cvy_plan_fn plan;       /* required                                                 */
    void* plan_user;
    uint32_t poll_sleep_us; /* poller back-off when the ring is empty (0: 20 us)        */
} cvy_runtime_config;

typedef struct {
    const int32_t* forced;      /* teacher-forced generated tokens of the round (>= 1)  */
    uint32_t forced_len;
    int32_t tool_id;            /* -1: no tool                                          */
    const int32_t* observation; /* tokens injected after the round (before the next)    */
    uint32_t observation_len;
} cvy_round_desc;

typedef struct {
    const int32_t* prompt;
    uint32_t prompt_len;
    uint32_t synth_prefix_len;
    uint64_t synth_seed;
    const cvy_round_desc* rounds;
    uint32_t n_rounds;          /* >= 1 */
    double t_arrival;           /* seconds after cvy_runtime_run starts (0: at start); requests
                                   are admitted in arrival order once arrived (Poisson-arrival
                                   latency protocol)                        */
} cvy_rt_request;

/* Per request / round / piece logs (the inputs of the paper's latency model). */
typedef struct {
    uint64_t req_id;
    double t_arrival;                 /* as given; latency = t_done - t_arrival            */
    double t_submit, t_done, t_abort; /* t_submit: admitted; t_abort < 0: not aborted      */
    uint32_t n_rounds_run;
    uint32_t aborted;
} cvy_rt_request_log;
typedef struct {
    double t_start, t_final;          /* round start (submit / injection) and FINAL polled */
    uint32_t n_pieces;
} cvy_rt_round_log;
typedef struct {
    double t_avail, t_dispatch, t_begin, t_end; /* polled, released to the tool, started, done */
    double cost_ms;
    int32_t instance;
    uint32_t token_index;
    uint32_t n_deps;
    int32_t deps[8];
} cvy_rt_piece_log;
typedef struct {
    uint64_t steps, records, pieces, injections, cancels;
    double wall_s;
    double poller_cpu_s;    /* poller thread CPU time (polling + planning + dispatch)     */
    double dispatch_cpu_s;  /* of which: handling polled records                          */
    double driver_cpu_s;    /* the calling thread (cvy_step loop)                         */
    double worker_cpu_s;    /* executor threads (stub executors sleep: ~0)                */
} cvy_rt_stats;

cvy_status cvy_runtime_create(cvy_engine* e, const cvy_runtime_config* cfg, cvy_runtime** out);
/* Runs every request to completion (copies the descriptors; blocks the calling thread, which
 * drives cvy_step).  E_INVAL bad descriptors, E_FULL a request could not be admitted even
 * with the engine idle (a full engine otherwise queues the request until a slot frees), E_STATE
 * timeout or an engine error (see cvy_last_error).  May be
 * called again: each call replaces the previous logs. */
cvy_status cvy_runtime_run(cvy_runtime* rt, const cvy_rt_request* reqs, uint32_t n, double timeout_s);
cvy_status cvy_runtime_request_log(cvy_runtime* rt, uint32_t request, cvy_rt_request_log* out);
cvy_status cvy_runtime_round_log(cvy_runtime* rt, uint32_t request, uint32_t round, cvy_rt_round_log* out);
cvy_status cvy_runtime_piece_log(cvy_runtime* rt, uint32_t request, uint32_t round, uint32_t piece,
                                 cvy_rt_piece_log* out);
cvy_status cvy_runtime_stats(cvy_runtime* rt, cvy_rt_stats* out);
void cvy_runtime_destroy(cvy_runtime* rt);

#ifdef __cplusplus
}
#endif
#endif /* CONVEYOR_H */
