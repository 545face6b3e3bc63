/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the Conveyor
 * (arXiv 2406.00059) decode hot path computes.  Only tests/, the smoke() entry
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA path in
 * paper_2406_00059_b200/csrc (which re-implements the counter hash itself).
 *
 * Contents
 *   O-1  decoder forward (Mistral-7B family, random init), fp64 arithmetic.
 *        PAPER.md:71-73 (sec 2.1: KV cache, prefill/decode, autoregressive
 *        decoding), PAPER.md:191 (sec 4.1: Mistral-7B-Instruct-v0.2, temperature
 *        0 => greedy).  The paper is silent on the architecture; the steps follow
 *        the Mistral/Llama definition (DESIGN.md readings
 *        R1-R4) and are pinned against HF MistralForCausalLM in tests/.
 *   O-2  byte-stream segmentation ("parser ... emits completed pieces of data
 *        immediately"; "\n" or ";" indicators, PAPER.md:49;
 *        wait only for needed data).  Plain definition of
 *        SURVEY.md 8(c) O-2 / DESIGN.md R5-R12.
 *
 * Parity status: every function here is pinned by tests in tests/test_oracle_*.py
 * (HF cross-check, closed forms, brute force).  See DESIGN.md "Oracle pins".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------- */
/* Counter-based weight generator.                  */
/* w[tid][i] = a * (2*U(splitmix64(seed ^ tid*GOLD ^ i)) - 1),  U = top53 * 2^-53 */
/* The value is then rounded to fp32 (RNE) and, for bf16 models, to bf16 (RNE). */
/* ------------------------------------------------------------------------- */
static uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

static double bf16_round(double v) {
    /* round to fp32 (RNE), then fp32 -> bf16 (RNE); NaN never occurs here */
    float f = (float)v;
    uint32_t u;
    memcpy(&u, &f, 4);
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7FFFu + lsb;
    u &= 0xFFFF0000u;
    memcpy(&f, &u, 4);
    return (double)f;
}

static double hash_value(uint64_t seed, uint64_t tid, uint64_t i, double a, int bf16) {
    uint64_t h = splitmix64(seed ^ (tid * 0x9E3779B97F4A7C15ULL) ^ i);
    double u = (double)(h >> 11) * (1.0 / 9007199254740992.0);
    double v = a * (2.0 * u - 1.0);
    float f = (float)v;
    return bf16 ? bf16_round((double)f) : (double)f;
}

/* exported for tests: one generated value */
double orc_hash_value(uint64_t seed, uint64_t tid, uint64_t i, double a, int bf16) {
    return hash_value(seed, tid, i, a, bf16);
}
double orc_bf16_round(double v) { return bf16_round(v); }

/* ------------------------------------------------------------------------- */
/* O-1 model                                                                   */
/* ------------------------------------------------------------------------- */
typedef struct {
    int L, d, H, Hkv, hd, dff, V;
    double eps, rope_base;
} orc_model;

enum { W_Q = 0, W_K = 1, W_V = 2, W_O = 3, W_G = 4, W_U = 5, W_D = 6 };

typedef struct {
    orc_model m;
    uint64_t seed;
    int wbf16;     /* 1: weights are bf16 values, 0: fp32 values                  */
    int cache_weights;
    double** wcache; /* [1+8L+1] dense weight arrays when cached, else NULL       */
} orc_weights;

typedef struct {
    const orc_weights* w;
    int max_ctx;
    int len;        /* number of positions already in the cache */
    double* kv;     /* [L][max_ctx][2][Hkv][hd] */
} orc_req;

static uint64_t tensor_id(int l, int which) { return (uint64_t)(1 + 8 * l + which); }
static uint64_t lm_head_id(int L) { return (uint64_t)(1 + 8 * L); }

static void tensor_shape(const orc_model* m, uint64_t tid, int* rows, int* cols) {
    if (tid == 0) { *rows = m->V; *cols = m->d; return; }
    if (tid == lm_head_id(m->L)) { *rows = m->V; *cols = m->d; return; }
    int which = (int)((tid - 1) % 8);
    switch (which) {
        case W_Q: *rows = m->H * m->hd; *cols = m->d; break;
        case W_K: case W_V: *rows = m->Hkv * m->hd; *cols = m->d; break;
        case W_O: *rows = m->d; *cols = m->H * m->hd; break;
        case W_G: case W_U: *rows = m->dff; *cols = m->d; break;
        default: *rows = m->d; *cols = m->dff; break;
    }
}

static double weight_a(void) { return 0.02 * sqrt(3.0); }

orc_weights* orc_weights_create(const orc_model* m, uint64_t seed, int wbf16, int cache_weights) {
    orc_weights* w = (orc_weights*)calloc(1, sizeof(orc_weights));
    w->m = *m;
    w->seed = seed;
    w->wbf16 = wbf16;
    w->cache_weights = cache_weights;
    if (cache_weights) {
        int n = 2 + 8 * m->L;
        w->wcache = (double**)calloc((size_t)n, sizeof(double*));
        for (uint64_t tid = 0; tid < (uint64_t)n; ++tid) {
            if (tid != 0 && tid != lm_head_id(m->L) && ((tid - 1) % 8) == 7) continue;
            int r, c;
            tensor_shape(m, tid, &r, &c);
            double* buf = (double*)malloc((size_t)r * c * sizeof(double));
#pragma omp parallel for schedule(static)
            for (long i = 0; i < (long)r * c; ++i)
                buf[i] = hash_value(seed, tid, (uint64_t)i, weight_a(), wbf16);
            w->wcache[tid] = buf;
        }
    }
    return w;
}

void orc_weights_destroy(orc_weights* w) {
    if (!w) return;
    if (w->wcache) {
        for (int i = 0; i < 2 + 8 * w->m.L; ++i) free(w->wcache[i]);
        free(w->wcache);
    }
    free(w);
}

/* one row of a weight tensor, generated or from the cache */
static void weight_row(const orc_weights* w, uint64_t tid, int row, int cols, double* out) {
    if (w->wcache) {
        memcpy(out, w->wcache[tid] + (size_t)row * cols, (size_t)cols * sizeof(double));
        return;
    }
    for (int c = 0; c < cols; ++c)
        out[c] = hash_value(w->seed, tid, (uint64_t)row * cols + c, weight_a(), w->wbf16);
}

/* y_i[r] = sum_c W[r][c] * x_i[c] for n requests: a plain matrix-vector product
 * (row generated once, applied to every request). */
static void matvec(const orc_weights* w, uint64_t tid, int rows, int cols, int n,
                   double* const* x, double* const* y) {
#pragma omp parallel
    {
        double* row = (double*)malloc((size_t)cols * sizeof(double));
#pragma omp for schedule(static)
        for (int r = 0; r < rows; ++r) {
            weight_row(w, tid, r, cols, row);
            for (int i = 0; i < n; ++i) {
                double acc = 0.0;
                const double* xi = x[i];
                for (int c = 0; c < cols; ++c) acc += row[c] * xi[c];
                y[i][r] = acc;
            }
        }
        free(row);
    }
}

orc_req* orc_req_create(const orc_weights* w, int max_ctx) {
    orc_req* r = (orc_req*)calloc(1, sizeof(orc_req));
    r->w = w;
    r->max_ctx = max_ctx;
    const orc_model* m = &w->m;
    r->kv = (double*)calloc((size_t)m->L * max_ctx * 2 * m->Hkv * m->hd, sizeof(double));
    return r;
}
void orc_req_destroy(orc_req* r) {
    if (!r) return;
    free(r->kv);
    free(r);
}

static double* kv_at(orc_req* r, int l, int pos, int c, int g) {
    const orc_model* m = &r->w->m;
    return r->kv + ((((size_t)l * r->max_ctx + pos) * 2 + c) * m->Hkv + g) * m->hd;
}

/* Synthetic KV prefix: post-RoPE K/V values drawn from the
 * counter hash with tensor id 2^62 ^ (synth_seed*L + l), std 1, rounded to the cache
 * dtype (bf16 for bf16 models, fp32 otherwise). */
int orc_req_synth_prefix(orc_req* r, int prefix_len, uint64_t synth_seed) {
    const orc_model* m = &r->w->m;
    if (prefix_len > r->max_ctx) return -1;
    for (int l = 0; l < m->L; ++l) {
        uint64_t tid = (1ULL << 62) ^ (synth_seed * (uint64_t)m->L + (uint64_t)l);
        for (int pos = 0; pos < prefix_len; ++pos)
            for (int c = 0; c < 2; ++c)
                for (int g = 0; g < m->Hkv; ++g) {
                    double* dst = kv_at(r, l, pos, c, g);
                    for (int e = 0; e < m->hd; ++e) {
                        uint64_t i = ((((uint64_t)pos * 2 + c) * m->Hkv + g) * m->hd) + e;
                        dst[e] = hash_value(0, tid, i, sqrt(3.0), r->w->wbf16);
                    }
                }
    }
    r->len = prefix_len;
    return 0;
}

static double silu(double z) { return z / (1.0 + exp(-z)); }

/* RoPE, HF rotate_half convention: for i < hd/2, theta_i = base^(-2i/hd),
 * (a_i, a_{i+hd/2}) <- (a_i cos - a_{i+hd/2} sin, a_{i+hd/2} cos + a_i sin). */
static void rope(double* a, int hd, int pos, double base) {
    int half = hd / 2;
    for (int i = 0; i < half; ++i) {
        double theta = pow(base, -2.0 * (double)i / (double)hd);
        double ang = (double)pos * theta;
        double c = cos(ang), s = sin(ang);
        double x0 = a[i], x1 = a[i + half];
        a[i] = x0 * c - x1 * s;
        a[i + half] = x1 * c + x0 * s;
    }
}

/* RMSNorm input for the next GEMM: u = x * rsqrt(mean(x^2)+eps) * w, w (norm weight) = 1.0
 * (R3).  Returns the scale applied afterwards to the GEMM output (1: none; the activations
 * are exact). */
static double rms_input(const orc_weights* w, const double* x, int d, double* u) {
    double ms = 0.0;
    for (int i = 0; i < d; ++i) ms += x[i] * x[i];
    double s = 1.0 / sqrt(ms / (double)d + w->m.eps);
    for (int i = 0; i < d; ++i) u[i] = x[i] * s * 1.0;
    return 1.0;
}

/* One decode step for n independent requests: input token tok[i] at position
 * reqs[i]->len; appends K/V; writes logits [n][V]. Returns 0 or -1. */
int orc_step(orc_req* const* reqs, int n, const int32_t* tok, double* logits) {
    if (n <= 0) return 0;
    const orc_weights* w = reqs[0]->w;
    const orc_model* m = &w->m;
    const int d = m->d, H = m->H, Hkv = m->Hkv, hd = m->hd, dff = m->dff, V = m->V;
    for (int i = 0; i < n; ++i)
        if (reqs[i]->len >= reqs[i]->max_ctx || tok[i] < 0 || tok[i] >= V) return -1;

    double** h = (double**)malloc(n * sizeof(double*));
    double** u = (double**)malloc(n * sizeof(double*));
    double** q = (double**)malloc(n * sizeof(double*));
    double** k = (double**)malloc(n * sizeof(double*));
    double** v = (double**)malloc(n * sizeof(double*));
    double** o = (double**)malloc(n * sizeof(double*));
    double** y = (double**)malloc(n * sizeof(double*));
    double** g = (double**)malloc(n * sizeof(double*));
    double** up = (double**)malloc(n * sizeof(double*));
    double* sc = (double*)malloc(n * sizeof(double));
    int wide = dff > d ? dff : d;
    if (H * hd > wide) wide = H * hd;
    for (int i = 0; i < n; ++i) {
        h[i] = (double*)malloc(d * sizeof(double));
        u[i] = (double*)malloc(wide * sizeof(double));
        q[i] = (double*)malloc(H * hd * sizeof(double));
        k[i] = (double*)malloc(Hkv * hd * sizeof(double));
        v[i] = (double*)malloc(Hkv * hd * sizeof(double));
        o[i] = (double*)malloc(H * hd * sizeof(double));
        y[i] = (double*)malloc((V > wide ? V : wide) * sizeof(double));
        g[i] = (double*)malloc(dff * sizeof(double));
        up[i] = (double*)malloc(dff * sizeof(double));
        /* 1. h <- E[x] */
        weight_row(w, 0, tok[i], d, h[i]);
    }

    for (int l = 0; l < m->L; ++l) {
        /* 2.1 attention-input RMSNorm */
        for (int i = 0; i < n; ++i) sc[i] = rms_input(w, h[i], d, u[i]);
        /* 2.2 q, k, v projections */
        matvec(w, tensor_id(l, W_Q), H * hd, d, n, u, q);
        matvec(w, tensor_id(l, W_K), Hkv * hd, d, n, u, k);
        matvec(w, tensor_id(l, W_V), Hkv * hd, d, n, u, v);
#pragma omp parallel for schedule(dynamic)
        for (int i = 0; i < n; ++i) {
            orc_req* r = reqs[i];
            int pos = r->len;
            for (int e = 0; e < H * hd; ++e) q[i][e] *= sc[i];
            for (int e = 0; e < Hkv * hd; ++e) { k[i][e] *= sc[i]; v[i][e] *= sc[i]; }
            /* 2.3 RoPE on q and k at position pos */
            for (int j = 0; j < H; ++j) rope(q[i] + j * hd, hd, pos, m->rope_base);
            for (int j = 0; j < Hkv; ++j) rope(k[i] + j * hd, hd, pos, m->rope_base);
            /* 2.4 append (k, v) to the cache (bf16 cache format rounds, R4) */
            for (int j = 0; j < Hkv; ++j) {
                double* kd = kv_at(r, l, pos, 0, j);
                double* vd = kv_at(r, l, pos, 1, j);
                for (int e = 0; e < hd; ++e) {
                    double kk = k[i][j * hd + e], vv = v[i][j * hd + e];
                    if (w->wbf16) { kk = bf16_round(kk); vv = bf16_round(vv); }
                    else { kk = (double)(float)kk; vv = (double)(float)vv; }
                    kd[e] = kk;
                    vd[e] = vv;
                }
            }
            /* 2.5 attention over positions [0, pos], head j uses kv head floor(j*Hkv/H) */
            double* s = (double*)malloc((size_t)(pos + 1) * sizeof(double));
            for (int j = 0; j < H; ++j) {
                int gk = (j * Hkv) / H;
                const double* qj = q[i] + j * hd;
                double mx = -INFINITY;
                for (int t = 0; t <= pos; ++t) {
                    const double* kt = kv_at(r, l, t, 0, gk);
                    double acc = 0.0;
                    for (int e = 0; e < hd; ++e) acc += qj[e] * kt[e];
                    s[t] = acc / sqrt((double)hd);
                    if (s[t] > mx) mx = s[t];
                }
                double den = 0.0;
                for (int t = 0; t <= pos; ++t) { s[t] = exp(s[t] - mx); den += s[t]; }
                double* oj = o[i] + j * hd;
                for (int e = 0; e < hd; ++e) oj[e] = 0.0;
                for (int t = 0; t <= pos; ++t) {
                    const double* vt = kv_at(r, l, t, 1, gk);
                    double p = s[t] / den;
                    for (int e = 0; e < hd; ++e) oj[e] += p * vt[e];
                }
            }
            free(s);
        }
        /* 2.6 h <- h + o W_o^T */
        matvec(w, tensor_id(l, W_O), d, H * hd, n, o, y);
        for (int i = 0; i < n; ++i)
            for (int e = 0; e < d; ++e) h[i][e] += y[i][e];
        /* 2.7 MLP-input RMSNorm */
        for (int i = 0; i < n; ++i) sc[i] = rms_input(w, h[i], d, u[i]);
        /* 2.8 SwiGLU MLP */
        matvec(w, tensor_id(l, W_G), dff, d, n, u, g);
        matvec(w, tensor_id(l, W_U), dff, d, n, u, up);
        for (int i = 0; i < n; ++i)
            for (int e = 0; e < dff; ++e) {
                double a = silu(g[i][e] * sc[i]) * (up[i][e] * sc[i]);
                u[i][e] = a;
            }
        matvec(w, tensor_id(l, W_D), d, dff, n, u, y);
        for (int i = 0; i < n; ++i)
            for (int e = 0; e < d; ++e) h[i][e] += y[i][e];
    }
    /* 3. logits = RMSNorm(h) W_lm^T */
    for (int i = 0; i < n; ++i) sc[i] = rms_input(w, h[i], d, u[i]);
    matvec(w, lm_head_id(m->L), V, d, n, u, y);
    for (int i = 0; i < n; ++i) {
        for (int e = 0; e < V; ++e) logits[(size_t)i * V + e] = y[i][e] * sc[i];
        reqs[i]->len += 1;
    }
    for (int i = 0; i < n; ++i) {
        free(h[i]); free(u[i]); free(q[i]); free(k[i]); free(v[i]);
        free(o[i]); free(y[i]); free(g[i]); free(up[i]);
    }
    free(h); free(u); free(q); free(k); free(v); free(o); free(y); free(g); free(up); free(sc);
    return 0;
}

/* 4. greedy choice: argmax, lowest index wins ties, NaN treated as -inf (R6). */
int orc_argmax(const double* x, int n) {
    int best = -1;
    double bv = -INFINITY;
    for (int i = 0; i < n; ++i) {
        double v = x[i];
        if (v != v) v = -INFINITY;
        if (best < 0 || v > bv) { bv = v; best = i; }
    }
    return best;
}

/* Dump one generated weight tensor (fp64) for cross-checks; rows*cols doubles. */
int orc_dump_tensor(const orc_weights* w, uint64_t tid, double* out) {
    int r, c;
    tensor_shape(&w->m, tid, &r, &c);
    for (int i = 0; i < r; ++i) weight_row(w, tid, i, c, out + (size_t)i * c);
    return r * c;
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------------- */
/* O-2 segmentation: plain definition                                          */
/* ------------------------------------------------------------------------- */
enum { ORC_PARSER_LITERAL = 0, ORC_PARSER_JSON_MEMBER = 1, ORC_PARSER_JSON_OBJECT = 2 };
enum { ORC_FLAG_FINAL = 1, ORC_FLAG_OVERFLOW = 2, ORC_FLAG_CANCELLED = 4 };
#define ORC_DELIM_NONE 0xFFFF

/* Cuts of stream S[0,n).  LITERAL (R5-R8): c_0 = 0,
 *   c_{j+1} = min{ p > c_j : exists i, |d_i| <= p - c_j and S[p-|d_i|, p) = d_i },
 * delim_id = smallest matching i; if p - c_j reaches max_seg first: OVERFLOW cut.
 * JSON (R10-R11): automaton over (depth, in_str, esc); ',' at depth 1 cuts
 * (MEMBER only), a closing bracket that brings depth to 0 cuts (delim_id 1).
 * Output: cut end offsets, delim ids, flags.  Returns the number of cuts (the
 * tail S[c_last, n) is not a cut). */
int orc_segment(int kind, int n_delims, const uint8_t* delims /*[8][8]*/, const int* lens,
                int max_seg, const uint8_t* S, int n, int* cut_end, int* delim_id, int* flags,
                int cap) {
    int ncut = 0;
    int c = 0;
    if (kind == ORC_PARSER_LITERAL) {
        for (int p = c + 1; p <= n; ++p) {
            int hit = -1;
            for (int i = 0; i < n_delims && hit < 0; ++i) {
                int L = lens[i];
                if (L <= p - c && memcmp(S + p - L, delims + 8 * i, (size_t)L) == 0) hit = i;
            }
            if (hit >= 0 || p - c == max_seg) {
                if (ncut >= cap) return -1;
                cut_end[ncut] = p;
                delim_id[ncut] = hit >= 0 ? hit : ORC_DELIM_NONE;
                flags[ncut] = hit >= 0 ? 0 : ORC_FLAG_OVERFLOW;
                ++ncut;
                c = p;
            }
        }
        return ncut;
    }
    int depth = 0, in_str = 0, esc = 0;
    for (int p = 1; p <= n; ++p) {
        uint8_t b = S[p - 1];
        int cut = -1;
        if (in_str) {
            if (esc) esc = 0;
            else if (b == '\\') esc = 1;
            else if (b == '"') in_str = 0;
        } else if (depth == 0) {
            if (b == '{' || b == '[') depth = 1;
        } else {
            if (b == '"') in_str = 1;
            else if (b == '{' || b == '[') { if (depth < 127) depth += 1; }
            else if (b == '}' || b == ']') { depth -= 1; if (depth == 0) cut = 1; }
            else if (b == ',' && depth == 1 && kind == ORC_PARSER_JSON_MEMBER) cut = 0;
        }
        if (cut >= 0 || p - c == max_seg) {
            if (ncut >= cap) return -1;
            cut_end[ncut] = p;
            delim_id[ncut] = cut >= 0 ? cut : ORC_DELIM_NONE;
            flags[ncut] = cut >= 0 ? 0 : ORC_FLAG_OVERFLOW;
            ++ncut;
            c = p;
        }
    }
    return ncut;
}
