/*
 * oracle.c -- CPU ORACLE for the fused EmbeddingBag(sum) + All-to-All of arXiv 2305.06942.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_2305_06942_b200/) never links, imports or calls anything in oracle/, and the two
 * share no code: no headers, no helpers, no constants beyond what the paper states.
 *
 * Plain, slow, obviously correct, single-threaded C.  Compile with
 *     gcc -O2 -ffp-contract=off -fPIC -shared   (never -ffast-math)
 * so that every float add below is one IEEE-754 binary32 round-to-nearest-even add.
 *
 * Citations: "P:n" = PAPER.md line n (the paper's LaTeX source), with section;
 *            "S:n" = SPEC.md line n (a CPU-simulator spec written from the paper).
 *            "R#n" = reading n in DESIGN.md section "Readings of the paper".
 *
 * What is computed (plain definition):
 *   For every destination rank s, local row i in [0, b_s), global table g owned by rank r
 *   (local table t = g - toff_r), and d in [0, D):
 *       j  = p_s + i                                  contiguous batch blocks      P:145 (Sec 3.2)
 *       acc = +0                                      R#5
 *       for k = offsets_r[t*B + j] .. offsets_r[t*B + j + 1] - 1 (ascending):
 *           acc = acc + W_g[indices_r[k]][d]          sum pooling                  P:119 (Sec 3.1)
 *       out_s[i][g*D + d] = acc                       {local batch, numTables x D} P:147 (Sec 3.2)
 *   with g = toff_r + t, toff_r = sum_{q<r} T_q (rank-major table ids, R#2).
 *
 * Parity status of each function (pins in tests/test_oracle.py):
 *   oracle_destination      pinned: P:145 worked example (Fig. superOp), bijection
 *   oracle_emb_a2a          pinned: hand golden example, brute-force one-hot, torch embedding_bag
 *                           special case (W=1), exact-int invariants, fp64 error bound,
 *                           mass conservation, bag permutation
 *   oracle_emb_a2a_rows     pinned: equals oracle_emb_a2a on every row at small sizes +
 *                           procedural values pinned independently (closed-form values)
 *   oracle_table_value      pinned: closed-form value ranges / grid, splitmix64 published vectors
 *   oracle_slice_plan       pinned: P:145-147 example (B=4, N=2, S=2 -> 2 slices/table),
 *                           S:144 clipping example (S=3, b=4 -> 3,1), partition invariant
 *   oracle_round_to_half    pinned: numpy float32 -> float16 and torch float32 -> bfloat16
 *                           (both round-to-nearest-even) on every 16-bit high half x boundary /
 *                           tie / random low halves, hand-worked ties, overflow, subnormals
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_OK 0
#define ORACLE_EINVAL 1   /* malformed problem (partition, offsets) */
#define ORACLE_EINDEX 8   /* index out of range: a workload error */
#define ORACLE_ECAP 9     /* output capacity too small */

/* ------------------------------------------------------------------------------------------
 * Input generator for procedural tables.  This is NOT the
 * method's arithmetic: it is the oracle's own copy of the counter-based generator that
 * the device fill kernel (synth/) implements independently.  splitmix64 is the
 * standard Steele/Lea/Flood finaliser.
 * ---------------------------------------------------------------------------------------- */
uint64_t oracle_splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* value of W_g[row][d]; mode 0 = fp32 grid values in [-1,1), mode 1 = exact-int in [-8,7],
 * mode 2 = k * 2^-7, k in [-128, 127] (exactly representable in bf16 and fp16) */
float oracle_table_value(uint64_t seed, int mode, int64_t g, int64_t row, int64_t d) {
    uint64_t key = (((uint64_t)g * 8388608ULL + (uint64_t)row) * 1024ULL) + (uint64_t)d;
    uint64_t x = oracle_splitmix64(key ^ oracle_splitmix64(seed));
    if (mode == 1) {
        int64_t v = (int64_t)(x >> 60) - 8;
        return (float)v;
    }
    if (mode == 2) {
        int64_t k = (int64_t)(x >> 56) - 128;
        return (float)((double)k / 128.0);
    }
    int64_t q = (int64_t)(x >> 40) - 8388608;   /* [-2^23, 2^23) */
    return (float)((double)q / 8388608.0);      /* exact: |q| < 2^24 */
}

/* ------------------------------------------------------------------------------------------
 * Tables: either materialised (host arrays, row-major [rows][D]) or procedural.
 * ---------------------------------------------------------------------------------------- */
#define ORACLE_F32 0
#define ORACLE_BF16 1
#define ORACLE_F16 2
#define ORACLE_SUM 0
#define ORACLE_MEAN 1

typedef struct {
    int procedural;
    uint64_t seed;
    int mode;
    const void* const* ptr;    /* G pointers when materialised */
    int dtype;                 /* element type of materialised tables */
    int D;
} tables_t;

/* bfloat16 bits -> float: the bf16 value is the top 16 bits of the binary32 (exact) */
float oracle_bf16_to_float(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* IEEE binary16 bits -> float (exact; subnormals, infinities and NaN included) */
float oracle_f16_to_float(uint16_t h) {
    uint32_t sign = (uint32_t)(h >> 15) << 31;
    uint32_t exp = (h >> 10) & 0x1F;
    uint32_t man = h & 0x3FF;
    uint32_t u;
    if (exp == 0) {
        if (man == 0) {
            u = sign;
        } else {                         /* subnormal: man * 2^-24 */
            float f = (float)man * (1.0f / 16777216.0f);
            memcpy(&u, &f, 4);
            u |= sign;
        }
    } else if (exp == 31) {
        u = sign | 0x7F800000u | (man << 13);
    } else {
        u = sign | ((exp - 15 + 127) << 23) | (man << 13);
    }
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* ------------------------------------------------------------------------------------------
 * 16-bit output (f2, SURVEY 8(f) item 2 "fp16 output to halve NVLink bytes"; reading R#32):
 * the pooled value is the fp32 result above, then rounded ONCE to the output type, to nearest,
 * ties to even (IEEE 754 roundTiesToEven).  Written from that definition: over the positive
 * patterns 0 .. +inf the values of a 16-bit float grow with the bit pattern, so the two
 * candidates bracketing |v| are found by bisection over the patterns; the nearer one wins, a
 * tie goes to the even pattern (last mantissa bit 0).  +inf stands in as the next value after
 * the largest finite one with its unbounded-exponent value (2^128 for bfloat16, 2^16 for
 * binary16), which is IEEE's overflow rule for roundTiesToEven.  The sign is copied (-0 -> -0).
 * NaN -> the quiet NaN of the type (never produced by finite tables).
 * ---------------------------------------------------------------------------------------- */
static double half_pattern_value(uint16_t h, int dtype) {   /* positive patterns only */
    if (dtype == ORACLE_BF16) {
        if (h == 0x7F80) return 340282366920938463463374607431768211456.0;   /* 2^128 */
        return (double)oracle_bf16_to_float(h);
    }
    if (h == 0x7C00) return 65536.0;                                           /* 2^16 */
    return (double)oracle_f16_to_float(h);
}

uint16_t oracle_round_to_half(float v, int dtype) {
    const uint16_t inf = dtype == ORACLE_BF16 ? 0x7F80 : 0x7C00;
    const uint16_t qnan = dtype == ORACLE_BF16 ? 0x7FC0 : 0x7E00;
    uint32_t u;
    memcpy(&u, &v, 4);
    const uint16_t sign = (uint16_t)((u >> 31) << 15);
    if (v != v) return (uint16_t)(sign | qnan);
    const double a = v < 0 ? -(double)v : (double)v;       /* exact */
    if (a >= half_pattern_value(inf, dtype)) return (uint16_t)(sign | inf);
    /* largest positive pattern lo with value(lo) <= a (lo < inf) */
    uint16_t lo = 0, hi = inf;                               /* value(lo) <= a < value(hi) */
    while (hi - lo > 1) {
        const uint16_t mid = (uint16_t)(lo + (hi - lo) / 2);
        if (half_pattern_value(mid, dtype) <= a) lo = mid; else hi = mid;
    }
    const double dlo = a - half_pattern_value(lo, dtype);
    const double dhi = half_pattern_value(hi, dtype) - a;
    uint16_t r;
    if (dlo < dhi) r = lo;
    else if (dhi < dlo) r = hi;
    else r = (lo & 1) ? hi : lo;                             /* tie: even pattern */
    return (uint16_t)(sign | r);
}

/* Element-wise over an array (the oracle's fp32 output -> 16-bit output bits). */
void oracle_round_array(const float* in, uint16_t* out, int64_t n, int dtype) {
    for (int64_t k = 0; k < n; ++k) out[k] = oracle_round_to_half(in[k], dtype);
}

static float table_at(const tables_t* tb, int64_t g, int64_t row, int64_t d) {
    if (tb->procedural) return oracle_table_value(tb->seed, tb->mode, g, row, d);
    int64_t e = row * tb->D + d;
    if (tb->dtype == ORACLE_BF16) return oracle_bf16_to_float(((const uint16_t*)tb->ptr[g])[e]);
    if (tb->dtype == ORACLE_F16) return oracle_f16_to_float(((const uint16_t*)tb->ptr[g])[e]);
    return ((const float*)tb->ptr[g])[e];
}

/* ------------------------------------------------------------------------------------------
 * Placement.  P:145 (Sec 3.2): "first half of global batch stored in node 0 and second half
 * in node 1" -> contiguous batch blocks given by the prefix p (R#1).  Returns the destination
 * rank s with p_s <= j < p_{s+1} and the local row i = j - p_s.  Linear scan: plain.
 * ---------------------------------------------------------------------------------------- */
int oracle_destination(int W, const int64_t* part, int64_t j, int* s_out, int64_t* i_out) {
    if (j < 0 || j >= part[W]) return ORACLE_EINVAL;
    for (int s = 0; s < W; ++s) {
        if (part[s] <= j && j < part[s + 1]) {
            *s_out = s;
            *i_out = j - part[s];
            return ORACLE_OK;
        }
    }
    return ORACLE_EINVAL;
}

/* ------------------------------------------------------------------------------------------
 * Validation, S:113 (out-of-range index is a workload error) and R#1/R#8 (CSR conventions).
 * ---------------------------------------------------------------------------------------- */
static int validate(int W, const int64_t* part, int64_t B, const int32_t* T,
                    const int64_t* rows, const int32_t* const* indices,
                    const int32_t* const* offsets, const int64_t* nnz) {
    if (W < 1 || B < 0) return ORACLE_EINVAL;
    if (part[0] != 0 || part[W] != B) return ORACLE_EINVAL;
    for (int s = 0; s < W; ++s) if (part[s + 1] < part[s]) return ORACLE_EINVAL;
    int64_t g = 0;
    for (int r = 0; r < W; ++r) {
        if (T[r] < 0) return ORACLE_EINVAL;
        const int32_t* off = offsets[r];
        int64_t n = (int64_t)T[r] * B;
        if (n > 0) {
            if (off[0] != 0) return ORACLE_EINVAL;
            for (int64_t q = 0; q < n; ++q) if (off[q + 1] < off[q]) return ORACLE_EINVAL;
            if (off[n] != nnz[r]) return ORACLE_EINVAL;
        }
        for (int t = 0; t < T[r]; ++t, ++g) {
            for (int64_t q = (int64_t)t * B; q < (int64_t)(t + 1) * B; ++q) {
                for (int64_t k = off[q]; k < off[q + 1]; ++k) {
                    int32_t idx = indices[r][k];
                    if (idx < 0 || (int64_t)idx >= rows[g]) return ORACLE_EINDEX;
                }
            }
        }
    }
    return ORACLE_OK;
}

/* ------------------------------------------------------------------------------------------
 * Pooling of one bag, P:119 (Sec 3.1): the embedding operator "accesses one or more vectors
 * from the embedding table and pools (reduction-like operation) them" (the paper names
 * EmbeddingBag_updateOutputKernel_sum_mean).  Ascending k, start from +0.0 (R#5), one binary32
 * add per element (fp32: R#14); an empty bag gives +0.0 (R#4).  Optional per-sample weight w_k:
 * acc = acc + fl(w_k * x) (R#26).  Mean: acc / L with IEEE binary32 division; empty bag 0 (R#27).
 * bf16 / fp16 tables are converted exactly to binary32 before the add (R#28).
 * ---------------------------------------------------------------------------------------- */
static void pool_bag_f32(const tables_t* tb, int64_t g, const int32_t* idx, const float* w,
                         int64_t lo, int64_t hi, int D, int pooling, float* out) {
    for (int d = 0; d < D; ++d) {
        float acc = +0.0f;
        for (int64_t k = lo; k < hi; ++k) {
            volatile float x = table_at(tb, g, idx[k], d);   /* volatile: no reassociation */
            if (w) {                      /* per-sample weight: product rounded, then added (R#26) */
                volatile float y = w[k] * x;
                acc = acc + y;
            } else {
                acc = acc + x;
            }
        }
        if (pooling == ORACLE_MEAN && hi > lo) acc = acc / (float)(hi - lo);   /* R#27 */
        out[d] = acc;
    }
}

/* The same sum in binary64: the exact-arithmetic reference used to pin the fp32 result within
 * the textbook bound |fl(sum) - sum| <= gamma_{L-1} * sum|x| (tests). */
static void pool_bag_f64(const tables_t* tb, int64_t g, const int32_t* idx, const float* w,
                         int64_t lo, int64_t hi, int D, int pooling, double* out) {
    for (int d = 0; d < D; ++d) {
        double acc = 0.0;
        for (int64_t k = lo; k < hi; ++k)
            acc = acc + (w ? (double)w[k] : 1.0) * (double)table_at(tb, g, idx[k], d);
        if (pooling == ORACLE_MEAN && hi > lo) acc = acc / (double)(hi - lo);
        out[d] = acc;
    }
}

/* ------------------------------------------------------------------------------------------
 * The whole reshuffled output for one destination row (s, i): all G tables, in g order.
 * output shape {local batch size, numTables x D}; column block of g is [gD, (g+1)D).
 * ---------------------------------------------------------------------------------------- */
static void one_row(int W, const int64_t* part, int D, int64_t B, const int32_t* T,
                    const tables_t* tb, const int32_t* const* indices,
                    const int32_t* const* offsets, const float* const* weights, int pooling,
                    int s, int64_t i, int precision, void* row_out /* G*D elements */) {
    int64_t j = part[s] + i;
    int64_t g = 0;
    for (int r = 0; r < W; ++r) {                              /* owner rank of table g */
        for (int t = 0; t < T[r]; ++t, ++g) {                  /* g = toff_r + t (R#2) */
            int64_t lo = offsets[r][(int64_t)t * B + j];
            int64_t hi = offsets[r][(int64_t)t * B + j + 1];
            const float* w = weights ? weights[r] : NULL;
            if (precision == 64)
                pool_bag_f64(tb, g, indices[r], w, lo, hi, D, pooling, (double*)row_out + g * D);
            else
                pool_bag_f32(tb, g, indices[r], w, lo, hi, D, pooling, (float*)row_out + g * D);
        }
    }
}

/* Full oracle over materialised tables.  out[s] -> [b_s][G*D], float (precision 32) or double
 * (precision 64).  Every cell is written exactly once (placement is a bijection).
 * tables: G pointers to [rows_g][D] elements of `dtype` (ORACLE_F32 / BF16 / F16);
 * weights: NULL, or W per-rank arrays of per-sample weights aligned with indices (sum only);
 * pooling: ORACLE_SUM or ORACLE_MEAN (P:119 EmbeddingBag_..._sum_mean). */
int oracle_emb_a2a_ex(int W, const int64_t* part, int D, int64_t B, const int32_t* T,
                      const void* const* tables, int dtype, const int64_t* rows,
                      const int32_t* const* indices, const int32_t* const* offsets,
                      const float* const* weights, const int64_t* nnz, int pooling,
                      int precision, void* const* out) {
    int rc = validate(W, part, B, T, rows, indices, offsets, nnz);
    if (rc) return rc;
    if (weights && pooling != ORACLE_SUM) return ORACLE_EINVAL;   /* as torch: sum only */
    int64_t G = 0;
    for (int r = 0; r < W; ++r) G += T[r];
    tables_t tb = {0, 0, 0, tables, dtype, D};
    size_t esz = precision == 64 ? sizeof(double) : sizeof(float);
    for (int s = 0; s < W; ++s)
        for (int64_t i = 0; i < part[s + 1] - part[s]; ++i)
            one_row(W, part, D, B, T, &tb, indices, offsets, weights, pooling, s, i, precision,
                    (char*)out[s] + (size_t)(i * G * D) * esz);
    return ORACLE_OK;
}

int oracle_emb_a2a(int W, const int64_t* part, int D, int64_t B, const int32_t* T,
                   const float* const* tables, const int64_t* rows,
                   const int32_t* const* indices, const int32_t* const* offsets,
                   const int64_t* nnz, int precision, void* const* out) {
    return oracle_emb_a2a_ex(W, part, D, B, T, (const void* const*)tables, ORACLE_F32, rows,
                             indices, offsets, NULL, nnz, ORACLE_SUM, precision, out);
}

/* Selected rows of out_s with procedural tables (for full-size sampled parity).
 * sel_i: n_sel local row ids of destination s; out: [n_sel][G*D]. */
int oracle_emb_a2a_rows_ex(uint64_t seed, int mode, int W, const int64_t* part, int D, int64_t B,
                           const int32_t* T, const int64_t* rows, const int32_t* const* indices,
                           const int32_t* const* offsets, const float* const* weights,
                           const int64_t* nnz, int pooling, int s, const int64_t* sel_i,
                           int64_t n_sel, int precision, void* out, int check_inputs) {
    if (check_inputs) {
        int rc = validate(W, part, B, T, rows, indices, offsets, nnz);
        if (rc) return rc;
    }
    if (s < 0 || s >= W) return ORACLE_EINVAL;
    if (weights && pooling != ORACLE_SUM) return ORACLE_EINVAL;
    int64_t G = 0;
    for (int r = 0; r < W; ++r) G += T[r];
    tables_t tb = {1, seed, mode, NULL, ORACLE_F32, D};
    size_t esz = precision == 64 ? sizeof(double) : sizeof(float);
    for (int64_t q = 0; q < n_sel; ++q) {
        if (sel_i[q] < 0 || sel_i[q] >= part[s + 1] - part[s]) return ORACLE_EINVAL;
        one_row(W, part, D, B, T, &tb, indices, offsets, weights, pooling, s, sel_i[q], precision,
                (char*)out + (size_t)(q * G * D) * esz);
    }
    return ORACLE_OK;
}

int oracle_emb_a2a_rows(uint64_t seed, int mode, int W, const int64_t* part, int D, int64_t B,
                        const int32_t* T, const int64_t* rows, const int32_t* const* indices,
                        const int32_t* const* offsets, const int64_t* nnz, int s,
                        const int64_t* sel_i, int64_t n_sel, int precision, void* out,
                        int check_inputs) {
    return oracle_emb_a2a_rows_ex(seed, mode, W, part, D, B, T, rows, indices, offsets, NULL, nnz,
                                  ORACLE_SUM, s, sel_i, n_sel, precision, out, check_inputs);
}

/* ------------------------------------------------------------------------------------------
 * Backward + SGD update (the paper's future work): the DP -> MP
 * All-to-All of the pooled-output gradient and the embedding-gradient scatter/update.
 * For every global table g (owner r, local t) and row x:
 *     acc = +0;  for k ascending over table t's positions in indices_r with indices_r[k] == x:
 *         j = bag of k (offsets_r[t*B + j] <= k < offsets_r[t*B + j + 1]), s = dest(j), i = j - p_s
 *         c = grad_s[i][g*D + d]            (sum)
 *         c = fl(w_k * grad_s[i][g*D + d])  (weighted)          R#26
 *         c = fl(grad_s[i][g*D + d] / L_j)  (mean)              R#27
 *         acc = fl(acc + c)
 *     if x occurs at all:  W_g[x][d] = fl(W_g[x][d] - fl(lr * acc))          R#29
 * tables: G fp32 arrays, updated in place.  grad: W per-destination arrays [b_s][G*D] fp32.
 * Plain and slow: for every row, a scan over all of the table's positions.
 * ---------------------------------------------------------------------------------------- */
int oracle_backward_sgd(int W, const int64_t* part, int D, int64_t B, const int32_t* T,
                        float* const* tables, const int64_t* rows,
                        const int32_t* const* indices, const int32_t* const* offsets,
                        const float* const* weights, const int64_t* nnz, int pooling,
                        const float* const* grad, float lr) {
    int rc = validate(W, part, B, T, rows, indices, offsets, nnz);
    if (rc) return rc;
    if (weights && pooling != ORACLE_SUM) return ORACLE_EINVAL;
    int64_t G = 0;
    for (int r = 0; r < W; ++r) G += T[r];
    float* acc = (float*)malloc(sizeof(float) * (D > 0 ? D : 1));
    if (!acc) return ORACLE_EINVAL;
    int64_t g = 0;
    for (int r = 0; r < W; ++r) {
        for (int t = 0; t < T[r]; ++t, ++g) {
            const int32_t* off = offsets[r];
            const int64_t k0 = off[(int64_t)t * B], k1 = off[(int64_t)(t + 1) * B];
            for (int64_t x = 0; x < rows[g]; ++x) {
                int found = 0;
                for (int d = 0; d < D; ++d) acc[d] = +0.0f;
                int64_t j = 0;
                for (int64_t k = k0; k < k1; ++k) {
                    while (off[(int64_t)t * B + j + 1] <= k) ++j;      /* bag of position k */
                    if (indices[r][k] != x) continue;
                    found = 1;
                    int s;
                    int64_t i;
                    oracle_destination(W, part, j, &s, &i);
                    const float* gr = grad[s] + (i * G + g) * D;
                    const int64_t L = off[(int64_t)t * B + j + 1] - off[(int64_t)t * B + j];
                    for (int d = 0; d < D; ++d) {
                        volatile float c = gr[d];
                        if (weights) c = weights[r][k] * c;
                        else if (pooling == ORACLE_MEAN) c = c / (float)L;
                        acc[d] = acc[d] + c;
                    }
                }
                if (!found) continue;
                for (int d = 0; d < D; ++d) {
                    volatile float step = lr * acc[d];
                    tables[g][x * D + d] = tables[g][x * D + d] - step;
                }
            }
        }
    }
    free(acc);
    return ORACLE_OK;
}

/* ------------------------------------------------------------------------------------------
 * Slice plan of rank r (row a1).  P:147: communication happens per *slice* of S output vectors;
 * "the slice index along with the global batch size and node count can then be used to
 * determine if the slice needs to be communicated remotely"; slices never cross a
 * destination block (clipped at block ends).  P:151: "logical WGs computing slices for remote
 * communication are computed ahead of WGs computing locally consumed slices".
 *
 * Order (R#19):  order 0 = comm-aware, staggered destinations s = (r+1..r+W-1) mod W, then s = r;
 *                order 1 = comm-aware, ascending remote s (skipping r), then s = r;
 *                order 2 = oblivious, s = 0..W-1.
 * Within one destination: table-major (t outer, slice c inner).
 * out: [n][4] = (s, t, i0, nb).  Returns the slice count via *n_out.
 * ---------------------------------------------------------------------------------------- */
int oracle_slice_plan(int r, int W, const int64_t* part, int T_r, int64_t S, int order,
                      int32_t* out, int64_t cap, int64_t* n_out) {
    if (S < 1 || r < 0 || r >= W || T_r < 0) return ORACLE_EINVAL;
    int64_t n = 0;
    for (int k = 0; k < W; ++k) {
        int s;
        if (order == 0)      s = (k < W - 1) ? (r + 1 + k) % W : r;
        else if (order == 1) s = (k < W - 1) ? (k < r ? k : k + 1) : r;
        else                 s = k;
        int64_t b_s = part[s + 1] - part[s];
        for (int t = 0; t < T_r; ++t) {
            for (int64_t i0 = 0; i0 < b_s; i0 += S) {
                int64_t nb = b_s - i0 < S ? b_s - i0 : S;
                if (n < cap) {
                    out[4 * n + 0] = s;
                    out[4 * n + 1] = t;
                    out[4 * n + 2] = (int32_t)i0;
                    out[4 * n + 3] = (int32_t)nb;
                }
                ++n;
            }
        }
    }
    *n_out = n;
    return n <= cap ? ORACLE_OK : ORACLE_ECAP;
}

/* Number of slice-ready signals rank src sends to rank dst per forward (rows a7/a8): one per
 * remote slice (the last finisher of a slice sets that slice's sliceRdy flag on the
 * remote node), i.e. T_src * ceil(b_dst / S); 0 when src == dst (R#13: local slices need none). */
int64_t oracle_signal_count(int src, int dst, const int32_t* T, const int64_t* part, int64_t S) {
    if (src == dst) return 0;
    int64_t b = part[dst + 1] - part[dst];
    int64_t nsl = 0;
    for (int64_t i0 = 0; i0 < b; i0 += S) ++nsl;
    return (int64_t)T[src] * nsl;
}
