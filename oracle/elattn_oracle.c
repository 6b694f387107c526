/*
 * elattn_oracle.c — CPU restatement of the reference EL-attention hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it.  The product library
 * (paper_2105_04779_b200/libelattn_gpu.so) never links or calls it.
 *
 * Parity is pinned two ways (see tests/test_oracle.py):
 *   - against golden vectors produced by the reference itself
 *     (tests/golden/make_golden.py drives oracle/_ref, which is compiled
 *     from /root/reference/proj/include by oracle/Makefile), and
 *   - against the reference's own known-answer tests (SplitMix64 seed 0,
 *     identity-parameter cases, EL == MHA sweeps) restated in pytest.
 *
 * Every function restates one reference function in plain C, fp64, in the
 * same loop / accumulation order so the results are bit-identical to the
 * reference's default (Precision::f64) mode:
 *   orc_rng_*                  tensor.hpp:133-150   (SplitMix64)
 *   orc_seeded_uniform         tensor.hpp:236-241
 *   orc_params_random          attention.hpp:53-80  (draw order Wq,Wk,Wv,Wo,bq,bk,bv,bo)
 *   mm / softmax               tensor.hpp:161-178, 213-234
 *   orc_build_el_query         attention.hpp:197-215
 *   orc_el_bias_terms          attention.hpp:221-231
 *   orc_el_attention           attention.hpp:239-257
 *   orc_el_attention_folded    attention.hpp:262-290
 *   orc_fold_el_queries        attention.hpp:293-304
 *   orc_multi_head_attention   attention.hpp:96-113
 *   orc_kv_append              attention.hpp:134-150 (KvCache::append)
 *   orc_mixed_self_attention   attention.hpp:309-365 (decoder-only: EL over the shared
 *                              prefix + MHA over the generated-token cache, joint softmax)
 *   orc_beam_candidates        beam_search candidate generation + order
 *                              (decoding.hpp:186-205; candidate_better :163-167)
 *   orc_el_layer_step          build_el_query x g + fold + el_attention_folded per
 *                              input (the batched cross-attention step the GPU
 *                              path computes; SURVEY.md §8 math contract)
 *
 * Status codes mirror include/elattn_gpu.h (ShapeError=1, ParamError=2,
 * StateError=3, NumericError=4; errors.hpp:8-31).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_SHAPE 1
#define ORC_PARAM 2
#define ORC_STATE 3
#define ORC_NUMERIC 4
#define ORC_OOM 6

typedef struct {
    int h, d_m, d_k;
    int include_key_bias, include_value_bias;
    const double *Wq, *Wk, *Wv; /* [h][d_m][d_k] */
    const double *Wo;           /* [h][d_k][d_m] */
    const double *bq, *bk, *bv; /* [h][d_k] */
    const double *bo;           /* [d_m] */
} orc_params;

/* ---- SplitMix64 (tensor.hpp:133-150) ---------------------------------- */
uint64_t orc_rng_next_u64(uint64_t* state) {
    *state += 0x9E3779B97F4A7C15ULL;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

double orc_rng_next_double(uint64_t* state) {
    return (double)(orc_rng_next_u64(state) >> 11) * 0x1.0p-53;
}

/* seeded_uniform (tensor.hpp:236-241): row-major fill, lo + (hi-lo)*u. */
int orc_seeded_uniform(uint64_t* state, int64_t count, double lo, double hi, double* out) {
    if (!(lo < hi)) return ORC_PARAM;
    for (int64_t i = 0; i < count; ++i) out[i] = lo + (hi - lo) * orc_rng_next_double(state);
    return ORC_OK;
}

/* AttentionParams::random (attention.hpp:53-80): per-head tensors drawn in
 * the order Wq[0..h), Wk[0..h), Wv[0..h), Wo[0..h), bq, bk, bv, bo. */
int orc_params_random(int h, int d_m, int d_k, uint64_t* state, double lo, double hi, double* Wq,
                      double* Wk, double* Wv, double* Wo, double* bq, double* bk, double* bv,
                      double* bo) {
    if (h < 1 || d_m < 1 || d_k < 1) return ORC_PARAM;
    const int64_t mk = (int64_t)d_m * d_k;
    int rc = ORC_OK;
    for (int i = 0; i < h && !rc; ++i) rc = orc_seeded_uniform(state, mk, lo, hi, Wq + i * mk);
    for (int i = 0; i < h && !rc; ++i) rc = orc_seeded_uniform(state, mk, lo, hi, Wk + i * mk);
    for (int i = 0; i < h && !rc; ++i) rc = orc_seeded_uniform(state, mk, lo, hi, Wv + i * mk);
    for (int i = 0; i < h && !rc; ++i) rc = orc_seeded_uniform(state, mk, lo, hi, Wo + i * mk);
    for (int i = 0; i < h && !rc; ++i) rc = orc_seeded_uniform(state, d_k, lo, hi, bq + (int64_t)i * d_k);
    for (int i = 0; i < h && !rc; ++i) rc = orc_seeded_uniform(state, d_k, lo, hi, bk + (int64_t)i * d_k);
    for (int i = 0; i < h && !rc; ++i) rc = orc_seeded_uniform(state, d_k, lo, hi, bv + (int64_t)i * d_k);
    if (!rc) rc = orc_seeded_uniform(state, d_m, lo, hi, bo);
    return rc;
}

/* ---- tensor primitives -------------------------------------------------- */

/* matmul (tensor.hpp:161-178): c[m x p] = a[m x k] . b[k x p], i-t-j loop,
 * zero-skip on a, strides let callers pass transposed views without the
 * reference's explicit transpose() copy (the arithmetic order is unchanged).
 * b(t, j) = b[t * bs_t + j * bs_j]. */
static int mm(const double* a, int64_t lda, const double* b, int64_t bs_t, int64_t bs_j,
              int64_t m, int64_t k, int64_t p, double* c, int64_t ldc) {
    for (int64_t i = 0; i < m; ++i) {
        double* ci = c + i * ldc;
        for (int64_t j = 0; j < p; ++j) ci[j] = 0.0;
        for (int64_t t = 0; t < k; ++t) {
            const double av = a[i * lda + t];
            if (av == 0.0) continue;
            const double* bt = b + t * bs_t;
            for (int64_t j = 0; j < p; ++j) ci[j] += av * bt[j * bs_j];
        }
    }
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < p; ++j)
            if (!isfinite(c[i * ldc + j])) return ORC_NUMERIC;
    return ORC_OK;
}

/* scaled_softmax_rows (tensor.hpp:213-234), in place on rows x n. */
static int softmax_rows(double* x, int64_t rows, int64_t n, int64_t d) {
    if (d < 1) return ORC_PARAM;
    if (n < 1) return ORC_SHAPE;
    for (int64_t i = 0; i < rows * n; ++i)
        if (!isfinite(x[i])) return ORC_NUMERIC;
    const double inv = 1.0 / sqrt((double)d);
    for (int64_t r = 0; r < rows; ++r) {
        double* p = x + r * n;
        double mx = p[0] * inv;
        for (int64_t j = 1; j < n; ++j) mx = fmax(mx, p[j] * inv);
        double sum = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            p[j] = exp(p[j] * inv - mx);
            sum += p[j];
        }
        for (int64_t j = 0; j < n; ++j) p[j] = p[j] / sum;
    }
    for (int64_t i = 0; i < rows * n; ++i)
        if (!isfinite(x[i])) return ORC_NUMERIC;
    return ORC_OK;
}

/* AttentionParams::validate (attention.hpp:24-50): shapes are implied by
 * the flat layout here, so only the scalar checks remain. */
static int validate(const orc_params* p) {
    if (p->h < 1 || p->d_m < 1 || p->d_k < 1) return ORC_PARAM;
    return ORC_OK;
}

#define TRY(x)                 \
    do {                       \
        rc = (x);              \
        if (rc) goto done;     \
    } while (0)
#define ALLOC(ptr, count)                                                    \
    do {                                                                     \
        ptr = (double*)calloc((size_t)((count) > 0 ? (count) : 1), sizeof(double)); \
        if (!ptr) {                                                          \
            rc = ORC_OOM;                                                    \
            goto done;                                                       \
        }                                                                    \
    } while (0)

/* ---- build_el_query (attention.hpp:197-215) ------------------------------
 * q [1 x d_m] -> elq [h x d_m], s [h] (zero when include_key_bias is off). */
int orc_build_el_query(const orc_params* p, const double* q, double* elq, double* s) {
    int rc = validate(p);
    if (rc) return rc;
    const int d_m = p->d_m, d_k = p->d_k;
    double *Qi = NULL;
    ALLOC(Qi, d_k);
    for (int i = 0; i < p->h; ++i) {
        const double* Wq = p->Wq + (int64_t)i * d_m * d_k;
        const double* Wk = p->Wk + (int64_t)i * d_m * d_k;
        TRY(mm(q, d_m, Wq, d_k, 1, 1, d_m, d_k, Qi, d_k));   /* q . Wq_i            */
        for (int c = 0; c < d_k; ++c) Qi[c] = Qi[c] + p->bq[(int64_t)i * d_k + c]; /* + bq_i */
        /* Qi . Wk_i^T : b(t=c, j) = Wk[j][c] */
        TRY(mm(Qi, d_k, Wk, 1, d_k, 1, d_k, d_m, elq + (int64_t)i * d_m, d_m));
        s[i] = 0.0;
        if (p->include_key_bias) {
            double acc = 0.0;
            for (int c = 0; c < d_k; ++c) acc += Qi[c] * p->bk[(int64_t)i * d_k + c];
            s[i] = acc;
        }
    }
done:
    free(Qi);
    return rc;
}

/* fold_el_queries (attention.hpp:293-304): g ElQuery -> [(g*h) x d_m] and
 * [(g*h)], row = b*h + i.  The per-query elq blocks are already [h x d_m]
 * contiguous, so folding is a concatenation. */
int orc_fold_el_queries(int g, int h, int d_m, const double* const* elqs, const double* const* ss,
                        double* q_out, double* s_out) {
    for (int b = 0; b < g; ++b) {
        memcpy(q_out + (int64_t)b * h * d_m, elqs[b], sizeof(double) * (size_t)h * d_m);
        memcpy(s_out + (int64_t)b * h, ss[b], sizeof(double) * (size_t)h);
    }
    return ORC_OK;
}

/* detail::el_bias_terms (attention.hpp:221-231): sum_i bv_i . Wo_i + bo. */
int orc_el_bias_terms(const orc_params* p, double* out) {
    int rc = ORC_OK;
    const int d_m = p->d_m, d_k = p->d_k;
    double* tmp = NULL;
    ALLOC(tmp, d_m);
    for (int j = 0; j < d_m; ++j) out[j] = 0.0;
    if (p->include_value_bias) {
        for (int i = 0; i < p->h; ++i) {
            TRY(mm(p->bv + (int64_t)i * d_k, d_k, p->Wo + (int64_t)i * d_k * d_m, d_m, 1, 1, d_k, d_m,
                   tmp, d_m));
            for (int j = 0; j < d_m; ++j) out[j] = out[j] + tmp[j];
        }
    }
    for (int j = 0; j < d_m; ++j) out[j] = out[j] + p->bo[j];
done:
    free(tmp);
    return rc;
}

/* el_attention_folded (attention.hpp:262-290).
 * queries [(g*h) x d_m], H [n x d_m], bias_scalars [g*h] -> out [g x d_m]. */
int orc_el_attention_folded(const orc_params* p, const double* queries, int64_t rows,
                            const double* H, int64_t n, const double* bias_scalars, double* out) {
    int rc = validate(p);
    if (rc) return rc;
    if (rows % p->h != 0) return ORC_SHAPE;
    if (n < 1) return ORC_STATE;
    const int d_m = p->d_m, d_k = p->d_k, h = p->h;
    const int64_t g = rows / h;
    double *scores = NULL, *ctx = NULL, *bias = NULL, *acc = NULL, *cv = NULL, *co = NULL;
    ALLOC(scores, rows * n);
    ALLOC(ctx, rows * d_m);
    ALLOC(bias, d_m);
    ALLOC(acc, d_m);
    ALLOC(cv, d_k);
    ALLOC(co, d_m);
    /* scores = queries . H^T : b(t, j) = H[j][t] (:272) */
    TRY(mm(queries, d_m, H, 1, d_m, rows, d_m, n, scores, n));
    for (int64_t r = 0; r < rows; ++r) { /* + s (:273-278) */
        const double s = bias_scalars ? bias_scalars[r] : 0.0;
        if (s != 0.0)
            for (int64_t j = 0; j < n; ++j) scores[r * n + j] = scores[r * n + j] + s;
    }
    TRY(softmax_rows(scores, rows, n, d_k));                 /* (:279) */
    TRY(mm(scores, n, H, d_m, 1, rows, n, d_m, ctx, d_m));   /* ctx = P . H (:280) */
    TRY(orc_el_bias_terms(p, bias));                         /* (:281) */
    for (int64_t b = 0; b < g; ++b) {                        /* (:283-288) */
        for (int j = 0; j < d_m; ++j) acc[j] = 0.0;
        for (int i = 0; i < h; ++i) {
            TRY(mm(ctx + (b * h + i) * d_m, d_m, p->Wv + (int64_t)i * d_m * d_k, d_k, 1, 1, d_m, d_k,
                   cv, d_k));
            TRY(mm(cv, d_k, p->Wo + (int64_t)i * d_k * d_m, d_m, 1, 1, d_k, d_m, co, d_m));
            for (int j = 0; j < d_m; ++j) acc[j] = acc[j] + co[j];
        }
        for (int j = 0; j < d_m; ++j) out[b * d_m + j] = acc[j] + bias[j];
    }
done:
    free(scores);
    free(ctx);
    free(bias);
    free(acc);
    free(cv);
    free(co);
    return rc;
}

/* el_attention (attention.hpp:239-257): one query row, per-head loop. */
int orc_el_attention(const orc_params* p, const double* q, const double* H, int64_t n, double* out) {
    int rc = validate(p);
    if (rc) return rc;
    if (n < 1) return ORC_STATE;
    const int d_m = p->d_m, d_k = p->d_k, h = p->h;
    double *elq = NULL, *s = NULL, *scores = NULL, *ctx = NULL, *cv = NULL, *co = NULL, *bias = NULL;
    ALLOC(elq, (int64_t)h * d_m);
    ALLOC(s, h);
    ALLOC(scores, n);
    ALLOC(ctx, d_m);
    ALLOC(cv, d_k);
    ALLOC(co, d_m);
    ALLOC(bias, d_m);
    TRY(orc_build_el_query(p, q, elq, s));
    for (int j = 0; j < d_m; ++j) out[j] = 0.0;
    for (int i = 0; i < h; ++i) {
        TRY(mm(elq + (int64_t)i * d_m, d_m, H, 1, d_m, 1, d_m, n, scores, n));
        if (s[i] != 0.0)
            for (int64_t t = 0; t < n; ++t) scores[t] = scores[t] + s[i];
        TRY(softmax_rows(scores, 1, n, d_k));
        TRY(mm(scores, n, H, d_m, 1, 1, n, d_m, ctx, d_m));
        TRY(mm(ctx, d_m, p->Wv + (int64_t)i * d_m * d_k, d_k, 1, 1, d_m, d_k, cv, d_k));
        TRY(mm(cv, d_k, p->Wo + (int64_t)i * d_k * d_m, d_m, 1, 1, d_k, d_m, co, d_m));
        for (int j = 0; j < d_m; ++j) out[j] = out[j] + co[j];
    }
    TRY(orc_el_bias_terms(p, bias));
    for (int j = 0; j < d_m; ++j) out[j] = out[j] + bias[j];
done:
    free(elq);
    free(s);
    free(scores);
    free(ctx);
    free(cv);
    free(co);
    free(bias);
    return rc;
}

/* multi_head_attention (attention.hpp:96-113): q [g x d_m], H [n x d_m]. */
int orc_multi_head_attention(const orc_params* p, const double* q, int64_t g, const double* H,
                             int64_t n, double* out) {
    int rc = validate(p);
    if (rc) return rc;
    if (n < 1) return ORC_STATE;
    const int d_m = p->d_m, d_k = p->d_k, h = p->h;
    double *Qi = NULL, *Ki = NULL, *Vi = NULL, *sc = NULL, *cx = NULL, *o = NULL;
    ALLOC(Qi, g * d_k);
    ALLOC(Ki, n * d_k);
    ALLOC(Vi, n * d_k);
    ALLOC(sc, g * n);
    ALLOC(cx, g * d_k);
    ALLOC(o, g * d_m);
    for (int64_t j = 0; j < g * d_m; ++j) out[j] = 0.0;
    for (int i = 0; i < h; ++i) {
        const int64_t wo = (int64_t)i * d_m * d_k;
        TRY(mm(q, d_m, p->Wq + wo, d_k, 1, g, d_m, d_k, Qi, d_k));
        for (int64_t r = 0; r < g; ++r)
            for (int c = 0; c < d_k; ++c) Qi[r * d_k + c] = Qi[r * d_k + c] + p->bq[(int64_t)i * d_k + c];
        TRY(mm(H, d_m, p->Wk + wo, d_k, 1, n, d_m, d_k, Ki, d_k));
        if (p->include_key_bias)
            for (int64_t r = 0; r < n; ++r)
                for (int c = 0; c < d_k; ++c) Ki[r * d_k + c] = Ki[r * d_k + c] + p->bk[(int64_t)i * d_k + c];
        TRY(mm(H, d_m, p->Wv + wo, d_k, 1, n, d_m, d_k, Vi, d_k));
        if (p->include_value_bias)
            for (int64_t r = 0; r < n; ++r)
                for (int c = 0; c < d_k; ++c) Vi[r * d_k + c] = Vi[r * d_k + c] + p->bv[(int64_t)i * d_k + c];
        TRY(mm(Qi, d_k, Ki, 1, d_k, g, d_k, n, sc, n)); /* Qi . Ki^T */
        TRY(softmax_rows(sc, g, n, d_k));
        TRY(mm(sc, n, Vi, d_k, 1, g, n, d_k, cx, d_k));
        TRY(mm(cx, d_k, p->Wo + (int64_t)i * d_k * d_m, d_m, 1, g, d_k, d_m, o, d_m));
        for (int64_t j = 0; j < g * d_m; ++j) out[j] = out[j] + o[j];
    }
    for (int64_t r = 0; r < g; ++r)
        for (int j = 0; j < d_m; ++j) out[r * d_m + j] = out[r * d_m + j] + p->bo[j];
done:
    free(Qi);
    free(Ki);
    free(Vi);
    free(sc);
    free(cx);
    free(o);
    return rc;
}

/* The batched cross-attention step the GPU path computes:
 * for each input b (own H_b [n_b x d_m], rows padded to n_stride) and its x
 * beam queries Y[b*x + k], build_el_query per beam, fold, el_attention_folded.
 * out [B*x x d_m], row b*x + k.  n_per_input may be NULL (all = n_stride).
 * inputs [b0, b1) only, so callers can sample or thread over inputs. */
int orc_el_layer_step(const orc_params* p, const double* Y, const double* H, const int* n_per_input,
                      int B, int x, int64_t n_stride, int b0, int b1, double* out) {
    int rc = validate(p);
    if (rc) return rc;
    const int d_m = p->d_m, h = p->h;
    double *q = NULL, *s = NULL;
    ALLOC(q, (int64_t)x * h * d_m);
    ALLOC(s, (int64_t)x * h);
    (void)B;
    for (int b = b0; b < b1; ++b) {
        const int64_t n = n_per_input ? n_per_input[b] : n_stride;
        for (int k = 0; k < x; ++k)
            TRY(orc_build_el_query(p, Y + ((int64_t)b * x + k) * d_m, q + (int64_t)k * h * d_m,
                                   s + (int64_t)k * h));
        TRY(orc_el_attention_folded(p, q, (int64_t)x * h, H + (int64_t)b * n_stride * d_m, n, s,
                                    out + (int64_t)b * x * d_m));
    }
done:
    free(q);
    free(s);
    return rc;
}


/* KvCache::append (attention.hpp:134-150): project one hidden row through every head's
 * key/value weights (+ biases when enabled) and store it at position t of caches
 * K, V laid out [h][t_max][d_k]. */
int orc_kv_append(const orc_params* p, const double* y, double* K, double* V, int64_t t_max, int64_t t) {
    int rc = validate(p);
    if (rc) return rc;
    if (t < 0 || t >= t_max) return ORC_STATE;
    const int d_m = p->d_m, d_k = p->d_k, h = p->h;
    double *k = NULL, *v = NULL;
    ALLOC(k, d_k);
    ALLOC(v, d_k);
    for (int i = 0; i < h; ++i) {
        const int64_t wo = (int64_t)i * d_m * d_k;
        TRY(mm(y, d_m, p->Wk + wo, d_k, 1, 1, d_m, d_k, k, d_k));
        if (p->include_key_bias)
            for (int c = 0; c < d_k; ++c) k[c] = k[c] + p->bk[(int64_t)i * d_k + c];
        TRY(mm(y, d_m, p->Wv + wo, d_k, 1, 1, d_m, d_k, v, d_k));
        if (p->include_value_bias)
            for (int c = 0; c < d_k; ++c) v[c] = v[c] + p->bv[(int64_t)i * d_k + c];
        for (int c = 0; c < d_k; ++c) {
            K[((int64_t)i * t_max + t) * d_k + c] = k[c];
            V[((int64_t)i * t_max + t) * d_k + c] = v[c];
        }
    }
done:
    free(k);
    free(v);
    return rc;
}

/* mixed_self_attention (attention.hpp:309-365): q [1 x d_m], prefix Hp [t_in x d_m],
 * generated-token cache K, V [h][t_max][d_k] with t_out valid rows -> out [1 x d_m].
 * Per head: EL scores over the prefix (+ s_i) and Q_i . K_r over the cache, one joint
 * softmax; the prefix part goes through Wv_i Wo_i with the value bias scaled by the
 * prefix probability mass, the cached part (values already biased) through Wo_i. */
int orc_mixed_self_attention(const orc_params* p, const double* q, const double* Hp, int64_t t_in,
                             const double* K, const double* V, int64_t t_max, int64_t t_out, double* out) {
    int rc = validate(p);
    if (rc) return rc;
    if (t_in < 1) return ORC_STATE;
    const int d_m = p->d_m, d_k = p->d_k, h = p->h;
    const int64_t n = t_in + t_out;
    double *elq = NULL, *s = NULL, *Qi = NULL, *scores = NULL, *ctx = NULL, *cv = NULL, *head = NULL,
           *tmp = NULL, *b = NULL, *co = NULL;
    ALLOC(elq, (int64_t)h * d_m);
    ALLOC(s, h);
    ALLOC(Qi, d_k);
    ALLOC(scores, n);
    ALLOC(ctx, d_m);
    ALLOC(cv, d_k);
    ALLOC(head, d_m);
    ALLOC(tmp, d_m);
    ALLOC(b, d_k);
    ALLOC(co, d_k);
    TRY(orc_build_el_query(p, q, elq, s));
    for (int j = 0; j < d_m; ++j) out[j] = 0.0;
    for (int i = 0; i < h; ++i) {
        const int64_t wo = (int64_t)i * d_m * d_k;
        TRY(mm(q, d_m, p->Wq + wo, d_k, 1, 1, d_m, d_k, Qi, d_k)); /* Qi = q Wq_i + bq_i */
        for (int c = 0; c < d_k; ++c) Qi[c] = Qi[c] + p->bq[(int64_t)i * d_k + c];
        TRY(mm(elq + (int64_t)i * d_m, d_m, Hp, 1, d_m, 1, d_m, t_in, scores, t_in)); /* prefix scores */
        for (int64_t j = 0; j < t_in; ++j) scores[j] = scores[j] + s[i];
        for (int64_t r = 0; r < t_out; ++r) { /* generated-token scores */
            double sc = 0.0;
            for (int c = 0; c < d_k; ++c) sc += Qi[c] * K[((int64_t)i * t_max + r) * d_k + c];
            scores[t_in + r] = sc;
        }
        TRY(softmax_rows(scores, 1, n, d_k));
        double mass = 0.0;
        for (int64_t j = 0; j < t_in; ++j) mass += scores[j];
        TRY(mm(scores, t_in, Hp, d_m, 1, 1, t_in, d_m, ctx, d_m)); /* probs_in . Hp */
        TRY(mm(ctx, d_m, p->Wv + wo, d_k, 1, 1, d_m, d_k, cv, d_k));
        TRY(mm(cv, d_k, p->Wo + (int64_t)i * d_k * d_m, d_m, 1, 1, d_k, d_m, head, d_m));
        if (p->include_value_bias) {
            for (int c = 0; c < d_k; ++c) b[c] = p->bv[(int64_t)i * d_k + c] * mass;
            TRY(mm(b, d_k, p->Wo + (int64_t)i * d_k * d_m, d_m, 1, 1, d_k, d_m, tmp, d_m));
            for (int j = 0; j < d_m; ++j) head[j] = head[j] + tmp[j];
        }
        if (t_out > 0) {
            for (int c = 0; c < d_k; ++c) co[c] = 0.0;
            for (int64_t r = 0; r < t_out; ++r)
                for (int c = 0; c < d_k; ++c) co[c] += scores[t_in + r] * V[((int64_t)i * t_max + r) * d_k + c];
            TRY(mm(co, d_k, p->Wo + (int64_t)i * d_k * d_m, d_m, 1, 1, d_k, d_m, tmp, d_m));
            for (int j = 0; j < d_m; ++j) head[j] = head[j] + tmp[j];
        }
        for (int j = 0; j < d_m; ++j) out[j] = out[j] + head[j];
    }
    for (int j = 0; j < d_m; ++j) out[j] = out[j] + p->bo[j];
done:
    free(elq);
    free(s);
    free(Qi);
    free(scores);
    free(ctx);
    free(cv);
    free(head);
    free(tmp);
    free(b);
    free(co);
    return rc;
}


/* ------------------------------------------------------------ beam-search candidates */
typedef struct {
    int parent, token;
    double lp_sum;
} orc_cand;

/* candidate_better (decoding.hpp:163-167) as a qsort order */
static int cand_cmp(const void* pa, const void* pb) {
    const orc_cand* a = (const orc_cand*)pa;
    const orc_cand* b = (const orc_cand*)pb;
    if (a->lp_sum != b->lp_sum) return a->lp_sum > b->lp_sum ? -1 : 1;
    if (a->token != b->token) return a->token < b->token ? -1 : 1;
    return (a->parent > b->parent) - (a->parent < b->parent);
}

/* decoding.hpp:192-205: for parents i < roots, every finite lprobs[i][tok] gives
 * (i, tok, live_lp[i] + v); sorted by candidate_better; the first k written (parent -1
 * beyond the candidate count).  One input; lprobs [lanes][V].  penalty (may be NULL):
 * [V], subtracted from v after the finiteness test (diverse_beam_search,
 * decoding.hpp:312-316: v -= strength * step_token_counts[tok]). */
int orc_beam_candidates(const double* lprobs, const double* live_lp, const double* penalty, int lanes, int roots,
                        int V, int k, int* parent, int* token, double* lp_sum) {
    if (roots < 1 || roots > lanes || V < 1 || k < 1) return ORC_SHAPE;
    orc_cand* c = (orc_cand*)malloc(sizeof(orc_cand) * (size_t)roots * (size_t)V);
    if (!c) return ORC_PARAM;
    size_t n = 0;
    for (int i = 0; i < roots; ++i)
        for (int t = 0; t < V; ++t) {
            double v = lprobs[(size_t)i * V + t];
            if (!isfinite(v)) continue;
            if (penalty) v -= penalty[t];
            c[n].parent = i, c[n].token = t, c[n].lp_sum = live_lp[i] + v;
            ++n;
        }
    qsort(c, n, sizeof(orc_cand), cand_cmp);
    for (int r = 0; r < k; ++r) {
        if ((size_t)r < n) {
            parent[r] = c[r].parent, token[r] = c[r].token, lp_sum[r] = c[r].lp_sum;
        } else {
            parent[r] = -1, token[r] = -1, lp_sum[r] = -INFINITY;
        }
    }
    free(c);
    return 0;
}
