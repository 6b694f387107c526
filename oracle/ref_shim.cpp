// ref_shim.cpp — C-ABI shim over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY (oracle).  Compiled by oracle/Makefile straight
// from /root/reference/proj/include (read-only, never copied) into
// oracle/_ref/libelattn_ref.so.  Used to (1) pin oracle/elattn_oracle.c
// and generate tests/golden fixtures, and (2) time the reference's own CPU
// path for bench.py's cpu_baseline / --impl reference leg.
//
// Every entry point calls the reference functions themselves:
//   AttentionParams            attention.hpp:13-81
//   build_el_query             attention.hpp:197-215
//   fold_el_queries            attention.hpp:293-304
//   el_attention               attention.hpp:239-257
//   el_attention_folded        attention.hpp:262-290
//   multi_head_attention       attention.hpp:96-113
//   KvCache::append            attention.hpp:134-150
//   mixed_self_attention       attention.hpp:309-365
//   Rng / seeded_uniform       tensor.hpp:133-150, 236-241
//   PrecisionGuard             tensor.hpp:25-29
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "elattn/attention.hpp"
#include "elattn/decoding.hpp"

using namespace elattn;

namespace {

thread_local std::string g_err;

int status_of(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const ShapeError*>(&e)) return 1;
    if (dynamic_cast<const ParamError*>(&e)) return 2;
    if (dynamic_cast<const StateError*>(&e)) return 3;
    if (dynamic_cast<const NumericError*>(&e)) return 4;
    return 9;
}

Tensor from_flat(std::vector<int64_t> shape, const double* p) {
    Tensor t(std::move(shape));
    std::memcpy(t.data().data(), p, sizeof(double) * static_cast<size_t>(t.size()));
    return t;
}

void to_flat(const Tensor& t, double* p) {
    std::memcpy(p, t.data().data(), sizeof(double) * static_cast<size_t>(t.size()));
}

AttentionParams make_params(int h, int d_m, int d_k, int kb, int vb, const double* Wq,
                            const double* Wk, const double* Wv, const double* Wo, const double* bq,
                            const double* bk, const double* bv, const double* bo) {
    AttentionParams p;
    p.h = h;
    p.d_m = d_m;
    p.d_k = d_k;
    const int64_t mk = int64_t(d_m) * d_k;
    for (int i = 0; i < h; ++i) {
        p.Wq.push_back(from_flat({d_m, d_k}, Wq + i * mk));
        p.Wk.push_back(from_flat({d_m, d_k}, Wk + i * mk));
        p.Wv.push_back(from_flat({d_m, d_k}, Wv + i * mk));
        p.Wo.push_back(from_flat({d_k, d_m}, Wo + i * mk));
        p.bq.push_back(from_flat({d_k}, bq + int64_t(i) * d_k));
        p.bk.push_back(from_flat({d_k}, bk + int64_t(i) * d_k));
        p.bv.push_back(from_flat({d_k}, bv + int64_t(i) * d_k));
    }
    p.bo = from_flat({d_m}, bo);
    p.include_key_bias = kb != 0;
    p.include_value_bias = vb != 0;
    return p;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_rng_first(uint64_t seed, int k) {
    Rng r(seed);
    uint64_t v = 0;
    for (int i = 0; i <= k; ++i) v = r.next_u64();
    return v;
}

// AttentionParams::random with the reference RNG; outputs flat per-head arrays.
int ref_params_random(int h, int d_m, int d_k, uint64_t seed, double* Wq, double* Wk, double* Wv,
                      double* Wo, double* bq, double* bk, double* bv, double* bo) {
    try {
        Rng rng(seed);
        AttentionParams p = AttentionParams::random(h, d_m, d_k, rng);
        const int64_t mk = int64_t(d_m) * d_k;
        for (int i = 0; i < h; ++i) {
            to_flat(p.Wq[i], Wq + i * mk);
            to_flat(p.Wk[i], Wk + i * mk);
            to_flat(p.Wv[i], Wv + i * mk);
            to_flat(p.Wo[i], Wo + i * mk);
            to_flat(p.bq[i], bq + int64_t(i) * d_k);
            to_flat(p.bk[i], bk + int64_t(i) * d_k);
            to_flat(p.bv[i], bv + int64_t(i) * d_k);
        }
        to_flat(p.bo, bo);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

#define REF_PARAMS_ARGS                                                                   \
    int h, int d_m, int d_k, int kb, int vb, const double *Wq, const double *Wk,           \
        const double *Wv, const double *Wo, const double *bq, const double *bk, const double *bv, \
        const double *bo
#define REF_PARAMS make_params(h, d_m, d_k, kb, vb, Wq, Wk, Wv, Wo, bq, bk, bv, bo)

int ref_build_el_query(REF_PARAMS_ARGS, const double* q, double* elq, double* s) {
    try {
        ElQuery eq = build_el_query(from_flat({1, d_m}, q), REF_PARAMS);
        to_flat(eq.elq, elq);
        for (int i = 0; i < h; ++i) s[i] = eq.s[size_t(i)];
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_el_attention(REF_PARAMS_ARGS, const double* q, const double* H, int64_t n, double* out) {
    try {
        Tensor Ht = n > 0 ? from_flat({n, d_m}, H) : Tensor();
        to_flat(el_attention(from_flat({1, d_m}, q), Ht, REF_PARAMS), out);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_el_attention_folded(REF_PARAMS_ARGS, const double* queries, int64_t rows, const double* H,
                            int64_t n, const double* s, double* out) {
    try {
        Tensor Ht = n > 0 ? from_flat({n, d_m}, H) : Tensor();
        to_flat(el_attention_folded(from_flat({rows, d_m}, queries), Ht, from_flat({rows}, s),
                                    REF_PARAMS),
                out);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_multi_head_attention(REF_PARAMS_ARGS, const double* q, int64_t g, const double* H,
                             int64_t n, double* out) {
    try {
        Tensor Ht = n > 0 ? from_flat({n, d_m}, H) : Tensor();
        to_flat(multi_head_attention(from_flat({g, d_m}, q), Ht, REF_PARAMS), out);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// ---- batched layer step (the CPU baseline) --------------------------------
// Params are converted to reference Tensors once; each worker thread runs the
// reference call chain build_el_query x beams -> fold_el_queries ->
// el_attention_folded over its own contiguous block of inputs.  The
// reference functions are pure, so threads share params.
struct RefLayer {
    AttentionParams p;
};

void* ref_layer_create(REF_PARAMS_ARGS) {
    try {
        return new RefLayer{REF_PARAMS};
    } catch (const std::exception& e) {
        status_of(e);
        return nullptr;
    }
}

void ref_layer_destroy(void* layer) { delete static_cast<RefLayer*>(layer); }

int ref_layer_step(void* layer, const double* Y, const double* H, const int* n_per_input, int B,
                   int x, int64_t n_stride, int b0, int b1, double* out, int nthreads, int f32) {
    auto* L = static_cast<RefLayer*>(layer);
    const int d_m = L->p.d_m, h = L->p.h;
    (void)B;
    PrecisionGuard guard(f32 ? Precision::f32 : Precision::f64);  // set before threads start
    std::vector<int> rc(size_t(nthreads > 0 ? nthreads : 1), 0);
    std::vector<std::string> msg(rc.size());
    auto work = [&](int tid, int lo, int hi) {
        try {
            for (int b = lo; b < hi; ++b) {
                const int64_t n = n_per_input ? n_per_input[b] : n_stride;
                std::vector<ElQuery> eqs;
                for (int k = 0; k < x; ++k)
                    eqs.push_back(build_el_query(from_flat({1, d_m}, Y + (int64_t(b) * x + k) * d_m), L->p));
                auto [fq, fs] = fold_el_queries(eqs, h, d_m);
                Tensor o = el_attention_folded(fq, from_flat({n, d_m}, H + int64_t(b) * n_stride * d_m),
                                               fs, L->p);
                to_flat(o, out + int64_t(b) * x * d_m);
            }
        } catch (const std::exception& e) {
            rc[size_t(tid)] = status_of(e);
            msg[size_t(tid)] = e.what();
        }
    };
    const int T = int(rc.size());
    const int total = b1 - b0;
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) {
        const int lo = b0 + int(int64_t(total) * t / T), hi = b0 + int(int64_t(total) * (t + 1) / T);
        if (T == 1)
            work(t, lo, hi);
        else
            th.emplace_back(work, t, lo, hi);
    }
    for (auto& t : th) t.join();
    for (size_t t = 0; t < rc.size(); ++t)
        if (rc[t]) {
            g_err = msg[t];
            return rc[t];
        }
    return 0;
}

// KvCache built by the reference's own append from t hidden rows; K, V exported as
// [h][t_max][d_k] (rows t..t_max-1 untouched).
int ref_kv_build(REF_PARAMS_ARGS, const double* rows, int64_t t, int64_t t_max, double* K, double* V) {
    try {
        AttentionParams p = REF_PARAMS;
        KvCache c(h, d_k);
        for (int64_t r = 0; r < t; ++r) c.append(from_flat({1, d_m}, rows + r * d_m), p);
        for (int i = 0; i < h; ++i)
            for (int64_t r = 0; r < t; ++r)
                for (int j = 0; j < d_k; ++j) {
                    K[(int64_t(i) * t_max + r) * d_k + j] = c.K[size_t(i)][size_t(r * d_k + j)];
                    V[(int64_t(i) * t_max + r) * d_k + j] = c.V[size_t(i)][size_t(r * d_k + j)];
                }
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// mixed_self_attention with the generated-token cache built from t_out hidden rows by
// the reference's KvCache::append.
int ref_mixed_self_attention(REF_PARAMS_ARGS, const double* q, const double* Hp, int64_t t_in,
                             const double* gen_rows, int64_t t_out, double* out) {
    try {
        AttentionParams p = REF_PARAMS;
        KvCache c(h, d_k);
        for (int64_t r = 0; r < t_out; ++r) c.append(from_flat({1, d_m}, gen_rows + r * d_m), p);
        Tensor o = mixed_self_attention(from_flat({1, d_m}, q), from_flat({t_in, d_m}, Hp), c, p);
        to_flat(o, out);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// The reference's own candidate record and order (decoding.hpp:157-167) over one input's
// candidates (decoding.hpp:192-204; with penalty, diverse_beam_search's :312-316), first k
// written.
int ref_beam_candidates(const double* lprobs, const double* live_lp, const double* penalty, int lanes, int roots,
                        int V, int k, int* parent, int* token, double* lp_sum) {
    (void)lanes;
    try {
        std::vector<elattn::detail::Candidate> cands;
        for (int i = 0; i < roots; ++i)
            for (int tok = 0; tok < V; ++tok) {
                double v = lprobs[int64_t(i) * V + tok];
                if (!std::isfinite(v)) continue;
                if (penalty) v -= penalty[tok];
                cands.push_back({i, tok, live_lp[i] + v});
            }
        std::sort(cands.begin(), cands.end(), elattn::detail::candidate_better);
        for (int r = 0; r < k; ++r) {
            const bool have = size_t(r) < cands.size();
            parent[r] = have ? cands[size_t(r)].parent : -1;
            token[r] = have ? cands[size_t(r)].token : -1;
            lp_sum[r] = have ? cands[size_t(r)].lp_sum : -std::numeric_limits<double>::infinity();
        }
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

}  // extern "C"
