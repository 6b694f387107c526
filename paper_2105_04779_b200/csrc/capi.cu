// capi.cu — the extern "C" boundary (include/elattn_gpu.h).
//
// Host-side orchestration of the three hot-path stages, each stream-ordered:
//   (1) query expansion  (build_el_query, attention.hpp:197-215)
//   (2) fused decode     (el_attention_folded core, attention.hpp:272-280)
//   (3) output proj.     (el_attention_folded tail + el_bias_terms, :281-288, :221-231)
// No CPU compute path exists: every arithmetic step is a device kernel.
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

struct elattn_gpu_params_s {
    int h = 0, d_m = 0, d_k = 0, dtype = 0;
    int include_key_bias = 1, include_value_bias = 1;
    // Device buffers, element type `dtype` unless noted.
    void* WqT = nullptr;  // [h*d_k][d_m]
    void* WkT = nullptr;  // [h][d_k][d_m]: K-major B operand of the K/V-cache append
    void* Wk = nullptr;   // [h][d_m][d_k]
    void* WvT = nullptr;  // [h][d_k][d_m]
    void* WoT = nullptr;  // [d_m][h*d_k]
    float* bq = nullptr;  // [h*d_k]
    float* bk = nullptr;  // [h*d_k]
    float* bv = nullptr;  // [h*d_k] (zero when include_value_bias == 0)
    float* bo = nullptr;  // [d_m]
    // fp32 path on the tensor cores (3xTF32, tf32_gemm.cu): tf32 hi / lo parts of the
    // weights, split once here [0] = hi, [1] = lo; same layouts as above
    float* WqT_s[2] = {nullptr, nullptr};
    float* Wk_s[2] = {nullptr, nullptr};
    float* WvT_s[2] = {nullptr, nullptr};
    float* WoT_s[2] = {nullptr, nullptr};
};

namespace elattn_gpu {

namespace {
thread_local std::string g_last_error;
thread_local int64_t g_launches = 0;
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }

int g_pdl = -1;
bool pdl_enabled() {
    if (g_pdl < 0) {
        const char* e = getenv("ELATTN_PDL");
        g_pdl = (e && std::string(e) == "0") ? 0 : 1;
    }
    return g_pdl != 0;
}
void count_launch(int n) { g_launches += n; }

namespace {

template <typename F>
int guarded(F&& f) {
    try {
        f();
        g_last_error.clear();
        return ELATTN_OK;
    } catch (const Status& s) {
        g_last_error = s.msg;
        return s.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return ELATTN_ERR_OOM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return ELATTN_ERR_CUDA;
    }
}

uint16_t f32_to_bf16_rne(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return uint16_t((u >> 16) | 0x40);  // NaN stays NaN
    u += 0x7fffu + ((u >> 16) & 1u);
    return uint16_t(u >> 16);
}

// Upload an fp64 host array as `dtype` (fp32 or bf16, RNE).
void* upload(const std::vector<double>& v, int dtype) {
    void* d = nullptr;
    const size_t n = v.size();
    if (dtype == ELATTN_DTYPE_BF16) {
        std::vector<uint16_t> h(n);
        for (size_t i = 0; i < n; ++i) h[i] = f32_to_bf16_rne(float(v[i]));
        ELA_CHECK_CUDA(cudaMalloc(&d, n * 2));
        ELA_CHECK_CUDA(cudaMemcpy(d, h.data(), n * 2, cudaMemcpyHostToDevice));
    } else {
        std::vector<float> h(n);
        for (size_t i = 0; i < n; ++i) h[i] = float(v[i]);
        ELA_CHECK_CUDA(cudaMalloc(&d, n * 4));
        ELA_CHECK_CUDA(cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice));
    }
    return d;
}

float* upload_f32(const std::vector<double>& v) {
    return static_cast<float*>(upload(v, ELATTN_DTYPE_F32));
}

void free_params(elattn_gpu_params_s* p) {
    if (!p) return;
    for (void* ptr : {p->WqT, p->WkT, p->Wk, p->WvT, p->WoT, (void*)p->bq, (void*)p->bk, (void*)p->bv,
                      (void*)p->bo})
        if (ptr) cudaFree(ptr);
    for (int s = 0; s < 2; ++s)
        for (float* ptr : {p->WqT_s[s], p->Wk_s[s], p->WvT_s[s], p->WoT_s[s]})
            if (ptr) cudaFree(ptr);
    delete p;
}

// tf32 rounding of the host side (cvt.rna.tf32.f32: nearest, ties away from zero)
float tf32_rna_host(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
}

// fp32 weights as (hi, lo) device arrays
void upload_split(const std::vector<double>& v, float* (&dst)[2]) {
    std::vector<double> hi(v.size()), lo(v.size());
    for (size_t i = 0; i < v.size(); ++i) {
        const float f = float(v[i]), h = tf32_rna_host(f);
        hi[i] = h;
        lo[i] = f - h;
    }
    dst[0] = upload_f32(hi);
    dst[1] = upload_f32(lo);
}

// Stream-ordered scratch: caller-provided or cudaMallocAsync'd for this call.
class Scratch {
   public:
    Scratch(void* ws, size_t ws_bytes, size_t need, cudaStream_t st) : st_(st), cap_(need) {
        if (need == 0) return;
        if (ws) {
            ELA_REQUIRE(ws_bytes >= need, ELATTN_ERR_PARAM,
                        "workspace too small: need " + std::to_string(need) + " bytes");
            base_ = static_cast<char*>(ws);
        } else {
            ELA_CHECK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&base_), need, st));
            owned_ = true;
        }
    }
    ~Scratch() {
        if (owned_) cudaFreeAsync(base_, st_);
    }
    void* take(size_t bytes) {
        ELA_REQUIRE(base_ != nullptr || bytes == 0, ELATTN_ERR_PARAM, "workspace: no scratch reserved");
        void* p = base_ + off_;
        off_ += (bytes + 255) & ~size_t(255);
        ELA_REQUIRE(off_ <= cap_, ELATTN_ERR_PARAM, "workspace: scratch layout exceeds its reservation");
        return p;
    }
    size_t mark() const { return off_; }
    void reset(size_t m) { off_ = m; }

   private:
    char* base_ = nullptr;
    size_t off_ = 0;
    bool owned_ = false;
    cudaStream_t st_;
    size_t cap_ = 0;
};

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// Partial records of inputs the tcgen05 decode splits across clusters (bf16 path).
size_t decode_scratch(const elattn_gpu_params_s* p) {
    return p->dtype == ELATTN_DTYPE_BF16 ? align256(el_decode_tc_scratch_bytes(p->d_m)) : 0;
}

// Scratch layout of a full step: Q [R][h*d_k], q' [R*h][d_m], C [R*h][d_m], V [R][h*d_k],
// decode records.
size_t step_workspace(const elattn_gpu_params_s* p, int64_t R) {
    const size_t e = dtype_bytes(p->dtype);
    const size_t hk = size_t(p->h) * p->d_k, hm = size_t(p->h) * p->d_m;
    return align256(R * hk * e) * 2 + align256(R * hm * e) * 2 + decode_scratch(p);
}

// Every bf16 projection runs on the tcgen05 GEMM family (tc_gemm.cu); shapes outside its
// envelope (K not a multiple of 64, unaligned rows) and the fp32 path use the SIMT kernel.
void gemm(const elattn_gpu_params_s* p, const GemmArgs& g_in, cudaStream_t st) {
    GemmArgs g = g_in;
    g.b_static = 1;  // every B here is a packed weight of the params handle (written once, at create)
    if (p->dtype == ELATTN_DTYPE_BF16 && tc_gemm_supported(g))
        launch_tc_gemm(g, st);
    else
        launch_simt_gemm(p->dtype, g, st);
}

// (1a) Q = Y.W_Q + b_Q ; (1b) q'_{r,i} = Q_{r,i}.W_K,i^T   (attention.hpp:205-206)
// need_Q: the caller reads Q afterwards (key-bias scalars, mixed self-attention); otherwise a
// small batch takes the fused one-launch expansion (Q stays on chip)
void query_expansion(const elattn_gpu_params_s* p, const void* Y, int64_t R, void* Q, void* qp,
                     cudaStream_t st, bool need_Q = true) {
    const int h = p->h, d_m = p->d_m, d_k = p->d_k, hk = h * d_k;
    if (!need_Q && p->dtype == ELATTN_DTYPE_BF16 && R < (int64_t(1) << 30) &&
        tc_qexp_fused(Y, int(R), p->WqT, p->bq, p->Wk, qp, h, d_m, d_k, st))
        return;
    GemmArgs a{};
    a.A = Y, a.lda = d_m, a.B = p->WqT, a.ldb = d_m, a.C = Q, a.ldc = hk, a.bias = p->bq;
    a.M = int(R), a.N = hk, a.K = d_m, a.Z = 1, a.alpha = 1.f;
    gemm(p, a, st);
    const size_t e = dtype_bytes(p->dtype);
    GemmArgs b{};
    b.A = Q, b.lda = hk, b.sAz = d_k;                         // head i: columns i*d_k..
    b.B = p->Wk, b.ldb = d_k, b.sBz = int64_t(d_m) * d_k;     // W_K,i [d_m][d_k] is K-major
    b.C = qp, b.ldc = int64_t(h) * d_m, b.sCz = d_m;          // row r*h + i
    b.c_keep = 1;  // q' is read back by the decode while H streams through L2
    b.M = int(R), b.N = d_m, b.K = d_k, b.Z = h, b.alpha = 1.f;
    (void)e;
    gemm(p, b, st);
}

// (3a) V_{r,i} = C_{r*h+i}.W_V,i + b_V,i ; (3b) out = V.W_O + b_O   (attention.hpp:283-288)
void v_projection(const elattn_gpu_params_s* p, const void* C, int64_t R, void* V, cudaStream_t st) {
    const int h = p->h, d_m = p->d_m, d_k = p->d_k, hk = h * d_k;
    GemmArgs a{};
    a.A = C, a.lda = int64_t(h) * d_m, a.sAz = d_m;
    a.B = p->WvT, a.ldb = d_m, a.sBz = int64_t(d_k) * d_m;
    a.C = V, a.ldc = hk, a.sCz = d_k;
    a.bias = p->bv, a.sbz = d_k;
    a.M = int(R), a.N = d_k, a.K = d_m, a.Z = h, a.alpha = 1.f;
    gemm(p, a, st);
}

void o_projection(const elattn_gpu_params_s* p, const void* V, int64_t R, void* out, cudaStream_t st) {
    const int d_m = p->d_m, hk = p->h * p->d_k;
    GemmArgs b{};
    b.A = V, b.lda = hk, b.B = p->WoT, b.ldb = hk, b.C = out, b.ldc = d_m, b.bias = p->bo;
    b.M = int(R), b.N = d_m, b.K = hk, b.Z = 1, b.alpha = 1.f;
    gemm(p, b, st);
}

void output_projection(const elattn_gpu_params_s* p, const void* C, int64_t R, void* V, void* out,
                       cudaStream_t st) {
    v_projection(p, C, R, V, st);
    o_projection(p, V, R, out, st);
}

// ---------------------------------------------------------------- fp32 path on tensor cores
// 3xTF32 (tf32_gemm.cu): every stage of a layer step as a tcgen05 kind::tf32 GEMM at fp32
// accuracy; the decode as S = q'.H^T (per input), softmax, C = P.H (with a transposed hi/lo
// copy of H).  Envelope: d_m, d_k, h*d_k multiples of 32, 16-byte aligned buffers.
bool al16p(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; }

bool use_tf32_path(const elattn_gpu_params_s* p) {
    return p->dtype == ELATTN_DTYPE_F32 && p->WqT_s[0] != nullptr && p->d_m % 32 == 0 && p->d_k % 32 == 0 &&
           (p->h * p->d_k) % 32 == 0;
}

int64_t pad32(int64_t n) { return (n + 31) / 32 * 32; }

// hi / lo views of one fp32 operand in the workspace
struct Split {
    float* hi = nullptr;
    float* lo = nullptr;
};
Split take_split(Scratch& s, size_t count) {
    Split r;
    r.hi = static_cast<float*>(s.take(count * 4));
    r.lo = static_cast<float*>(s.take(count * 4));
    return r;
}
size_t split_bytes(size_t count) { return 2 * align256(count * 4); }

// H split once per call (or per decoder step): H_s [B][n][d_m], HT_s [B][d_m][n_pad]
size_t tf32_h_bytes(const elattn_gpu_params_s* p, int B, int n) {
    return split_bytes(size_t(B) * n * p->d_m) + split_bytes(size_t(B) * p->d_m * pad32(n));
}
// per-layer intermediates for R = B * x query rows
size_t tf32_layer_bytes(const elattn_gpu_params_s* p, int B, int x, int n) {
    const size_t R = size_t(B) * x, hk = size_t(p->h) * p->d_k, hm = size_t(p->h) * p->d_m;
    const size_t rows = size_t(x) * p->h;
    return split_bytes(R * p->d_m) + split_bytes(R * hk) + split_bytes(R * hm) +
           align256(size_t(B) * rows * pad32(n) * 4) + split_bytes(size_t(B) * rows * pad32(n)) + split_bytes(R * hm) +
           split_bytes(R * hk);
}

void tf32_gemm(const Split& A, int64_t lda, int64_t sAz, const float* const (&W)[2], const Split* Bop,
               int64_t ldb, int64_t sBz, float* C, float* C_lo, int64_t ldc, int64_t sCz, const float* bias,
               int64_t sbz, int M, int N, int K, int Z, cudaStream_t st) {
    Tf32GemmArgs g{};
    g.A_hi = A.hi, g.A_lo = A.lo, g.lda = lda, g.sAz = sAz;
    g.B_hi = Bop ? Bop->hi : W[0], g.B_lo = Bop ? Bop->lo : W[1], g.ldb = ldb, g.sBz = sBz;
    g.C = C, g.C_lo = C_lo, g.ldc = ldc, g.sCz = sCz, g.bias = bias, g.sbz = sbz;
    g.M = M, g.N = N, g.K = K, g.Z = Z, g.alpha = 1.f;
    launch_tf32_gemm(g, st);
}

struct Tf32H {
    Split H, HT;
    int B = 0, n = 0;
};
Tf32H tf32_split_h(const elattn_gpu_params_s* p, Scratch& s, const float* H, const int* npi, int B, int n,
                   cudaStream_t st, const int* h_index = nullptr) {
    Tf32H h;
    h.B = B, h.n = n;
    h.H = take_split(s, size_t(B) * n * p->d_m);
    h.HT = take_split(s, size_t(B) * p->d_m * pad32(n));
    launch_tf32_split(H, int64_t(B) * n, p->d_m, p->d_m, h.H.hi, h.H.lo, npi, n, st, h_index);
    launch_tf32_split_t(H, B, n, p->d_m, int(pad32(n)), npi, h.HT.hi, h.HT.lo, st, h_index);
    return h;
}

// stage (1) from split rows Y: Q (split) and q' (split, or plain into qp_out)
void tf32_query(const elattn_gpu_params_s* p, const Split& Y, int64_t R, const Split& Q, const Split& qp,
                float* qp_out, cudaStream_t st) {
    const int h = p->h, d_m = p->d_m, d_k = p->d_k, hk = h * d_k;
    const float* const Wq[2] = {p->WqT_s[0], p->WqT_s[1]};
    const float* const Wk[2] = {p->Wk_s[0], p->Wk_s[1]};
    tf32_gemm(Y, d_m, 0, Wq, nullptr, d_m, 0, Q.hi, Q.lo, hk, 0, p->bq, 0, int(R), hk, d_m, 1, st);
    tf32_gemm(Q, hk, d_k, Wk, nullptr, d_k, int64_t(d_m) * d_k, qp_out ? qp_out : qp.hi, qp_out ? nullptr : qp.lo,
              int64_t(h) * d_m, d_m, nullptr, 0, int(R), d_m, d_k, h, st);
}

// stage (2): ctx rows (split, or plain into ctx_out) from split q' over the split H
void tf32_decode(const elattn_gpu_params_s* p, Scratch& s, const Split& qp, const Tf32H& hs, const int* npi,
                 int rows, const Split& ctx, float* ctx_out, float2* stats, cudaStream_t st) {
    const int B = hs.B, n = hs.n, d_m = p->d_m;
    const int64_t np = pad32(n);
    float* S = static_cast<float*>(s.take(size_t(B) * rows * np * 4));
    const Split P = take_split(s, size_t(B) * rows * np);
    const float* const none[2] = {nullptr, nullptr};
    // S_b = q'_b . H_b^T  (scores, scale applied in the softmax)
    // (all n_pad columns: keys past n read as zeros; the softmax uses the first n_b)
    tf32_gemm(qp, d_m, int64_t(rows) * d_m, none, &hs.H, d_m, int64_t(n) * d_m, S, nullptr, np, int64_t(rows) * np,
              nullptr, 0, rows, int(np), d_m, B, st);
    launch_tf32_softmax(S, int64_t(B) * rows, rows, n, int(np), npi, float(1.0 / std::sqrt(double(p->d_k))), P.hi,
                        P.lo, stats, st);
    // C_b = P_b . H_b  (B operand: H_b^T [d_m][n_pad], K-major over keys)
    tf32_gemm(P, np, int64_t(rows) * np, none, &hs.HT, np, int64_t(d_m) * np, ctx_out ? ctx_out : ctx.hi,
              ctx_out ? nullptr : ctx.lo, d_m, int64_t(rows) * d_m, nullptr, 0, rows, d_m, int(np), B, st);
}

// stage (3): out = sum_i (C_i.W_V,i + b_V,i).W_O,i + b_O from split ctx rows
void tf32_output(const elattn_gpu_params_s* p, const Split& ctx, int64_t R, const Split& V, float* out,
                 cudaStream_t st) {
    const int h = p->h, d_m = p->d_m, d_k = p->d_k, hk = h * d_k;
    const float* const Wv[2] = {p->WvT_s[0], p->WvT_s[1]};
    const float* const Wo[2] = {p->WoT_s[0], p->WoT_s[1]};
    tf32_gemm(ctx, int64_t(h) * d_m, d_m, Wv, nullptr, d_m, int64_t(d_k) * d_m, V.hi, V.lo, hk, d_k, p->bv, d_k,
              int(R), d_k, d_m, h, st);
    tf32_gemm(V, hk, 0, Wo, nullptr, hk, 0, out, nullptr, d_m, 0, p->bo, 0, int(R), d_m, hk, 1, st);
}

// one layer step on the fp32 tensor-core path (H already split)
void tf32_layer(const elattn_gpu_params_s* p, Scratch& s, const float* Y, const Tf32H& hs, const int* npi, int x,
                float* out, cudaStream_t st) {
    const int64_t R = int64_t(hs.B) * x;
    const size_t hk = size_t(p->h) * p->d_k, hm = size_t(p->h) * p->d_m;
    const Split Ys = take_split(s, size_t(R) * p->d_m);
    const Split Q = take_split(s, size_t(R) * hk);
    const Split qp = take_split(s, size_t(R) * hm);
    launch_tf32_split(Y, R, p->d_m, p->d_m, Ys.hi, Ys.lo, nullptr, 1, st);
    tf32_query(p, Ys, R, Q, qp, nullptr, st);
    const Split ctx = take_split(s, size_t(R) * hm);
    tf32_decode(p, s, qp, hs, npi, x * p->h, ctx, nullptr, nullptr, st);
    const Split V = take_split(s, size_t(R) * hk);
    tf32_output(p, ctx, R, V, out, st);
}

bool use_tc_decode(const elattn_gpu_params_s* p, int rows_per_input) {
    return p->dtype == ELATTN_DTYPE_BF16 && el_decode_tc_supported(rows_per_input, p->d_m);
}

// (2) fused decode: C = softmax(q'.H^T / sqrt(d_k)) . H   (attention.hpp:272-280)
// h_static: H is not written by any kernel of the stream while these kernels run (the
// decoder step's graph), so the decode may start streaming it before its PDL wait
// h_index (slot-indexed caches): input b reads H[h_index[b]] of h_slots blocks
void decode(const elattn_gpu_params_s* p, const void* qp, const void* H, const int* npi, int B,
            int rows_per_input, int n, void* C, float* part, cudaStream_t st, float2* stats = nullptr,
            bool h_static = false, const int* h_index = nullptr, int h_slots = 0) {
    const float scale = float(1.0 / std::sqrt(double(p->d_k)));
    if (use_tc_decode(p, rows_per_input))
        launch_el_decode_tc(qp, H, npi, B, rows_per_input, n, p->d_m, scale, C, st, stats, part, h_static, h_index,
                            h_slots);
    else
        launch_el_decode_simt(p->dtype, qp, H, npi, B, rows_per_input, n, p->d_m, scale, C, st, stats, h_index);
}

void check_handle(const elattn_gpu_params_s* p) {
    ELA_REQUIRE(p != nullptr, ELATTN_ERR_PARAM, "null params handle");
}

}  // namespace
}  // namespace elattn_gpu

using namespace elattn_gpu;

extern "C" {

const char* elattn_gpu_version(void) {
    return "elattn-b200 0.1 (sm_100a: SIMT fp32/bf16, tcgen05 GEMM, tcgen05 fused EL decode)";
}

const char* elattn_gpu_last_error_message(void) { return g_last_error.c_str(); }

int64_t elattn_gpu_launch_count(void) { return g_launches; }
void elattn_gpu_reset_launch_count(void) { g_launches = 0; }

int elattn_gpu_params_create(int h, int d_m, int d_k, int dtype, int include_key_bias,
                             int include_value_bias, const double* Wq, const double* Wk,
                             const double* Wv, const double* Wo, const double* bq,
                             const double* bk, const double* bv, const double* bo,
                             elattn_gpu_params_t* out) {
    return guarded([&] {
        // AttentionParams::validate (attention.hpp:24-50)
        ELA_REQUIRE(out != nullptr, ELATTN_ERR_PARAM, "null output handle pointer");
        *out = nullptr;
        ELA_REQUIRE(h >= 1 && d_m >= 1 && d_k >= 1, ELATTN_ERR_PARAM,
                    "AttentionParams: h, d_m, d_k must be >= 1");
        ELA_REQUIRE(dtype == ELATTN_DTYPE_F32 || dtype == ELATTN_DTYPE_BF16, ELATTN_ERR_PARAM,
                    "unknown dtype");
        ELA_REQUIRE(Wq && Wk && Wv && Wo && bq && bk && bv && bo, ELATTN_ERR_SHAPE,
                    "AttentionParams: null weight array");
        const size_t H_ = size_t(h), M = size_t(d_m), K = size_t(d_k);
        std::vector<double> wqT(H_ * K * M), wkT(H_ * K * M), wk(H_ * M * K), wvT(H_ * K * M), woT(M * H_ * K);
        for (size_t i = 0; i < H_; ++i)
            for (size_t j = 0; j < M; ++j)
                for (size_t c = 0; c < K; ++c) {
                    const size_t src = (i * M + j) * K + c;  // [h][d_m][d_k]
                    wqT[(i * K + c) * M + j] = Wq[src];
                    wk[src] = Wk[src];
                    wkT[(i * K + c) * M + j] = Wk[src];
                    wvT[(i * K + c) * M + j] = Wv[src];
                }
        for (size_t i = 0; i < H_; ++i)
            for (size_t c = 0; c < K; ++c)
                for (size_t j = 0; j < M; ++j) woT[j * H_ * K + i * K + c] = Wo[(i * K + c) * M + j];
        std::vector<double> vbq(bq, bq + H_ * K), vbk(bk, bk + H_ * K), vbv(H_ * K, 0.0),
            vbo(bo, bo + M);
        if (include_value_bias) vbv.assign(bv, bv + H_ * K);
        std::unique_ptr<elattn_gpu_params_s, void (*)(elattn_gpu_params_s*)> p(
            new elattn_gpu_params_s, free_params);
        p->h = h, p->d_m = d_m, p->d_k = d_k, p->dtype = dtype;
        p->include_key_bias = include_key_bias != 0;
        p->include_value_bias = include_value_bias != 0;
        p->WqT = upload(wqT, dtype);
        p->Wk = upload(wk, dtype);
        p->WkT = upload(wkT, dtype);
        p->WvT = upload(wvT, dtype);
        p->WoT = upload(woT, dtype);
        p->bq = upload_f32(vbq);
        p->bk = upload_f32(vbk);
        p->bv = upload_f32(vbv);
        p->bo = upload_f32(vbo);
        if (dtype == ELATTN_DTYPE_F32) {
            upload_split(wqT, p->WqT_s);
            upload_split(wk, p->Wk_s);
            upload_split(wvT, p->WvT_s);
            upload_split(woT, p->WoT_s);
        }
        *out = p.release();
    });
}

int elattn_gpu_params_destroy(elattn_gpu_params_t params) {
    return guarded([&] { free_params(params); });
}

int elattn_gpu_params_info(elattn_gpu_params_t p, int* h, int* d_m, int* d_k, int* dtype) {
    return guarded([&] {
        check_handle(p);
        if (h) *h = p->h;
        if (d_m) *d_m = p->d_m;
        if (d_k) *d_k = p->d_k;
        if (dtype) *dtype = p->dtype;
    });
}

size_t elattn_gpu_workspace_size(elattn_gpu_params_t p, int B, int g, int n) {
    if (!p || B < 1 || g < 1) return 0;
    if (use_tf32_path(p) && n >= 1) return tf32_h_bytes(p, B, n) + tf32_layer_bytes(p, B, g, n);
    return step_workspace(p, int64_t(B) * g);
}

int elattn_gpu_decode_kernel_kind(elattn_gpu_params_t p, int g) {
    if (!p || g < 1) return -1;
    if (use_tf32_path(p)) return 2;
    return use_tc_decode(p, g * p->h) ? 1 : 0;
}

int elattn_gpu_build_el_query(elattn_gpu_params_t p, const void* Y, int R, void* qprime, float* s,
                              void* ws, size_t ws_bytes, elattn_stream_t stream) {
    return guarded([&] {
        check_handle(p);
        ELA_REQUIRE(R >= 1, ELATTN_ERR_SHAPE, "build_el_query: need at least one query row");
        ELA_REQUIRE(Y && qprime, ELATTN_ERR_PARAM, "build_el_query: null buffer");
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        const size_t qbytes = size_t(R) * p->h * p->d_k * dtype_bytes(p->dtype);
        if (use_tf32_path(p) && al16p(Y) && al16p(qprime)) {
            // fp32 on the tensor cores: Q plain (for s), then split for q' = Q_i.W_K,i^T
            const size_t hk = size_t(p->h) * p->d_k;
            Scratch scratch(ws, ws_bytes, split_bytes(size_t(R) * p->d_m) + align256(qbytes) + split_bytes(R * hk), st);
            const Split Ys = take_split(scratch, size_t(R) * p->d_m);
            float* Q = static_cast<float*>(scratch.take(qbytes));
            const Split Qs = take_split(scratch, size_t(R) * hk);
            launch_tf32_split(static_cast<const float*>(Y), R, p->d_m, p->d_m, Ys.hi, Ys.lo, nullptr, 1, st);
            const float* const Wq[2] = {p->WqT_s[0], p->WqT_s[1]};
            const float* const Wk[2] = {p->Wk_s[0], p->Wk_s[1]};
            tf32_gemm(Ys, p->d_m, 0, Wq, nullptr, p->d_m, 0, Q, nullptr, int64_t(hk), 0, p->bq, 0, R, int(hk), p->d_m,
                      1, st);
            launch_tf32_split(Q, R, int(hk), int64_t(hk), Qs.hi, Qs.lo, nullptr, 1, st);
            tf32_gemm(Qs, int64_t(hk), p->d_k, Wk, nullptr, p->d_k, int64_t(p->d_m) * p->d_k,
                      static_cast<float*>(qprime), nullptr, int64_t(p->h) * p->d_m, p->d_m, nullptr, 0, R, p->d_m,
                      p->d_k, p->h, st);
            if (s) {
                if (p->include_key_bias)
                    launch_key_bias_scalars(p->dtype, Q, p->bk, R, p->h, p->d_k, s, st);
                else
                    ELA_CHECK_CUDA(cudaMemsetAsync(s, 0, sizeof(float) * size_t(R) * p->h, st));
            }
            return;
        }
        Scratch scratch(ws, ws_bytes, align256(qbytes), st);
        void* Q = scratch.take(qbytes);
        query_expansion(p, Y, R, Q, qprime, st, /*need_Q=*/s != nullptr && p->include_key_bias);
        if (s) {
            if (p->include_key_bias)
                launch_key_bias_scalars(p->dtype, Q, p->bk, R, p->h, p->d_k, s, st);
            else
                ELA_CHECK_CUDA(cudaMemsetAsync(s, 0, sizeof(float) * size_t(R) * p->h, st));
        }
    });
}

int elattn_gpu_el_attention_folded(elattn_gpu_params_t p, const void* qprime, const float* s,
                                   const void* H, const int* n_per_input, int B, int g, int n,
                                   void* out, void* ws, size_t ws_bytes, elattn_stream_t stream) {
    (void)s;  // shift invariance: see header
    return guarded([&] {
        check_handle(p);
        ELA_REQUIRE(B >= 1 && g >= 1, ELATTN_ERR_SHAPE,
                    "el_attention_folded: query row count must be a positive multiple of h");
        ELA_REQUIRE(n >= 1, ELATTN_ERR_STATE, "el_attention_folded: empty context");
        ELA_REQUIRE(qprime && H && out, ELATTN_ERR_PARAM, "el_attention_folded: null buffer");
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        const int64_t R = int64_t(B) * g;
        if (use_tf32_path(p) && al16p(qprime) && al16p(H) && al16p(out)) {
            Scratch scratch(ws, ws_bytes, tf32_h_bytes(p, B, n) + tf32_layer_bytes(p, B, g, n), st);
            const size_t hm = size_t(R) * p->h * p->d_m;
            const Split qs = take_split(scratch, hm);
            launch_tf32_split(static_cast<const float*>(qprime), int64_t(R) * p->h, p->d_m, p->d_m, qs.hi, qs.lo,
                              nullptr, 1, st);
            const Tf32H hs = tf32_split_h(p, scratch, static_cast<const float*>(H), n_per_input, B, n, st);
            const Split ctx = take_split(scratch, hm);
            tf32_decode(p, scratch, qs, hs, n_per_input, g * p->h, ctx, nullptr, nullptr, st);
            const Split V = take_split(scratch, size_t(R) * p->h * p->d_k);
            tf32_output(p, ctx, R, V, static_cast<float*>(out), st);
            return;
        }
        const size_t e = dtype_bytes(p->dtype);
        const size_t cbytes = size_t(R) * p->h * p->d_m * e, vbytes = size_t(R) * p->h * p->d_k * e;
        Scratch scratch(ws, ws_bytes, align256(cbytes) + align256(vbytes) + decode_scratch(p), st);
        void* C = scratch.take(cbytes);
        void* V = scratch.take(vbytes);
        float* part = static_cast<float*>(scratch.take(decode_scratch(p)));
        decode(p, qprime, H, n_per_input, B, g * p->h, n, C, part, st);
        output_projection(p, C, R, V, out, st);
    });
}

int elattn_gpu_el_attention_decode(elattn_gpu_params_t p, const void* qprime, const void* H,
                                   const int* n_per_input, int B, int rows, int n, void* ctx,
                                   elattn_stream_t stream) {
    return guarded([&] {
        check_handle(p);
        ELA_REQUIRE(B >= 1 && rows >= 1, ELATTN_ERR_SHAPE, "el_attention_decode: B, rows must be >= 1");
        ELA_REQUIRE(n >= 1, ELATTN_ERR_STATE, "el_attention_decode: empty context");
        ELA_REQUIRE(qprime && H && ctx, ELATTN_ERR_PARAM, "el_attention_decode: null buffer");
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        if (use_tf32_path(p) && al16p(qprime) && al16p(H) && al16p(ctx)) {
            const size_t qn = size_t(B) * rows * p->d_m, np = size_t(pad32(n));
            Scratch scratch(nullptr, 0,
                            split_bytes(qn) + tf32_h_bytes(p, B, n) + align256(size_t(B) * rows * np * 4) +
                                split_bytes(size_t(B) * rows * np),
                            st);
            const Split qs = take_split(scratch, qn);
            launch_tf32_split(static_cast<const float*>(qprime), int64_t(B) * rows, p->d_m, p->d_m, qs.hi, qs.lo,
                              nullptr, 1, st);
            const Tf32H hs = tf32_split_h(p, scratch, static_cast<const float*>(H), n_per_input, B, n, st);
            tf32_decode(p, scratch, qs, hs, n_per_input, rows, Split{}, static_cast<float*>(ctx), nullptr, st);
            return;
        }
        Scratch scratch(nullptr, 0, decode_scratch(p), st);
        decode(p, qprime, H, n_per_input, B, rows, n, ctx, static_cast<float*>(scratch.take(decode_scratch(p))), st);
    });
}

int elattn_gpu_el_attention_step(elattn_gpu_params_t p, const void* Y, const void* H,
                                 const int* n_per_input, int B, int x, int n, void* out, void* ws,
                                 size_t ws_bytes, elattn_stream_t stream) {
    return elattn_gpu_el_attention_step_indexed(p, Y, H, n_per_input, nullptr, 0, B, x, n, out, ws, ws_bytes,
                                                stream);
}

int elattn_gpu_el_attention_step_indexed(elattn_gpu_params_t p, const void* Y, const void* H,
                                         const int* n_per_input, const int* h_index, int h_slots, int B, int x,
                                         int n, void* out, void* ws, size_t ws_bytes, elattn_stream_t stream) {
    return guarded([&] {
        check_handle(p);
        ELA_REQUIRE(B >= 1 && x >= 1, ELATTN_ERR_SHAPE, "el_attention_step: B and x must be >= 1");
        ELA_REQUIRE(n >= 1, ELATTN_ERR_STATE, "el_attention: empty context");
        ELA_REQUIRE(Y && H && out, ELATTN_ERR_PARAM, "el_attention_step: null buffer");
        ELA_REQUIRE(h_index == nullptr || h_slots >= 1, ELATTN_ERR_SHAPE, "el_attention_step: h_slots must be >= 1");
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        const int64_t R = int64_t(B) * x;
        if (use_tf32_path(p) && al16p(Y) && al16p(H) && al16p(out)) {
            Scratch scratch(ws, ws_bytes, tf32_h_bytes(p, B, n) + tf32_layer_bytes(p, B, x, n), st);
            const Tf32H hs = tf32_split_h(p, scratch, static_cast<const float*>(H), n_per_input, B, n, st, h_index);
            tf32_layer(p, scratch, static_cast<const float*>(Y), hs, n_per_input, x, static_cast<float*>(out), st);
            return;
        }
        const size_t e = dtype_bytes(p->dtype);
        const size_t qb = size_t(R) * p->h * p->d_k * e, qpb = size_t(R) * p->h * p->d_m * e;
        Scratch scratch(ws, ws_bytes, step_workspace(p, R), st);
        void* Q = scratch.take(qb);
        void* qp = scratch.take(qpb);
        void* C = scratch.take(qpb);
        void* V = scratch.take(qb);
        float* part = static_cast<float*>(scratch.take(decode_scratch(p)));
        query_expansion(p, Y, R, Q, qp, st, /*need_Q=*/false);
        decode(p, qp, H, n_per_input, B, x * p->h, n, C, part, st, nullptr, false, h_index, h_slots);
        output_projection(p, C, R, V, out, st);
    });
}

}  // extern "C"

#include "elattn_gpu_testing.h"

extern "C" int elattn_gpu_testing_gemm_bf16(const void* A, int64_t lda, int64_t sAz, const void* B, int64_t ldb,
                                            int64_t sBz, void* C, int64_t ldc, int64_t sCz, const float* bias,
                                            int64_t sbz, int M, int N, int K, int Z, float alpha, int kernel,
                                            elattn_stream_t stream) {
    return guarded([&] {
        GemmArgs g{};
        g.A = A, g.lda = lda, g.sAz = sAz, g.B = B, g.ldb = ldb, g.sBz = sBz, g.C = C, g.ldc = ldc, g.sCz = sCz;
        g.bias = bias, g.sbz = sbz, g.M = M, g.N = N, g.K = K, g.Z = Z, g.alpha = alpha;
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        if (kernel == 1) {
            ELA_REQUIRE(tc_gemm_supported(g), ELATTN_ERR_UNSUPPORTED, "shape outside the tcgen05 GEMM envelope");
            launch_tc_gemm(g, st);
        } else {
            launch_simt_gemm(ELATTN_DTYPE_BF16, g, st);
        }
    });
}

extern "C" int elattn_gpu_testing_gemm_config(int bn, int mt, int kbp) {
    return guarded([&] {
        ELA_REQUIRE((bn == 0 || bn == 64 || bn == 128 || bn == 256) && mt >= 0 && mt <= 2 && kbp >= 0 && kbp <= 2,
                    ELATTN_ERR_PARAM, "gemm_config: bn in {0, 64, 128, 256}, mt and kbp in {0, 1, 2}");
        g_gemm_force_bn = bn, g_gemm_force_mt = mt, g_gemm_force_kbp = kbp;
    });
}

extern "C" int elattn_gpu_testing_decode_sched(int mode) {
    return guarded([&] {
        ELA_REQUIRE(mode >= 0 && mode <= 3, ELATTN_ERR_PARAM, "decode_sched: 0 auto, 1 stream-K, 2 whole, 3 tail");
        g_decode_sched_override = mode;
    });
}

extern "C" int elattn_gpu_testing_qexp_fused(int mode) {
    g_qexp_fused = mode < 0 ? -1 : (mode ? 1 : 0);  // 1: forced (the tests sweep it up to 256 rows)
    return ELATTN_OK;
}

extern "C" int elattn_gpu_testing_gemm_splitk(int sk) {
    return guarded([&] {
        ELA_REQUIRE(sk == -1 || sk == 0 || sk == 2 || sk == 4 || sk == 8, ELATTN_ERR_PARAM,
                    "gemm_splitk: sk in {-1, 0, 2, 4, 8}");
        g_gemm_force_splitk = sk;
    });
}

extern "C" int elattn_gpu_testing_gemm_epilogue(int tma) {
    g_gemm_epilogue_tma = tma < 0 ? -1 : (tma ? 1 : 0);
    return ELATTN_OK;
}

extern "C" int elattn_gpu_testing_set_pdl(int on) {
    g_pdl = on ? 1 : 0;
    return ELATTN_OK;
}

extern "C" int elattn_gpu_testing_set_gemm_trace(unsigned long long* trace) {
    g_gemm_trace = trace;
    return ELATTN_OK;
}

extern "C" int elattn_gpu_testing_gemm_tf32x3(const float* A, int64_t lda, int64_t sAz, const float* B, int64_t ldb,
                                              int64_t sBz, float* C, float* C_lo, int64_t ldc,
                                              int64_t sCz, const float* bias, int64_t sbz, int M, int N, int K, int Z,
                                              float alpha, elattn_stream_t stream) {
    return guarded([&] {
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        // operands split into (hi, lo) copies, then the 3xTF32 GEMM
        const int64_t a_rows = (sAz == 0 || Z == 1) ? M : int64_t(Z) * sAz / lda;
        const int64_t b_rows = (sBz == 0 || Z == 1) ? N : int64_t(Z) * sBz / ldb;
        const size_t abytes = sizeof(float) * size_t(a_rows) * lda, bbytes = sizeof(float) * size_t(b_rows) * ldb;
        Scratch sc(nullptr, 0, 2 * align256(abytes) + 2 * align256(bbytes), st);
        float* Ah = static_cast<float*>(sc.take(abytes));
        float* Al = static_cast<float*>(sc.take(abytes));
        float* Bh = static_cast<float*>(sc.take(bbytes));
        float* Bl = static_cast<float*>(sc.take(bbytes));
        launch_tf32_split(A, a_rows, int(lda), lda, Ah, Al, nullptr, 1, st);
        launch_tf32_split(B, b_rows, int(ldb), ldb, Bh, Bl, nullptr, 1, st);
        Tf32GemmArgs g{};
        g.A_hi = Ah, g.A_lo = Al, g.lda = lda, g.sAz = sAz;
        g.B_hi = Bh, g.B_lo = Bl, g.ldb = ldb, g.sBz = sBz;
        g.C = C, g.C_lo = C_lo, g.ldc = ldc, g.sCz = sCz, g.bias = bias, g.sbz = sbz;
        g.M = M, g.N = N, g.K = K, g.Z = Z, g.alpha = alpha;
        launch_tf32_gemm(g, st);
    });
}

extern "C" int elattn_gpu_testing_timeline(void* records, unsigned* count, unsigned capacity) {
    const bool ok = tl_set_gemm(static_cast<TlRec*>(records), count, capacity) &
                    tl_set_decode(static_cast<TlRec*>(records), count, capacity);
    return ok ? ELATTN_OK : ELATTN_ERR_UNSUPPORTED;
}

extern "C" int elattn_gpu_testing_set_decode_trace(unsigned long long* trace) {
    g_decode_trace = trace;
    return ELATTN_OK;
}

extern "C" int elattn_gpu_testing_decode_bf16(const void* qprime, const void* H, const int* n_per_input, int B,
                                              int rows, int n, int d_m, float scale, void* ctx, int kernel,
                                              elattn_stream_t stream) {
    return guarded([&] {
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        if (kernel == 1) {
            ELA_REQUIRE(el_decode_tc_supported(rows, d_m), ELATTN_ERR_UNSUPPORTED,
                        "shape outside the tcgen05 decode envelope");
            Scratch scratch(nullptr, 0, align256(el_decode_tc_scratch_bytes(d_m)), st);
            launch_el_decode_tc(qprime, H, n_per_input, B, rows, n, d_m, scale, ctx, st, nullptr,
                                static_cast<float*>(scratch.take(el_decode_tc_scratch_bytes(d_m))));
        } else {
            launch_el_decode_simt(ELATTN_DTYPE_BF16, qprime, H, n_per_input, B, rows, n, d_m, scale, ctx, st);
        }
    });
}

// ---------------------------------------------------------------- batched decoder step
struct elattn_gpu_decoder_s {
    std::vector<elattn_gpu_params_t> layers;
    int B = 0, x = 0, n = 0;
    cudaStream_t st = nullptr;  // private capture stream (owns its per-stream scratch)
    void* ybuf[2] = {nullptr, nullptr};
    void* ws = nullptr;
    size_t ws_bytes = 0;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int64_t kernels = 0;
    bool tf32 = false;  // fp32 layers on the tensor-core path
};

namespace elattn_gpu {
}  // namespace elattn_gpu

namespace {
void decoder_free(elattn_gpu_decoder_s* d) {
    if (!d) return;
    if (d->exec) cudaGraphExecDestroy(d->exec);
    if (d->graph) cudaGraphDestroy(d->graph);
    for (void* p : {d->ybuf[0], d->ybuf[1], d->ws})
        if (p) cudaFree(p);
    if (d->st) {
        cudaStreamSynchronize(d->st);
        cudaStreamDestroy(d->st);
    }
    delete d;
}

// one step: L layers, ping-pong intermediate rows, last layer writes `out`
void decoder_enqueue(elattn_gpu_decoder_s* d, const void* H, const int* npi, const void* Y_in, void* out) {
    const elattn_gpu_params_s* p0 = d->layers[0];
    const int64_t R = int64_t(d->B) * d->x;
    if (d->tf32) {
        // fp32 on the tensor cores: H split once per step, shared by the L layers
        Scratch s(d->ws, d->ws_bytes, d->ws_bytes, d->st);
        const Tf32H hs = tf32_split_h(p0, s, static_cast<const float*>(H), npi, d->B, d->n, d->st);
        const size_t mark = s.mark();
        const float* y = static_cast<const float*>(Y_in);
        const int L = int(d->layers.size());
        for (int l = 0; l < L; ++l) {
            float* dst = static_cast<float*>((l == L - 1) ? out : d->ybuf[l & 1]);
            s.reset(mark);
            tf32_layer(d->layers[l], s, y, hs, npi, d->x, dst, d->st);
            y = dst;
        }
        return;
    }
    const size_t e = dtype_bytes(p0->dtype);
    const size_t qb = size_t(R) * p0->h * p0->d_k * e, qpb = size_t(R) * p0->h * p0->d_m * e;
    char* base = static_cast<char*>(d->ws);
    void* Q = base;
    void* qp = base + align256(qb);
    void* C = base + align256(qb) + align256(qpb);
    void* V = base + align256(qb) + 2 * align256(qpb);
    float* part = reinterpret_cast<float*>(base + 2 * align256(qb) + 2 * align256(qpb));
    const void* y = Y_in;
    const int L = int(d->layers.size());
    for (int l = 0; l < L; ++l) {
        void* dst = (l == L - 1) ? out : d->ybuf[l & 1];
        const elattn_gpu_params_s* p = d->layers[l];
        query_expansion(p, y, R, Q, qp, d->st, /*need_Q=*/false);
        decode(p, qp, H, npi, d->B, d->x * p->h, d->n, C, part, d->st, nullptr, /*h_static=*/true);
        output_projection(p, C, R, V, dst, d->st);
        y = dst;
    }
}
}  // namespace

extern "C" int elattn_gpu_decoder_create(const elattn_gpu_params_t* layers, int L, const void* H,
                                         const int* n_per_input, int B, int x, int n, const void* Y_in, void* out,
                                         elattn_gpu_decoder_t* dec) {
    return guarded([&] {
        ELA_REQUIRE(dec != nullptr, ELATTN_ERR_PARAM, "decoder_create: null output handle pointer");
        *dec = nullptr;
        ELA_REQUIRE(layers != nullptr && L >= 1, ELATTN_ERR_PARAM, "decoder_create: need at least one layer");
        ELA_REQUIRE(B >= 1 && x >= 1, ELATTN_ERR_SHAPE, "decoder_create: B and x must be >= 1");
        ELA_REQUIRE(n >= 1, ELATTN_ERR_STATE, "decoder_create: empty context");
        ELA_REQUIRE(H && Y_in && out, ELATTN_ERR_PARAM, "decoder_create: null buffer");
        const elattn_gpu_params_s* p0 = layers[0];
        ELA_REQUIRE(p0 != nullptr, ELATTN_ERR_PARAM, "decoder_create: null layer");
        for (int l = 0; l < L; ++l) {
            const elattn_gpu_params_s* p = layers[l];
            ELA_REQUIRE(p && p->h == p0->h && p->d_m == p0->d_m && p->d_k == p0->d_k && p->dtype == p0->dtype,
                        ELATTN_ERR_PARAM, "decoder_create: layers must share h, d_m, d_k and dtype");
        }
        std::unique_ptr<elattn_gpu_decoder_s, void (*)(elattn_gpu_decoder_s*)> d(new elattn_gpu_decoder_s,
                                                                                 decoder_free);
        d->layers.assign(layers, layers + L);
        d->B = B, d->x = x, d->n = n;
        const int64_t R = int64_t(B) * x;
        const size_t rows_bytes = size_t(R) * p0->d_m * dtype_bytes(p0->dtype);
        ELA_CHECK_CUDA(cudaStreamCreateWithFlags(&d->st, cudaStreamNonBlocking));
        ELA_CHECK_CUDA(cudaMalloc(&d->ybuf[0], rows_bytes));
        ELA_CHECK_CUDA(cudaMalloc(&d->ybuf[1], rows_bytes));
        d->tf32 = use_tf32_path(p0) && al16p(H) && al16p(Y_in) && al16p(out);
        d->ws_bytes = d->tf32 ? tf32_h_bytes(p0, B, n) + tf32_layer_bytes(p0, B, x, n) : step_workspace(p0, R);
        ELA_CHECK_CUDA(cudaMalloc(&d->ws, d->ws_bytes));
        // eager run first (surfaces launch errors directly).  The private stream does not
        // order after the caller's streams: wait for all prior device work (the caller may
        // still be writing Y_in / H / n_per_input) and write the warm-up result into scratch,
        // not into `out`, which the caller may still be reading.
        ELA_CHECK_CUDA(cudaDeviceSynchronize());
        void* warm_out = nullptr;
        ELA_CHECK_CUDA(cudaMalloc(&warm_out, rows_bytes));
        try {
            decoder_enqueue(d.get(), H, n_per_input, Y_in, warm_out);
        } catch (...) {
            cudaStreamSynchronize(d->st);
            cudaFree(warm_out);
            throw;
        }
        const cudaError_t warm_err = cudaStreamSynchronize(d->st);
        cudaFree(warm_out);
        ELA_CHECK_CUDA(warm_err);
        const int64_t before = g_launches;
        ELA_CHECK_CUDA(cudaStreamBeginCapture(d->st, cudaStreamCaptureModeThreadLocal));
        try {
            decoder_enqueue(d.get(), H, n_per_input, Y_in, out);
        } catch (...) {
            cudaGraph_t g = nullptr;
            cudaStreamEndCapture(d->st, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        d->kernels = g_launches - before;
        g_launches = before;
        ELA_CHECK_CUDA(cudaStreamEndCapture(d->st, &d->graph));
        ELA_CHECK_CUDA(cudaGraphInstantiate(&d->exec, d->graph, 0));
        *dec = d.release();
    });
}

extern "C" int elattn_gpu_decoder_run(elattn_gpu_decoder_t dec, elattn_stream_t stream) {
    return guarded([&] {
        ELA_REQUIRE(dec != nullptr, ELATTN_ERR_PARAM, "decoder_run: null handle");
        ELA_CHECK_CUDA(cudaGraphLaunch(dec->exec, reinterpret_cast<cudaStream_t>(stream)));
        count_launch(int(dec->kernels));
    });
}

extern "C" int elattn_gpu_decoder_destroy(elattn_gpu_decoder_t dec) {
    return guarded([&] { decoder_free(dec); });
}

extern "C" int64_t elattn_gpu_decoder_kernels_per_run(elattn_gpu_decoder_t dec) { return dec ? dec->kernels : -1; }

// ---------------------------------------------------------------- per-lane hidden-state caches
extern "C" int elattn_gpu_cache_append(void* cache, const void* Y, int* lengths, int lanes, int n_max, int d_m,
                                       int dtype, elattn_stream_t stream) {
    return guarded([&] {
        ELA_REQUIRE(cache && Y && lengths, ELATTN_ERR_PARAM, "cache_append: null buffer");
        ELA_REQUIRE(lanes >= 1 && n_max >= 1 && d_m >= 1, ELATTN_ERR_SHAPE, "cache_append: bad shape");
        ELA_REQUIRE(dtype == ELATTN_DTYPE_F32 || dtype == ELATTN_DTYPE_BF16, ELATTN_ERR_PARAM, "unknown dtype");
        launch_cache_append(cache, Y, lengths, lanes, n_max, d_m, dtype, reinterpret_cast<cudaStream_t>(stream));
    });
}

extern "C" int elattn_gpu_cache_append_indexed(void* cache, const void* Y, int* lengths, const int* lane_slot,
                                               int lanes, int n_max, int d_m, int dtype, elattn_stream_t stream) {
    return guarded([&] {
        ELA_REQUIRE(cache && Y && lengths && lane_slot, ELATTN_ERR_PARAM, "cache_append: null buffer");
        ELA_REQUIRE(lanes >= 1 && n_max >= 1 && d_m >= 1, ELATTN_ERR_SHAPE, "cache_append: bad shape");
        ELA_REQUIRE(dtype == ELATTN_DTYPE_F32 || dtype == ELATTN_DTYPE_BF16, ELATTN_ERR_PARAM, "unknown dtype");
        launch_cache_append(cache, Y, lengths, lanes, n_max, d_m, dtype, reinterpret_cast<cudaStream_t>(stream),
                            lane_slot);
    });
}

extern "C" size_t elattn_gpu_cache_fork_workspace(int slots, int lanes_in, int lanes_out) {
    return cache_fork_workspace(slots, lanes_in, lanes_out);
}

extern "C" int elattn_gpu_cache_fork(void* cache, int layers, int slots, int n_max, int d_m, int dtype,
                                     const int* lengths_in, int* lengths_out, const int* slot_in, int* slot_out,
                                     const int* parent, int lanes_in, int lanes_out, int rows_hint, void* workspace,
                                     size_t workspace_bytes, elattn_stream_t stream) {
    return guarded([&] {
        ELA_REQUIRE(cache && lengths_in && lengths_out && slot_in && slot_out && parent, ELATTN_ERR_PARAM,
                    "cache_fork: null buffer");
        ELA_REQUIRE(lengths_in != lengths_out && slot_in != slot_out, ELATTN_ERR_PARAM,
                    "cache_fork: the lengths / slot maps in and out must differ");
        ELA_REQUIRE(lanes_out >= 1, ELATTN_ERR_STATE, "gather_lanes: all lanes dropped");
        ELA_REQUIRE(layers >= 1 && lanes_in >= 1 && slots >= 1 && n_max >= 1 && d_m >= 1, ELATTN_ERR_SHAPE,
                    "cache_fork: bad shape");
        ELA_REQUIRE(dtype == ELATTN_DTYPE_F32 || dtype == ELATTN_DTYPE_BF16, ELATTN_ERR_PARAM, "unknown dtype");
        launch_cache_fork(cache, layers, slots, n_max, d_m, dtype, lengths_in, lengths_out, slot_in, slot_out, parent,
                          lanes_in, lanes_out, rows_hint, workspace, workspace_bytes,
                          reinterpret_cast<cudaStream_t>(stream));
    });
}

extern "C" int elattn_gpu_cache_gather(const void* src, const int* src_lengths, void* dst, int* dst_lengths,
                                       const int* parent, int lanes_in, int lanes_out, int n_max, int d_m, int dtype,
                                       int rows_hint, elattn_stream_t stream) {
    return guarded([&] {
        ELA_REQUIRE(src && src_lengths && dst && dst_lengths && parent, ELATTN_ERR_PARAM, "cache_gather: null buffer");
        ELA_REQUIRE(src != dst, ELATTN_ERR_PARAM, "cache_gather: src and dst must differ");
        ELA_REQUIRE(lanes_out >= 1, ELATTN_ERR_STATE, "gather_lanes: all lanes dropped");
        ELA_REQUIRE(lanes_in >= 1 && n_max >= 1 && d_m >= 1, ELATTN_ERR_SHAPE, "cache_gather: bad shape");
        ELA_REQUIRE(dtype == ELATTN_DTYPE_F32 || dtype == ELATTN_DTYPE_BF16, ELATTN_ERR_PARAM, "unknown dtype");
        launch_cache_gather(src, src_lengths, dst, dst_lengths, parent, lanes_in, lanes_out, n_max, d_m, dtype,
                            rows_hint, reinterpret_cast<cudaStream_t>(stream));
    });
}

// ---------------------------------------------------------------- decoder-only mixed self-attention
extern "C" int elattn_gpu_kv_append(elattn_gpu_params_t p, const void* Y, int R, void* Kc, void* Vc, int t_max, int t,
                                    elattn_stream_t stream) {
    return guarded([&] {
        check_handle(p);
        ELA_REQUIRE(Y && Kc && Vc, ELATTN_ERR_PARAM, "kv_append: null buffer");
        ELA_REQUIRE(R >= 1 && t_max >= 1, ELATTN_ERR_SHAPE, "kv_append: bad shape");
        ELA_REQUIRE(t >= 0 && t < t_max, ELATTN_ERR_STATE, "kv_append: cache full");
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        const int h = p->h, d_m = p->d_m, d_k = p->d_k;
        const size_t e = dtype_bytes(p->dtype);
        // K_i / V_i of every lane at position t of [R][h][t_max][d_k]  (KvCache::append,
        // attention.hpp:134-150): one head-batched GEMM each, Y shared by the heads
        for (int kv = 0; kv < 2; ++kv) {
            GemmArgs a{};
            a.A = Y, a.lda = d_m, a.sAz = 0;
            a.B = kv == 0 ? p->WkT : p->WvT, a.ldb = d_m, a.sBz = int64_t(d_k) * d_m;
            a.C = static_cast<char*>(kv == 0 ? Kc : Vc) + size_t(t) * d_k * e;
            a.ldc = int64_t(h) * t_max * d_k, a.sCz = int64_t(t_max) * d_k;
            a.bias = kv == 0 ? (p->include_key_bias ? p->bk : nullptr) : p->bv, a.sbz = d_k;
            a.M = R, a.N = d_k, a.K = d_m, a.Z = h, a.alpha = 1.f;
            gemm(p, a, st);
        }
    });
}

extern "C" int elattn_gpu_mixed_self_attention(elattn_gpu_params_t p, const void* Y, const void* P,
                                               const int* n_per_input, int B, int x, int n, const void* Kc,
                                               const void* Vc, int t_max, int t_out, void* out, void* ws,
                                               size_t ws_bytes, elattn_stream_t stream) {
    return guarded([&] {
        check_handle(p);
        ELA_REQUIRE(B >= 1 && x >= 1, ELATTN_ERR_SHAPE, "mixed_self_attention: B and x must be >= 1");
        ELA_REQUIRE(n >= 1, ELATTN_ERR_STATE, "mixed_self_attention: empty prefix");
        ELA_REQUIRE(t_out >= 0 && t_out <= t_max, ELATTN_ERR_STATE,
                    "mixed_self_attention: cache does not match params");
        ELA_REQUIRE(Y && P && out && (t_out == 0 || (Kc && Vc)), ELATTN_ERR_PARAM, "mixed_self_attention: null buffer");
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        const int64_t R = int64_t(B) * x;
        const size_t e = dtype_bytes(p->dtype);
        const size_t qb = size_t(R) * p->h * p->d_k * e, qpb = size_t(R) * p->h * p->d_m * e;
        const size_t sb = size_t(R) * p->h * sizeof(float2);
        Scratch scratch(ws, ws_bytes, step_workspace(p, R) + align256(sb), st);
        void* Q = scratch.take(qb);
        void* qp = scratch.take(qpb);
        void* C = scratch.take(qpb);
        void* V = scratch.take(qb);
        float* part = static_cast<float*>(scratch.take(decode_scratch(p)));
        float2* stats = static_cast<float2*>(scratch.take(sb));
        query_expansion(p, Y, R, Q, qp, st);
        decode(p, qp, P, n_per_input, B, x * p->h, n, C, part, st, stats);
        v_projection(p, C, R, V, st);
        if (t_out > 0)
            launch_mixed_combine(p->dtype, Q, stats, V, Kc, Vc, int(R), p->h, p->d_k, t_max, t_out,
                                 p->include_key_bias ? p->bk : nullptr, float(1.0 / std::sqrt(double(p->d_k))), st);
        o_projection(p, V, R, out, st);
    });
}

extern "C" size_t elattn_gpu_mixed_workspace_size(elattn_gpu_params_t p, int B, int x) {
    if (!p || B < 1 || x < 1) return 0;
    const int64_t R = int64_t(B) * x;
    return step_workspace(p, R) + align256(size_t(R) * p->h * sizeof(float2));
}

// ---------------------------------------------------------------- MHA baseline (K/V caches)
extern "C" int elattn_gpu_mha_kv_build(elattn_gpu_params_t p, const void* H, int B, int n, void* Kc, void* Vc,
                                       elattn_stream_t stream) {
    return guarded([&] {
        check_handle(p);
        ELA_REQUIRE(H && Kc && Vc, ELATTN_ERR_PARAM, "mha_kv_build: null buffer");
        ELA_REQUIRE(B >= 1, ELATTN_ERR_SHAPE, "mha_kv_build: B must be >= 1");
        ELA_REQUIRE(n >= 1, ELATTN_ERR_STATE, "multi_head_attention: empty context");
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        const int h = p->h, d_m = p->d_m, d_k = p->d_k;
        const int64_t rows = int64_t(B) * n;
        ELA_REQUIRE(rows < (int64_t(1) << 31), ELATTN_ERR_UNSUPPORTED, "mha_kv_build: B * n too large");
        // K_i / V_i of every position of every input (KvCache::append, attention.hpp:134-150,
        // for all positions at once): A = H shared by the heads, output [h][B*n][d_k]
        for (int kv = 0; kv < 2; ++kv) {
            GemmArgs a{};
            a.A = H, a.lda = d_m, a.sAz = 0;
            a.B = kv == 0 ? p->WkT : p->WvT, a.ldb = d_m, a.sBz = int64_t(d_k) * d_m;
            a.C = kv == 0 ? Kc : Vc, a.ldc = d_k, a.sCz = rows * d_k;
            a.bias = kv == 0 ? (p->include_key_bias ? p->bk : nullptr) : (p->include_value_bias ? p->bv : nullptr);
            a.sbz = d_k;
            a.M = int(rows), a.N = d_k, a.K = d_m, a.Z = h, a.alpha = 1.f;
            gemm(p, a, st);
        }
    });
}

extern "C" size_t elattn_gpu_mha_workspace_size(elattn_gpu_params_t p, int B, int x) {
    if (!p || B < 1 || x < 1) return 0;
    const size_t qb = size_t(B) * x * p->h * p->d_k * dtype_bytes(p->dtype);
    return 2 * align256(qb);
}

extern "C" int elattn_gpu_mha_attention(elattn_gpu_params_t p, const void* Y, const void* Kc, const void* Vc,
                                        const int* n_per_input, int B, int x, int n, void* out, void* ws,
                                        size_t ws_bytes, elattn_stream_t stream) {
    return guarded([&] {
        check_handle(p);
        ELA_REQUIRE(B >= 1 && x >= 1, ELATTN_ERR_SHAPE, "mha_attention: B and x must be >= 1");
        ELA_REQUIRE(n >= 1, ELATTN_ERR_STATE, "multi_head_attention: empty context");
        ELA_REQUIRE(Y && Kc && Vc && out, ELATTN_ERR_PARAM, "mha_attention: null buffer");
        ELA_REQUIRE(mha_decode_supported(x, p->d_k, p->dtype), ELATTN_ERR_UNSUPPORTED,
                    "mha_attention: x <= 16 query rows per input, d_k a multiple of 8 up to 128");
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        const int64_t R = int64_t(B) * x;
        const int hk = p->h * p->d_k;
        const size_t qb = size_t(R) * hk * dtype_bytes(p->dtype);
        Scratch scratch(ws, ws_bytes, 2 * align256(qb), st);
        void* Q = scratch.take(qb);
        void* ctx = scratch.take(qb);
        GemmArgs a{};  // Q = Y.W_Q + b_Q (attention.hpp:106)
        a.A = Y, a.lda = p->d_m, a.B = p->WqT, a.ldb = p->d_m, a.C = Q, a.ldc = hk, a.bias = p->bq;
        a.M = int(R), a.N = hk, a.K = p->d_m, a.Z = 1, a.alpha = 1.f;
        gemm(p, a, st);
        launch_mha_decode(p->dtype, Q, Kc, Vc, n_per_input, B, x, p->h, p->d_k, n,
                          float(1.0 / std::sqrt(double(p->d_k))), ctx, st);
        o_projection(p, ctx, R, out, st);  // sum_i ctx_i . W_O,i + b_O (attention.hpp:111-113)
    });
}

// ---------------------------------------------------------------- beam-search candidates
extern "C" int elattn_gpu_beam_candidates(const float* lprobs, const float* live_lp, const float* penalty, int B,
                                          int lanes, int roots, int V, int k, int* parent, int* token, float* lp_sum,
                                          elattn_stream_t stream) {
    return guarded([&] {
        ELA_REQUIRE(lprobs && live_lp && parent && token && lp_sum, ELATTN_ERR_PARAM, "beam_candidates: null buffer");
        ELA_REQUIRE(B >= 1, ELATTN_ERR_SHAPE, "beam_candidates: B must be >= 1");
        ELA_REQUIRE(k >= 1, ELATTN_ERR_PARAM, "beam_candidates: k must be >= 1");
        ELA_REQUIRE(k <= 32, ELATTN_ERR_UNSUPPORTED, "beam_candidates: k <= 32 (2 x beam for beam <= 16)");
        ELA_REQUIRE(V >= 1, ELATTN_ERR_SHAPE, "beam_candidates: V must be >= 1");
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        const int splits = beam_splits(B, V);
        const size_t part_bytes = sizeof(uint64_t) * size_t(B) * splits * k;
        Scratch ws(nullptr, 0, align256(part_bytes), st);
        auto* part = static_cast<uint64_t*>(ws.take(part_bytes));
        launch_beam_topk(lprobs, live_lp, penalty, B, lanes, roots, V, k, part, splits, parent, token, lp_sum, st);
    });
}

// ---------------------------------------------------------------- whole-lane gather
extern "C" int elattn_gpu_lane_gather(const void* src, void* dst, const int* parent, int lanes_in, int lanes_out,
                                      int64_t bytes_per_lane, elattn_stream_t stream) {
    return guarded([&] {
        ELA_REQUIRE(src && dst && parent, ELATTN_ERR_PARAM, "lane_gather: null buffer");
        ELA_REQUIRE(src != dst, ELATTN_ERR_PARAM, "lane_gather: src and dst must differ");
        ELA_REQUIRE(lanes_in >= 1 && lanes_out >= 1, ELATTN_ERR_SHAPE, "lane_gather: bad lane counts");
        launch_lane_gather(src, dst, parent, lanes_in, lanes_out, bytes_per_lane, reinterpret_cast<cudaStream_t>(stream));
    });
}
