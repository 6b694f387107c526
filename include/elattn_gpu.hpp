// elattn_gpu.hpp — C++ drop-in for the reference's EL-attention entry points.
//
// Same names, signatures, argument meaning and exception types as
// /root/reference/proj/include/elattn/attention.hpp, in namespace elattn::gpu:
//
//   elattn::build_el_query(q, p)                          attention.hpp:197-215
//   elattn::fold_el_queries(queries, h, d_m)              attention.hpp:293-304
//   elattn::el_attention(q, H, p)                         attention.hpp:239-257
//   elattn::el_attention_folded(queries, H, s, p)         attention.hpp:262-290
//   elattn::mixed_self_attention(q, prefix, cache, p)     attention.hpp:309-365
//   elattn::multi_head_attention(q, H, p)                 attention.hpp:96-113 (GPU MHA baseline:
//                                                         K/V caches + attention over them)
//
// plus DecoderStep (the batched, graph-captured decoder step over L layers that replaces
// the per-lane loop of model.hpp:357-385) for device-resident decode loops.
//
// A reference caller switches by changing the namespace (optionally passing a
// Dtype; the default, f32, meets the 1e-5 parity gate).  The arithmetic runs in
// libelattn_gpu.so through the C ABI of elattn_gpu.h; this header only converts
// the reference's fp64 Tensors to device buffers and back.  For decode loops, keep
// weights and H resident with DeviceParams + ElAttentionLayer (no per-call upload).
//
// Requires the reference's headers on the include path (elattn/attention.hpp) —
// they define Tensor, AttentionParams, ElQuery and the error types — and links
// against libelattn_gpu.so and the CUDA runtime.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "elattn/attention.hpp"
#include "elattn_gpu.h"

namespace elattn {
namespace gpu {

enum class Dtype { f32 = ELATTN_DTYPE_F32, bf16 = ELATTN_DTYPE_BF16 };

// Status -> the reference's exception types (errors.hpp).
inline void check(int rc) {
    if (rc == ELATTN_OK) return;
    const std::string msg = elattn_gpu_last_error_message();
    switch (rc) {
        case ELATTN_ERR_SHAPE: throw ShapeError(msg);
        case ELATTN_ERR_PARAM: throw ParamError(msg);
        case ELATTN_ERR_STATE: throw StateError(msg);
        case ELATTN_ERR_NUMERIC: throw NumericError(msg);
        default: throw std::runtime_error("elattn_gpu: " + msg);
    }
}

inline void check_cuda(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}

namespace detail {

inline uint16_t to_bf16(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return uint16_t((u >> 16) | 0x40);
    u += 0x7fffu + ((u >> 16) & 1u);
    return uint16_t(u >> 16);
}
inline float from_bf16(uint16_t h) {
    uint32_t u = uint32_t(h) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

// Device buffer of `count` elements of the params dtype.
class DeviceBuffer {
   public:
    DeviceBuffer(size_t count, Dtype dt) : count_(count), dt_(dt) {
        check_cuda(cudaMalloc(&ptr_, bytes() ? bytes() : 1));
    }
    ~DeviceBuffer() { cudaFree(ptr_); }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    size_t bytes() const { return count_ * (dt_ == Dtype::bf16 ? 2 : 4); }
    void* get() const { return ptr_; }
    void upload(const double* src) {
        if (dt_ == Dtype::bf16) {
            std::vector<uint16_t> h(count_);
            for (size_t i = 0; i < count_; ++i) h[i] = to_bf16(float(src[i]));
            check_cuda(cudaMemcpy(ptr_, h.data(), bytes(), cudaMemcpyHostToDevice));
        } else {
            std::vector<float> h(src, src + count_);
            check_cuda(cudaMemcpy(ptr_, h.data(), bytes(), cudaMemcpyHostToDevice));
        }
    }
    void download(double* dst) const {
        if (dt_ == Dtype::bf16) {
            std::vector<uint16_t> h(count_);
            check_cuda(cudaMemcpy(h.data(), ptr_, bytes(), cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < count_; ++i) dst[i] = from_bf16(h[i]);
        } else {
            std::vector<float> h(count_);
            check_cuda(cudaMemcpy(h.data(), ptr_, bytes(), cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < count_; ++i) dst[i] = h[i];
        }
    }

   private:
    void* ptr_ = nullptr;
    size_t count_;
    Dtype dt_;
};

}  // namespace detail

// AttentionParams packed once on the device (elattn_gpu_params_t, RAII).
class DeviceParams {
   public:
    DeviceParams(const AttentionParams& p, Dtype dt = Dtype::f32) : h_(p.h), d_m(p.d_m), d_k(p.d_k), dt_(dt) {
        p.validate();  // attention.hpp:24-50
        const size_t mk = size_t(p.d_m) * p.d_k;
        std::vector<double> Wq, Wk, Wv, Wo, bq, bk, bv;
        for (int i = 0; i < p.h; ++i) {
            auto app = [](std::vector<double>& dst, const Tensor& t) {
                dst.insert(dst.end(), t.data().begin(), t.data().end());
            };
            app(Wq, p.Wq[i]), app(Wk, p.Wk[i]), app(Wv, p.Wv[i]), app(Wo, p.Wo[i]);
            app(bq, p.bq[i]), app(bk, p.bk[i]), app(bv, p.bv[i]);
        }
        (void)mk;
        check(elattn_gpu_params_create(p.h, p.d_m, p.d_k, int(dt), p.include_key_bias, p.include_value_bias,
                                       Wq.data(), Wk.data(), Wv.data(), Wo.data(), bq.data(), bk.data(), bv.data(),
                                       p.bo.data().data(), &handle_));
    }
    ~DeviceParams() {
        if (handle_) elattn_gpu_params_destroy(handle_);
    }
    DeviceParams(const DeviceParams&) = delete;
    DeviceParams& operator=(const DeviceParams&) = delete;
    elattn_gpu_params_t handle() const { return handle_; }
    Dtype dtype() const { return dt_; }
    int h() const { return h_; }
    int d_m, d_k;

   private:
    int h_;
    Dtype dt_;
    elattn_gpu_params_t handle_ = nullptr;
};

// build_el_query (attention.hpp:197-215).
inline ElQuery build_el_query(const Tensor& q, const DeviceParams& dp) {
    if (q.rows() != 1 || q.cols() != dp.d_m) throw ShapeError("build_el_query: q must be 1 x d_m");
    detail::DeviceBuffer dq(size_t(dp.d_m), dp.dtype()), dqp(size_t(dp.h()) * dp.d_m, dp.dtype());
    float* ds = nullptr;
    check_cuda(cudaMalloc(&ds, sizeof(float) * size_t(dp.h())));
    std::unique_ptr<float, void (*)(float*)> guard(ds, [](float* p) { cudaFree(p); });
    dq.upload(q.data().data());
    check(elattn_gpu_build_el_query(dp.handle(), dq.get(), 1, dqp.get(), ds, nullptr, 0, nullptr));
    check_cuda(cudaDeviceSynchronize());
    ElQuery eq;
    eq.elq = Tensor({dp.h(), dp.d_m});
    dqp.download(eq.elq.data().data());
    std::vector<float> s(size_t(dp.h()));
    check_cuda(cudaMemcpy(s.data(), ds, sizeof(float) * s.size(), cudaMemcpyDeviceToHost));
    eq.s.assign(s.begin(), s.end());
    return eq;
}
inline ElQuery build_el_query(const Tensor& q, const AttentionParams& p, Dtype dt = Dtype::f32) {
    DeviceParams dp(p, dt);
    return build_el_query(q, dp);
}

// fold_el_queries (attention.hpp:293-304): host bookkeeping only — query b's head i goes to
// row b*h + i of the folded [(g*h) x d_m] matrix, its key-bias scalar to entry b*h + i.
inline std::pair<Tensor, Tensor> fold_el_queries(const std::vector<ElQuery>& queries, int h, int d_m) {
    const int64_t g = static_cast<int64_t>(queries.size());
    Tensor q({g * h, static_cast<int64_t>(d_m)});
    Tensor s({g * h});
    for (int64_t b = 0; b < g; ++b) {
        const ElQuery& eq = queries[static_cast<size_t>(b)];
        for (int i = 0; i < h; ++i) {
            for (int64_t j = 0; j < d_m; ++j) q.at(b * h + i, j) = eq.elq.at(i, j);
            s.at(b * h + i) = eq.s[static_cast<size_t>(i)];
        }
    }
    return {q, s};
}

// el_attention_folded (attention.hpp:262-290).
inline Tensor el_attention_folded(const Tensor& queries, const Tensor& H, const Tensor& bias_scalars,
                                  const DeviceParams& dp) {
    const int h = dp.h();
    if (queries.rows() % h != 0)
        throw ShapeError("el_attention_folded: query row count " + std::to_string(queries.rows()) +
                         " not divisible by h=" + std::to_string(h));
    if (bias_scalars.size() != queries.rows())
        throw ShapeError("el_attention_folded: bias scalar count must equal query rows");
    if (H.empty() || H.rows() < 1) throw StateError("el_attention_folded: empty context");
    if (queries.cols() != dp.d_m || H.cols() != dp.d_m) throw ShapeError("el_attention_folded: width must equal d_m");
    const int g = int(queries.rows() / h), n = int(H.rows());
    detail::DeviceBuffer dq(size_t(queries.size()), dp.dtype()), dH(size_t(H.size()), dp.dtype()),
        dout(size_t(g) * dp.d_m, dp.dtype());
    dq.upload(queries.data().data());
    dH.upload(H.data().data());
    check(elattn_gpu_el_attention_folded(dp.handle(), dq.get(), nullptr, dH.get(), nullptr, 1, g, n, dout.get(),
                                         nullptr, 0, nullptr));
    check_cuda(cudaDeviceSynchronize());
    Tensor out({g, dp.d_m});
    dout.download(out.data().data());
    return out;
}
inline Tensor el_attention_folded(const Tensor& queries, const Tensor& H, const Tensor& bias_scalars,
                                  const AttentionParams& p, Dtype dt = Dtype::f32) {
    p.validate();
    DeviceParams dp(p, dt);
    return el_attention_folded(queries, H, bias_scalars, dp);
}

// el_attention (attention.hpp:239-257): query expansion + fused decode + projection.  One
// query row, as in the reference (build_el_query's check, :199-200); batches of rows and
// inputs go through el_attention_step / DecoderStep.
inline Tensor el_attention(const Tensor& q, const Tensor& H, const DeviceParams& dp) {
    if (H.empty() || H.rows() < 1) throw StateError("el_attention: empty context");
    if (q.cols() != dp.d_m || H.cols() != dp.d_m) throw ShapeError("el_attention: q/H width must equal d_m");
    if (q.rows() != 1) throw ShapeError("build_el_query: q must be 1 x d_m");
    const int x = int(q.rows()), n = int(H.rows());
    detail::DeviceBuffer dq(size_t(q.size()), dp.dtype()), dH(size_t(H.size()), dp.dtype()),
        dout(size_t(x) * dp.d_m, dp.dtype());
    dq.upload(q.data().data());
    dH.upload(H.data().data());
    check(elattn_gpu_el_attention_step(dp.handle(), dq.get(), dH.get(), nullptr, 1, x, n, dout.get(), nullptr, 0,
                                       nullptr));
    check_cuda(cudaDeviceSynchronize());
    Tensor out({x, dp.d_m});
    dout.download(out.data().data());
    return out;
}
inline Tensor el_attention(const Tensor& q, const Tensor& H, const AttentionParams& p, Dtype dt = Dtype::f32) {
    p.validate();
    DeviceParams dp(p, dt);
    return el_attention(q, H, dp);
}

// multi_head_attention (attention.hpp:96-113) on the GPU MHA path: the per-head K/V of H
// are projected once into device caches (elattn_gpu_mha_kv_build), then the g query rows
// attend over them in chunks of 16 (elattn_gpu_mha_attention).
inline Tensor multi_head_attention(const Tensor& q, const Tensor& H, const DeviceParams& dp) {
    if (q.cols() != dp.d_m || H.cols() != dp.d_m) throw ShapeError("multi_head_attention: q/H width must equal d_m");
    if (H.empty() || H.rows() < 1) throw StateError("multi_head_attention: empty context");
    const int g = int(q.rows()), n = int(H.rows());
    const size_t cache = size_t(dp.h()) * n * dp.d_k;
    detail::DeviceBuffer dH(size_t(H.size()), dp.dtype()), dK(cache, dp.dtype()), dV(cache, dp.dtype()),
        dq(size_t(q.size()) ? size_t(q.size()) : 1, dp.dtype()), dout(size_t(g) * dp.d_m ? size_t(g) * dp.d_m : 1, dp.dtype());
    dH.upload(H.data().data());
    check(elattn_gpu_mha_kv_build(dp.handle(), dH.get(), 1, n, dK.get(), dV.get(), nullptr));
    if (g > 0) dq.upload(q.data().data());
    const size_t e = dp.dtype() == Dtype::bf16 ? 2 : 4;
    for (int r = 0; r < g; r += 16) {
        const int x = g - r < 16 ? g - r : 16;
        check(elattn_gpu_mha_attention(dp.handle(), static_cast<const char*>(dq.get()) + size_t(r) * dp.d_m * e,
                                       dK.get(), dV.get(), nullptr, 1, x, n,
                                       static_cast<char*>(dout.get()) + size_t(r) * dp.d_m * e, nullptr, 0, nullptr));
    }
    check_cuda(cudaDeviceSynchronize());
    Tensor out({g, dp.d_m});
    if (g > 0) dout.download(out.data().data());
    return out;
}
inline Tensor multi_head_attention(const Tensor& q, const Tensor& H, const AttentionParams& p, Dtype dt = Dtype::f32) {
    p.validate();
    DeviceParams dp(p, dt);
    return multi_head_attention(q, H, dp);
}

// Device-resident batched sub-layer for decode loops (the caller keeps H and
// the weights in HBM; stream-ordered, no host round trip):
//   Y [B*x][d_m], H [B][n][d_m] -> out [B*x][d_m], all device pointers of dp.dtype().
inline void el_attention_step(const DeviceParams& dp, const void* Y, const void* H, const int* n_per_input, int B,
                              int x, int n, void* out, cudaStream_t stream = nullptr, void* workspace = nullptr,
                              size_t workspace_bytes = 0) {
    check(elattn_gpu_el_attention_step(dp.handle(), Y, H, n_per_input, B, x, n, out, workspace, workspace_bytes,
                                       reinterpret_cast<elattn_stream_t>(stream)));
}

// mixed_self_attention (attention.hpp:309-365): the reference's KvCache is uploaded as the
// generated-token cache [1][h][t][d_k] of elattn_gpu_mixed_self_attention.
inline Tensor mixed_self_attention(const Tensor& q, const Tensor& prefix_hidden, const KvCache& gen_cache,
                                   const DeviceParams& dp) {
    if (prefix_hidden.empty() || prefix_hidden.rows() < 1) throw StateError("mixed_self_attention: empty prefix");
    if (gen_cache.t > 0 && (gen_cache.h != dp.h() || gen_cache.d_k != dp.d_k))
        throw StateError("mixed_self_attention: cache does not match params");
    if (q.rows() != 1 || q.cols() != dp.d_m || prefix_hidden.cols() != dp.d_m)
        throw ShapeError("mixed_self_attention: q/prefix width must equal d_m");
    const int t = int(gen_cache.t), t_max = t > 0 ? t : 1, n = int(prefix_hidden.rows());
    std::vector<double> K(size_t(dp.h()) * t_max * dp.d_k, 0.0), V(K.size(), 0.0);
    for (int i = 0; i < dp.h() && t > 0; ++i)
        for (size_t j = 0; j < size_t(t) * dp.d_k; ++j) {
            K[size_t(i) * t_max * dp.d_k + j] = gen_cache.K[size_t(i)][j];
            V[size_t(i) * t_max * dp.d_k + j] = gen_cache.V[size_t(i)][j];
        }
    detail::DeviceBuffer dq(size_t(dp.d_m), dp.dtype()), dP(size_t(prefix_hidden.size()), dp.dtype()),
        dK(K.size(), dp.dtype()), dV(V.size(), dp.dtype()), dout(size_t(dp.d_m), dp.dtype());
    dq.upload(q.data().data());
    dP.upload(prefix_hidden.data().data());
    dK.upload(K.data());
    dV.upload(V.data());
    check(elattn_gpu_mixed_self_attention(dp.handle(), dq.get(), dP.get(), nullptr, 1, 1, n, dK.get(), dV.get(),
                                          t_max, t, dout.get(), nullptr, 0, nullptr));
    check_cuda(cudaDeviceSynchronize());
    Tensor out({1, dp.d_m});
    dout.download(out.data().data());
    return out;
}
inline Tensor mixed_self_attention(const Tensor& q, const Tensor& prefix_hidden, const KvCache& gen_cache,
                                   const AttentionParams& p, Dtype dt = Dtype::f32) {
    p.validate();
    DeviceParams dp(p, dt);
    return mixed_self_attention(q, prefix_hidden, gen_cache, dp);
}

// Batched decoder step over L layers sharing one encoder state per input (RAII over
// elattn_gpu_decoder_*): bind device buffers once, then run() per step.
class DecoderStep {
   public:
    DecoderStep(const std::vector<const DeviceParams*>& layers, const void* H, const int* n_per_input, int B, int x,
                int n, const void* Y_in, void* out) {
        std::vector<elattn_gpu_params_t> hs;
        for (const DeviceParams* l : layers) hs.push_back(l->handle());
        check(elattn_gpu_decoder_create(hs.data(), int(hs.size()), H, n_per_input, B, x, n, Y_in, out, &dec_));
    }
    ~DecoderStep() {
        if (dec_) elattn_gpu_decoder_destroy(dec_);
    }
    DecoderStep(const DecoderStep&) = delete;
    DecoderStep& operator=(const DecoderStep&) = delete;
    void run(cudaStream_t stream = nullptr) { check(elattn_gpu_decoder_run(dec_, reinterpret_cast<elattn_stream_t>(stream))); }

   private:
    elattn_gpu_decoder_t dec_ = nullptr;
};

}  // namespace gpu
}  // namespace elattn
