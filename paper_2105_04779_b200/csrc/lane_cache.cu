// lane_cache.cu — per-lane hidden-state caches for decoder-only EL self-attention
// (BASELINE config 4, "hidden-state-only cache").
//
// In the decoder-only form each lane (beam) attends over its OWN history of layer inputs
// (the EL "El" is the sequence of hidden states; model.hpp:438-466 ingests a prefix
// causally, and every generated token's normalised input joins the same per-layer store).
// The GPU keeps, per layer, a cache [lanes][n_max][d_m] and a device length per lane; the
// attention itself is the batched EL step with x = 1 and n_per_input = the lengths.
//   append : cache[l][len[l]] = Y[l]; ++len[l]            (a full lane gets len = n_max + 1,
//            which the decode turns into loud NaN rows)
//   gather : DecoderState::gather_lanes (model.hpp:291-306) on the device — lane i of the
//            destination becomes a copy of source lane parent[i] (rows 0..len-1) — so beam
//            reordering never leaves the GPU (keep_lanes / permute_lanes, model.hpp:305-325,
//            are gathers with a subset / a permutation as the parent list).
//   lane_gather: the same for fixed-size per-lane state (K/V caches of the mixed form).
#include "common.cuh"
#include "kernels.h"

namespace elattn_gpu {

namespace {

template <typename V>
__global__ void cache_append_kernel(V* __restrict__ cache, const V* __restrict__ Y, int* __restrict__ len,
                                    int n_max, int vec_per_row) {
    const int lane = blockIdx.x;
    const int t = len[lane];
    __syncthreads();  // every thread read len before thread 0 updates it
    if (t < 0 || t >= n_max) {
        if (threadIdx.x == 0) len[lane] = n_max + 1;  // out of contract: loud NaN rows downstream
        return;
    }
    V* dst = cache + (int64_t(lane) * n_max + t) * vec_per_row;
    const V* src = Y + int64_t(lane) * vec_per_row;
    for (int i = threadIdx.x; i < vec_per_row; i += blockDim.x) dst[i] = src[i];
    if (threadIdx.x == 0) len[lane] = t + 1;
}

template <typename V>
__global__ void cache_gather_kernel(const V* __restrict__ src, const int* __restrict__ src_len, V* __restrict__ dst,
                                    int* __restrict__ dst_len, const int* __restrict__ parent, int lanes_in,
                                    int n_max, int vec_per_row) {
    const int lane = blockIdx.y;
    const int p = parent[lane];
    const bool ok = p >= 0 && p < lanes_in;
    const int rows = ok ? min(max(src_len[p], 0), n_max) : 0;
    const int64_t count = int64_t(rows) * vec_per_row;
    const V* s = src + int64_t(ok ? p : 0) * n_max * vec_per_row;
    V* d = dst + int64_t(lane) * n_max * vec_per_row;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x)
        d[i] = s[i];
    if (blockIdx.x == 0 && threadIdx.x == 0) dst_len[lane] = ok ? src_len[p] : n_max + 1;  // bad parent: loud
}

// Whole-lane gather for fixed-size per-lane state (the mixed self-attention's K/V caches,
// [R][h][t_max][d_k]): dst lane i = src lane parent[i]; a bad parent fills the lane with
// 0xFF bytes (NaN in fp32 and bf16 — loud).
__global__ void lane_gather_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                   const int* __restrict__ parent, int lanes_in, int64_t vec_per_lane) {
    const int lane = blockIdx.y;
    const int p = parent[lane];
    const bool ok = p >= 0 && p < lanes_in;
    const uint4* s = src + int64_t(ok ? p : 0) * vec_per_lane;
    uint4* d = dst + int64_t(lane) * vec_per_lane;
    const uint4 nan4 = make_uint4(~0u, ~0u, ~0u, ~0u);
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < vec_per_lane;
         i += int64_t(gridDim.x) * blockDim.x)
        d[i] = ok ? s[i] : nan4;
}

}  // namespace

void launch_lane_gather(const void* src, void* dst, const int* parent, int lanes_in, int lanes_out,
                        int64_t bytes_per_lane, cudaStream_t st) {
    ELA_REQUIRE(bytes_per_lane > 0 && bytes_per_lane % 16 == 0, ELATTN_ERR_SHAPE,
                "lane_gather: bytes per lane must be a positive multiple of 16");
    const int64_t vec = bytes_per_lane / 16;
    const int gx = int(std::min<int64_t>(64, (vec + 4095) / 4096));
    lane_gather_kernel<<<dim3(gx, lanes_out), 256, 0, st>>>(static_cast<const uint4*>(src), static_cast<uint4*>(dst),
                                                             parent, lanes_in, vec);
    ELA_CHECK_LAUNCH();
}

void launch_cache_append(void* cache, const void* Y, int* len, int lanes, int n_max, int d_m, int dtype,
                         cudaStream_t st) {
    const size_t row_bytes = size_t(d_m) * dtype_bytes(dtype);
    ELA_REQUIRE(row_bytes % 16 == 0, ELATTN_ERR_SHAPE, "cache_append: d_m * sizeof(dtype) must be a multiple of 16");
    cache_append_kernel<uint4><<<lanes, 128, 0, st>>>(static_cast<uint4*>(cache), static_cast<const uint4*>(Y), len,
                                                      n_max, int(row_bytes / 16));
    ELA_CHECK_LAUNCH();
}

void launch_cache_gather(const void* src, const int* src_len, void* dst, int* dst_len, const int* parent,
                         int lanes_in, int lanes_out, int n_max, int d_m, int dtype, int rows_hint,
                         cudaStream_t st) {
    const size_t row_bytes = size_t(d_m) * dtype_bytes(dtype);
    ELA_REQUIRE(row_bytes % 16 == 0, ELATTN_ERR_SHAPE, "cache_gather: d_m * sizeof(dtype) must be a multiple of 16");
    const int vec = int(row_bytes / 16);
    // enough CTAs per lane to stream rows_hint rows at full bandwidth
    const int64_t per_lane = int64_t(std::max(1, rows_hint)) * vec;
    const int gx = int(std::min<int64_t>(64, (per_lane + 4095) / 4096));
    cache_gather_kernel<uint4><<<dim3(gx, lanes_out), 256, 0, st>>>(
        static_cast<const uint4*>(src), src_len, static_cast<uint4*>(dst), dst_len, parent, lanes_in, n_max, vec);
    ELA_CHECK_LAUNCH();
}

}  // namespace elattn_gpu
