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
//   fork   : the same reorder over SLOT-INDEXED caches ([layers][slots][n_max][d_m] plus a
//            lane -> slot map, read by the decode through its h_index): the first new lane
//            with a given parent takes over the parent's slot, only further children of that
//            parent get a free slot and a copy — a permutation (or keep_lanes) copies nothing,
//            a beam reorder copies one history per duplicated parent instead of every lane.
#include "common.cuh"
#include "kernels.h"

namespace elattn_gpu {

namespace {

template <typename V>
__global__ void cache_append_kernel(V* __restrict__ cache, const V* __restrict__ Y, int* __restrict__ len,
                                    int n_max, int vec_per_row, const int* __restrict__ lane_slot) {
    const int lane = blockIdx.x;
    const int slot = lane_slot ? lane_slot[lane] : lane;
    const int t = len[lane];
    __syncthreads();  // every thread read len before thread 0 updates it
    if (t < 0 || t >= n_max) {
        if (threadIdx.x == 0) len[lane] = n_max + 1;  // out of contract: loud NaN rows downstream
        return;
    }
    V* dst = cache + (int64_t(slot) * n_max + t) * vec_per_row;
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

// Exclusive block-wide prefix count of `flag` over the CTA (blockDim a multiple of 32,
// <= 1024); returns the prefix and leaves the block total in *total.
__device__ int block_scan_flag(bool flag, int* s_warp, int* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const unsigned m = __ballot_sync(0xffffffffu, flag);
    __syncthreads();  // s_warp reuse across calls
    if (lane == 0) s_warp[w] = __popc(m);
    __syncthreads();
    int before = 0, all = 0;
    for (int i = 0; i < nw; ++i) {
        const int c = s_warp[i];
        before += i < w ? c : 0;
        all += c;
    }
    *total = all;
    return before + __popc(m & ((1u << lane) - 1u));
}

// Fork plan (one CTA): slot_out[i], lengths_out[l][i] = lengths_in[l][parent[i]] for every
// layer, and the compacted copy orders {src slot, dst slot, parent} (count in *ncopy).
// ws: claimed[slots], first[lanes_in], freelist[slots].
__global__ void __launch_bounds__(1024) cache_fork_plan_kernel(
    const int* __restrict__ slot_in, int* __restrict__ slot_out, const int* __restrict__ parent, int lanes_in,
    int lanes_out, int slots, int layers, int n_max, const int* __restrict__ len_in, int* __restrict__ len_out,
    int4* __restrict__ copies, int* __restrict__ ncopy, int* __restrict__ claimed, int* __restrict__ first,
    int* __restrict__ freelist) {
    __shared__ int s_warp[32];
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int s = tid; s < slots; s += nt) claimed[s] = 0;
    for (int p = tid; p < lanes_in; p += nt) first[p] = 0x7fffffff;
    __syncthreads();
    for (int i = tid; i < lanes_out; i += nt) {
        const int p = parent[i];
        if (p >= 0 && p < lanes_in) atomicMin(&first[p], i);
    }
    __syncthreads();
    for (int i = tid; i < lanes_out; i += nt) {  // first child of a parent: keeps the parent's slot
        const int p = parent[i];
        if (p >= 0 && p < lanes_in && first[p] == i) claimed[slot_in[p]] = 1;
    }
    __syncthreads();
    int nfree = 0;  // free slots in increasing order
    for (int base = 0; base < slots; base += nt) {
        const int s = base + tid;
        const bool f = s < slots && claimed[s] == 0;
        int tot;
        const int k = block_scan_flag(f, s_warp, &tot);
        if (f) freelist[nfree + k] = s;
        nfree += tot;
    }
    __syncthreads();
    int used = 0, ncp = 0;  // lanes needing a slot take free slots in lane order
    for (int base = 0; base < lanes_out; base += nt) {
        const int i = base + tid;
        const int p = i < lanes_out ? parent[i] : -1;
        const bool ok = p >= 0 && p < lanes_in;
        const bool owner = i < lanes_out && ok && first[p] == i;
        const bool need = i < lanes_out && !owner;
        int tot, ctot;
        const int k = block_scan_flag(need, s_warp, &tot);
        const int kc = block_scan_flag(need && ok, s_warp, &ctot);  // a copy (valid parent, new slot)
        if (i < lanes_out) {
            const int dst = owner ? slot_in[p] : freelist[used + k];  // lanes_out <= slots: always a free slot
            slot_out[i] = dst;
            if (need && ok) copies[ncp + kc] = make_int4(slot_in[p], dst, p, 0);
            for (int l = 0; l < layers; ++l)
                len_out[int64_t(l) * lanes_out + i] = ok ? len_in[int64_t(l) * lanes_in + p] : n_max + 1;
        }
        used += tot;
        ncp += ctot;
    }
    if (tid == 0) *ncopy = ncp;
}

// Copy the forked histories: block (part c, order k, layer l) streams part c of rows
// 0..len-1 of the parent's slot into the new slot for compacted copy order k < *ncopy
// (blocks past the device-side count return at once: a permutation copies nothing).
__global__ void __launch_bounds__(256) cache_fork_copy_kernel(uint4* __restrict__ cache, const int4* __restrict__ copies,
                                                              const int* __restrict__ ncopy,
                                                              const int* __restrict__ len_in, int lanes_in, int slots,
                                                              int n_max, int vec_per_row) {
    if (int(blockIdx.y) >= *ncopy) return;
    const int4 c = copies[blockIdx.y];
    const int l = blockIdx.z;
    const int rows = min(max(len_in[int64_t(l) * lanes_in + c.z], 0), n_max);
    const int64_t count = int64_t(rows) * vec_per_row;
    uint4* layer = cache + int64_t(l) * slots * n_max * vec_per_row;
    const uint4* s = layer + int64_t(c.x) * n_max * vec_per_row;
    uint4* d = layer + int64_t(c.y) * n_max * vec_per_row;
    // four 16-byte loads in flight per thread (the copy is bound by bytes in flight)
    const int64_t step = int64_t(gridDim.x) * blockDim.x;
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + 3 * step < count; i += 4 * step) {
        const uint4 v0 = s[i], v1 = s[i + step], v2 = s[i + 2 * step], v3 = s[i + 3 * step];
        d[i] = v0, d[i + step] = v1, d[i + 2 * step] = v2, d[i + 3 * step] = v3;
    }
    for (; i < count; i += step) d[i] = s[i];
}

}  // namespace

size_t cache_fork_workspace(int slots, int lanes_in, int lanes_out) {
    return sizeof(int4) * size_t(lanes_out) + sizeof(int) * (2 * size_t(slots) + size_t(lanes_in) + 4) + 64;
}

void launch_cache_fork(void* cache, int layers, int slots, int n_max, int d_m, int dtype, const int* len_in,
                       int* len_out, const int* slot_in, int* slot_out, const int* parent, int lanes_in, int lanes_out,
                       int rows_hint, void* ws, size_t ws_bytes, cudaStream_t st) {
    const size_t row_bytes = size_t(d_m) * dtype_bytes(dtype);
    ELA_REQUIRE(row_bytes % 16 == 0, ELATTN_ERR_SHAPE, "cache_fork: d_m * sizeof(dtype) must be a multiple of 16");
    ELA_REQUIRE(lanes_out <= slots, ELATTN_ERR_SHAPE, "cache_fork: more lanes than cache slots");
    ELA_REQUIRE(ws != nullptr && ws_bytes >= cache_fork_workspace(slots, lanes_in, lanes_out), ELATTN_ERR_PARAM,
                "cache_fork: workspace too small");
    ELA_REQUIRE((reinterpret_cast<uintptr_t>(ws) & 15) == 0, ELATTN_ERR_PARAM, "cache_fork: workspace alignment");
    int4* copies = static_cast<int4*>(ws);
    int* ncopy = reinterpret_cast<int*>(copies + lanes_out);
    int* claimed = ncopy + 4;
    int* first = claimed + slots;
    int* freelist = first + lanes_in;
    const int threads = std::min(1024, std::max(32, ((std::max(slots, lanes_out) + 31) / 32) * 32));
    cache_fork_plan_kernel<<<1, threads, 0, st>>>(slot_in, slot_out, parent, lanes_in, lanes_out, slots, layers, n_max,
                                                  len_in, len_out, copies, ncopy, claimed, first, freelist);
    ELA_CHECK_LAUNCH();
    const int vec = int(row_bytes / 16);
    // parts per history: enough 256-thread blocks (4 loads in flight each) for rows_hint rows
    const int64_t per_lane = int64_t(std::max(1, rows_hint)) * vec;
    const int parts = int(std::min<int64_t>(16, (per_lane + 16383) / 16384));
    cache_fork_copy_kernel<<<dim3(parts, lanes_out, layers), 256, 0, st>>>(static_cast<uint4*>(cache), copies, ncopy,
                                                                             len_in, lanes_in, slots, n_max, vec);
    ELA_CHECK_LAUNCH();
}

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
                         cudaStream_t st, const int* lane_slot) {
    const size_t row_bytes = size_t(d_m) * dtype_bytes(dtype);
    ELA_REQUIRE(row_bytes % 16 == 0, ELATTN_ERR_SHAPE, "cache_append: d_m * sizeof(dtype) must be a multiple of 16");
    cache_append_kernel<uint4><<<lanes, 128, 0, st>>>(static_cast<uint4*>(cache), static_cast<const uint4*>(Y), len,
                                                      n_max, int(row_bytes / 16), lane_slot);
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
