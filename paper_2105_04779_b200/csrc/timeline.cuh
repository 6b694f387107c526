// timeline.cuh — in-graph step timeline (measurement builds only).
//
// Built with `make EXTRA=-DELA_TIMELINE BUILD=build_tl LIB=...`, every CTA of the step's
// kernels (projection GEMMs, fused query expansion, decode, merge) appends one record
// {kind, block, %globaltimer at entry, after the programmatic-dependent-launch wait, at
// exit} to a device buffer.  tools/step_timeline.py reads it after replaying a decoder-step
// graph: launch gaps, PDL overlap, per-kernel startup and tails, without a profiler (ncu
// serialises the kernels and so hides exactly these).  The production build compiles the
// macros to nothing.
#pragma once
#include "ptx_sm100.cuh"

namespace elattn_gpu {

struct TlRec {
    unsigned long long entry, wait, exit, mark[4];  // mark: kernel-specific phase ends (0 = unset)
    unsigned kind, block;
};
enum TlKind : unsigned { kTlGemm = 1, kTlSplitK = 2, kTlQexp = 3, kTlDecode = 4, kTlMerge = 5 };

#ifdef ELA_TIMELINE
namespace {
__device__ TlRec* tl_buf_;
__device__ unsigned* tl_cnt_;
__device__ unsigned tl_cap_;
}  // namespace
#define ELA_TL_DECL                                                                 \
    unsigned long long tl_entry_ = ::elattn_gpu::ptx::globaltimer(), tl_wait_ = tl_entry_; \
    __shared__ unsigned long long tl_mark_[4];                                      \
    if (threadIdx.x < 4) tl_mark_[threadIdx.x] = 0
#define ELA_TL_WAIT() (tl_wait_ = ::elattn_gpu::ptx::globaltimer())
// any thread; read by thread 0 at exit (after the kernel's final CTA barrier)
#define ELA_TL_MARK(i) (tl_mark_[i] = ::elattn_gpu::ptx::globaltimer())
#define ELA_TL_EXIT(kind)                                                                             \
    do {                                                                                              \
        if (threadIdx.x == 0 && tl_buf_ != nullptr) {                                                 \
            const unsigned long long tl_exit_ = ::elattn_gpu::ptx::globaltimer(); /* before the atomic */ \
            const unsigned i_ = atomicAdd(tl_cnt_, 1u);                                               \
            if (i_ < tl_cap_)                                                                         \
                tl_buf_[i_] = ::elattn_gpu::TlRec{tl_entry_, tl_wait_, tl_exit_,                        \
                                                  {tl_mark_[0], tl_mark_[1], tl_mark_[2], tl_mark_[3]}, \
                                                  unsigned(kind),                                     \
                                                  blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)}; \
        }                                                                                             \
    } while (0)
#define ELA_TL_SETTER(name)                                                     \
    bool name(TlRec* buf, unsigned* cnt, unsigned cap) {                        \
        return cudaMemcpyToSymbol(tl_buf_, &buf, sizeof buf) == cudaSuccess &&  \
               cudaMemcpyToSymbol(tl_cnt_, &cnt, sizeof cnt) == cudaSuccess &&  \
               cudaMemcpyToSymbol(tl_cap_, &cap, sizeof cap) == cudaSuccess;    \
    }
#else
#define ELA_TL_DECL
#define ELA_TL_WAIT() ((void)0)
#define ELA_TL_MARK(i) ((void)0)
#define ELA_TL_EXIT(kind) ((void)0)
#define ELA_TL_SETTER(name) \
    bool name(TlRec*, unsigned*, unsigned) { return false; }
#endif

}  // namespace elattn_gpu
