// The normalisation tree of tv_norm2 / tv_normalize (kernels.py:234-254),
// shared by k_norm (util.cu) and the TVC + normalize epilogue (tvc.cu) so both
// produce the same bits: one CTA of 1024 threads, per-thread strided FMA
// partials in the compute type, an xor-shuffle within each warp, then warp 0
// over the 32 warp partials, sqrt, and x <- demote(promote(x) / norm).  Every
// rank that holds the same vector computes the same bits (hopm.py:339-342).
#pragma once

#include "tv_types.cuh"

namespace tv {

constexpr int kNormThreads = 1024;

template <typename T>
__device__ __forceinline__ T ld_l2(const T* p) {  // bypass L1: data written by other CTAs
  return __ldcg(p);
}

// CG: read x through L2 only (x was just written by other CTAs of this grid)
template <int SD, typename C, bool CG>
__device__ __forceinline__ void norm_block(typename St<SD>::T* x, int64_t n, double* norm_out,
                                           int32_t* status, int do_scale) {
  __shared__ C part[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  C s = C(0);
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const C c = promote<SD, C>(CG ? ld_l2(x + i) : x[i]);
    s = fma(c, c, s);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) part[w] = s;
  __syncthreads();
  if (w == 0) {
    s = lane < (int)(blockDim.x >> 5) ? part[lane] : C(0);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) part[0] = s;
  }
  __syncthreads();
  const C nrm = sqrt(part[0]);
  if (threadIdx.x == 0) {
    norm_out[0] = (double)nrm;
    if (status) status[0] = (nrm == C(0)) ? TV_ENORM : TV_OK;
  }
  if (do_scale && nrm != C(0)) {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
      x[i] = demote<SD, C>(promote<SD, C>(CG ? ld_l2(x + i) : x[i]) / nrm);
  }
}

}  // namespace tv
