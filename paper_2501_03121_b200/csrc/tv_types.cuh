// Element types, bit-exact promote/demote and streaming loads shared by every
// kernel of libtenvec_b200.so.
//
// Semantics follow the reference precision module (pkg/src/tenvec/precision.py):
//   promote  (precision.py:109-115) is exact: bf16 bits << 16, half -> float,
//            float -> double;
//   demote   (precision.py:118-128): double -> float and float -> half round to
//            nearest even (half overflow -> +-inf, no saturation), brain is the
//            binary32 pattern shifted right by 16 (truncation, NOT
//            __float2bfloat16_rn), after an RNE double -> float step.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tenvec_b200.h"

namespace tv {

template <int SD>
struct St;
template <>
struct St<TV_F64> {
  using T = double;
};
template <>
struct St<TV_F32> {
  using T = float;
};
template <>
struct St<TV_F16> {
  using T = uint16_t;
};
template <>
struct St<TV_BF16> {
  using T = uint16_t;
};

// elements per 16-byte vector
template <int SD>
struct VecN {
  static constexpr int N = 16 / sizeof(typename St<SD>::T);
};

template <int SD, typename C>
__device__ __forceinline__ C promote(typename St<SD>::T v);

template <>
__device__ __forceinline__ double promote<TV_F64, double>(double v) { return v; }
template <>
__device__ __forceinline__ float promote<TV_F32, float>(float v) { return v; }
template <>
__device__ __forceinline__ double promote<TV_F32, double>(float v) { return (double)v; }
template <>
__device__ __forceinline__ float promote<TV_F16, float>(uint16_t v) {
  return __half2float(__ushort_as_half(v));
}
template <>
__device__ __forceinline__ float promote<TV_BF16, float>(uint16_t v) {
  return __uint_as_float(((uint32_t)v) << 16);
}

template <int SD, typename C>
__device__ __forceinline__ typename St<SD>::T demote(C v);

template <>
__device__ __forceinline__ double demote<TV_F64, double>(double v) { return v; }
template <>
__device__ __forceinline__ float demote<TV_F32, float>(float v) { return v; }
template <>
__device__ __forceinline__ float demote<TV_F32, double>(double v) { return __double2float_rn(v); }
template <>
__device__ __forceinline__ uint16_t demote<TV_F16, float>(float v) {
  return __half_as_ushort(__float2half_rn(v));
}
template <>
__device__ __forceinline__ uint16_t demote<TV_BF16, float>(float v) {
  return (uint16_t)(__float_as_uint(v) >> 16);
}

// non-contracted arithmetic for the alpha/beta epilogue: the reference computes
// al * dot, then += be * y, each rounded separately (kernels.py:113-118)
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }

// 16-byte streaming load: read-only path, no L1 allocation, 256B L2 prefetch.
// Programmatic dependent launch (tv_tvc_sweep): every TVC kernel lets the
// next grid of the stream launch as soon as all of its CTAs are resident
// (griddepcontrol.launch_dependents at entry) and, before exiting, waits for
// the grids it was launched after (griddepcontrol.wait) -- so a PDL-launched
// mode overlaps the previous mode's tail but still completes after it, and
// stream order holds for whatever follows.  Both are no-ops in a plain launch.
struct PdlScope {
  __device__ __forceinline__ PdlScope() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
  __device__ __forceinline__ ~PdlScope() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
};

__device__ __forceinline__ uint4 ld_stream16(const void* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}

// one streamed element (lane-interleaved scalar loads of unaligned views).
// volatile keeps a batch of these in issue order: without it the compiler
// sinks each load next to its FMA and only one load per lane is in flight.
__device__ __forceinline__ double ld_stream_elem(const double* p) {
  double r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ float ld_stream_elem(const float* p) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ uint16_t ld_stream_elem(const uint16_t* p) {
  uint16_t r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.u16 %0, [%1];" : "=h"(r) : "l"(p));
  return r;
}

template <int SD>
union Pack16 {
  uint4 u;
  typename St<SD>::T e[VecN<SD>::N];
};

template <int SD, typename C>
__device__ __forceinline__ void unpack(const uint4& raw, C (&out)[VecN<SD>::N]) {
  Pack16<SD> p;
  p.u = raw;
#pragma unroll
  for (int e = 0; e < VecN<SD>::N; ++e) out[e] = promote<SD, C>(p.e[e]);
}

// y = demote(alpha * acc [+ beta * promote(y_old)])
template <int SD, typename C>
__device__ __forceinline__ typename St<SD>::T epilogue(C acc, C alpha, C beta, bool has_beta,
                                                       const typename St<SD>::T* yold) {
  C r = mul_rn(alpha, acc);
  if (has_beta) r = add_rn(r, mul_rn(beta, promote<SD, C>(*yold)));
  return demote<SD, C>(r);
}

}  // namespace tv
