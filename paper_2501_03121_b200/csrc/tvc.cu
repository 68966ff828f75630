// Native mode-oblivious tensor-vector contraction (TVC) for sm_100a.
//
// Replaces the reference's tvc_native / getvc (pkg/src/tenvec/kernels.py:73-171):
// the order-d tensor is read through its (u, n_k, v) block view
// (tensor.py:85-102) -- u slabs of n_k x v, last index fastest -- so no mode
// ever needs an unfolding copy and every tensor byte is streamed from HBM
// exactly once.  The reference runs one BLAS matvec for k = d-1 and a Python
// loop of u BLAS vecmats otherwise; here one launch covers the whole view and
// the host picks one of five regimes from the view's shape:
//
//   ROWS       v == 1, rows of >= 8 16-byte vectors: G lanes per row (G in
//              {4,8,16,32}, chosen to minimise idle lanes), 128-bit loads,
//              x promoted once into shared memory, xor-shuffle row reduction.
//   ROWS_SHORT v == 1, rows of 1..7 vectors: lanes tile whole rows
//              (R = 32 / nkv rows per warp step), a segmented in-order
//              shuffle sum per row.
//   COLS       v >= 32 vectors: a CTA owns a 512-byte column stripe of one
//              slab; its 8 warps split the n_k rows round-robin, accumulate in
//              registers, and a fixed-order shared-memory reduction finishes.
//   SLABS      1 < v < 32 vectors: one warp streams a whole slab; R = 32 / vv
//              rows per step so every warp load is one contiguous run, then a
//              fixed-order cross-row reduction in shared memory.
//   GENERIC    anything not 16-byte aligned: scalar loads, same math.
//
// All regimes accumulate in the compute type, apply alpha after the dot
// product and beta * y after that (kernels.py:113-118), and demote once on
// store.  beta == 0 never reads y.  The reduction order of every output element
// depends only on (u, n_k, v, dtype): reruns and ranks reproduce bits.
// There are no tensor cores here: the arithmetic intensity is 0.25-1 FLOP/B.

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>

#include "tv_internal.h"
#include "tv_types.cuh"

namespace tv {

constexpr int kThreads = 256;

// ---------------------------------------------------------------- ROWS ----
template <int SD, typename C, int G, int UNR, bool XS>
__global__ void __launch_bounds__(kThreads)
    k_rows(const typename St<SD>::T* __restrict__ A, const typename St<SD>::T* __restrict__ x,
           typename St<SD>::T* __restrict__ y, int64_t u, int64_t nk, C alpha, C beta,
           int has_beta) {
  using T = typename St<SD>::T;
  constexpr int VEC = VecN<SD>::N;
  constexpr int RPW = 32 / G;  // rows per warp step
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* xs = reinterpret_cast<C*>(smem_raw);
  if (XS) {
    for (int64_t i = threadIdx.x; i < nk; i += blockDim.x) xs[i] = promote<SD, C>(x[i]);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int g = lane % G;
  const int rs = lane / G;
  const int64_t nkv = nk / VEC;
  const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  for (int64_t row0 = gw * RPW; row0 < u; row0 += warps_total * RPW) {
    const int64_t row = row0 + rs;
    C acc[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[e] = C(0);
    if (row < u) {
      const uint4* rp = reinterpret_cast<const uint4*>(A + row * nk);
      for (int64_t q0 = g; q0 < nkv; q0 += (int64_t)G * UNR) {
        uint4 buf[UNR];
#pragma unroll
        for (int t = 0; t < UNR; ++t) {
          const int64_t q = q0 + (int64_t)t * G;
          if (q < nkv) buf[t] = ld_stream16(rp + q);
        }
#pragma unroll
        for (int t = 0; t < UNR; ++t) {
          const int64_t q = q0 + (int64_t)t * G;
          if (q < nkv) {
            C a[VEC];
            unpack<SD, C>(buf[t], a);
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
              const C xv = XS ? xs[q * VEC + e] : promote<SD, C>(__ldg(x + q * VEC + e));
              acc[e] = fma(a[e], xv, acc[e]);
            }
          }
        }
      }
    }
    C s = acc[0];
#pragma unroll
    for (int e = 1; e < VEC; ++e) s += acc[e];
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (g == 0 && row < u) y[row] = epilogue<SD, C>(s, alpha, beta, has_beta != 0, y + row);
  }
}

// ---------------------------------------------------------- ROWS_SHORT ----
// rows of nkv in [1, 7] vectors; lanes (r = lane / nkv, c = lane % nkv)
template <int SD, typename C, int UNR>
__global__ void __launch_bounds__(kThreads)
    k_rows_short(const typename St<SD>::T* __restrict__ A, const typename St<SD>::T* __restrict__ x,
                 typename St<SD>::T* __restrict__ y, int64_t u, int nk, C alpha, C beta,
                 int has_beta) {
  constexpr int VEC = VecN<SD>::N;
  __shared__ C xs[8 * VEC];
  const int nkv = nk / VEC;
  for (int i = threadIdx.x; i < nk; i += blockDim.x) xs[i] = promote<SD, C>(x[i]);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int R = 32 / nkv;
  const int r = lane / nkv;
  const int c = lane - r * nkv;
  const bool active = r < R;
  const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t step = (int64_t)R * UNR;
  for (int64_t row0 = gw * step; row0 < u; row0 += warps_total * step) {
    uint4 buf[UNR];
#pragma unroll
    for (int t = 0; t < UNR; ++t) {
      const int64_t row = row0 + (int64_t)t * R + r;
      if (active && row < u) buf[t] = ld_stream16(A + row * nk + c * VEC);
    }
#pragma unroll
    for (int t = 0; t < UNR; ++t) {
      const int64_t row = row0 + (int64_t)t * R + r;
      C p = C(0);
      if (active && row < u) {
        C a[VEC];
        unpack<SD, C>(buf[t], a);
#pragma unroll
        for (int e = 0; e < VEC; ++e) p = fma(a[e], xs[c * VEC + e], p);
      }
      // in-order segmented sum over the nkv lanes of a row: ((p0 + p1) + p2) ...
      C s = p;
      for (int i = 1; i < nkv; ++i) {
        const C o = __shfl_down_sync(0xffffffffu, p, i);
        s += o;
      }
      if (active && c == 0 && row < u)
        y[row] = epilogue<SD, C>(s, alpha, beta, has_beta != 0, y + row);
    }
  }
}

// ---------------------------------------------------------------- COLS ----
// CTA = 8 warps over a 32-vector column stripe of slab i; warp w sums rows
// j = w, w + 8, ...; smem reduction over w in ascending order.
template <int SD, typename C, int UNR>
__global__ void __launch_bounds__(kThreads)
    k_cols(const typename St<SD>::T* __restrict__ A, const typename St<SD>::T* __restrict__ x,
           typename St<SD>::T* __restrict__ y, int64_t u, int64_t nk, int64_t v, int64_t ntile,
           C alpha, C beta, int has_beta) {
  constexpr int VEC = VecN<SD>::N;
  constexpr int JR = kThreads / 32;
  __shared__ C red[JR][32][VEC + (sizeof(C) == 8 ? 0 : 1)];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int64_t vv = v / VEC;
  const int64_t i = blockIdx.x / ntile;
  const int64_t tile = blockIdx.x - i * ntile;
  const int64_t col = tile * 32 + lane;
  const bool active = col < vv;
  const auto* base = A + i * nk * v + col * VEC;
  C acc[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) acc[e] = C(0);
  for (int64_t j0 = w; j0 < nk; j0 += (int64_t)JR * UNR) {
    uint4 buf[UNR];
#pragma unroll
    for (int t = 0; t < UNR; ++t) {
      const int64_t j = j0 + (int64_t)t * JR;
      if (active && j < nk) buf[t] = ld_stream16(base + j * v);
    }
#pragma unroll
    for (int t = 0; t < UNR; ++t) {
      const int64_t j = j0 + (int64_t)t * JR;
      if (active && j < nk) {
        const C xj = promote<SD, C>(__ldg(x + j));
        C a[VEC];
        unpack<SD, C>(buf[t], a);
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[e] = fma(a[e], xj, acc[e]);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < VEC; ++e) red[w][lane][e] = acc[e];
  __syncthreads();
  if (w == 0 && active) {
    const int64_t jr = nk < JR ? nk : JR;
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      C s = red[0][lane][e];
      for (int k = 1; k < jr; ++k) s += red[k][lane][e];
      const int64_t o = i * v + col * VEC + e;
      y[o] = epilogue<SD, C>(s, alpha, beta, has_beta != 0, y + o);
    }
  }
}

// --------------------------------------------------------------- SLABS ----
// one warp per slab of nk x v with vv = v / VEC in [1, 31] vectors per row;
// lanes (r = lane / vv, c = lane % vv), R = 32 / vv rows per step.
template <int SD, typename C, int UNR>
__global__ void __launch_bounds__(kThreads)
    k_slabs(const typename St<SD>::T* __restrict__ A, const typename St<SD>::T* __restrict__ x,
            typename St<SD>::T* __restrict__ y, int64_t u, int64_t nk, int v, C alpha, C beta,
            int has_beta) {
  constexpr int VEC = VecN<SD>::N;
  constexpr int NW = kThreads / 32;
  __shared__ C red[NW][32][VEC + (sizeof(C) == 8 ? 0 : 1)];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int vv = v / VEC;
  const int R = 32 / vv;
  const int r = lane / vv;
  const int c = lane - r * vv;
  const bool active = r < R;
  const int64_t warps_total = (int64_t)gridDim.x * NW;
  const int64_t gw = (int64_t)blockIdx.x * NW + w;
  for (int64_t i = gw; i < u; i += warps_total) {
    const auto* base = A + i * nk * v + c * VEC;
    C acc[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[e] = C(0);
    for (int64_t j0 = r; j0 < nk; j0 += (int64_t)R * UNR) {
      uint4 buf[UNR];
#pragma unroll
      for (int t = 0; t < UNR; ++t) {
        const int64_t j = j0 + (int64_t)t * R;
        if (active && j < nk) buf[t] = ld_stream16(base + j * v);
      }
#pragma unroll
      for (int t = 0; t < UNR; ++t) {
        const int64_t j = j0 + (int64_t)t * R;
        if (active && j < nk) {
          const C xj = promote<SD, C>(__ldg(x + j));
          C a[VEC];
          unpack<SD, C>(buf[t], a);
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc[e] = fma(a[e], xj, acc[e]);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < VEC; ++e) red[w][lane][e] = acc[e];
    __syncwarp();
    if (lane < vv) {
      const int64_t rr = nk < R ? nk : R;
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        C s = red[w][lane][e];
        for (int k = 1; k < rr; ++k) s += red[w][lane + k * vv][e];
        const int64_t o = i * v + (int64_t)lane * VEC + e;
        y[o] = epilogue<SD, C>(s, alpha, beta, has_beta != 0, y + o);
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------- GENERIC ----
// element (i, j, l) at A[i * su + j * sk + l]; used for unaligned views and the
// strided getvc.  v == 1: one warp per row, lanes stride the row (coalesced).
template <int SD, typename C>
__global__ void __launch_bounds__(kThreads)
    k_generic_rows(const typename St<SD>::T* __restrict__ A, const typename St<SD>::T* __restrict__ x,
                   typename St<SD>::T* __restrict__ y, int64_t u, int64_t nk, int64_t su,
                   int64_t sk, C alpha, C beta, int has_beta) {
  const int lane = threadIdx.x & 31;
  const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < u;
       i += warps_total) {
    C s = C(0);
    for (int64_t j = lane; j < nk; j += 32)
      s = fma(promote<SD, C>(A[i * su + j * sk]), promote<SD, C>(x[j]), s);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) y[i] = epilogue<SD, C>(s, alpha, beta, has_beta != 0, y + i);
  }
}

template <int SD, typename C>
__global__ void __launch_bounds__(kThreads)
    k_generic_cols(const typename St<SD>::T* __restrict__ A, const typename St<SD>::T* __restrict__ x,
                   typename St<SD>::T* __restrict__ y, int64_t u, int64_t nk, int64_t v,
                   int64_t su, int64_t sk, C alpha, C beta, int has_beta) {
  const int64_t total = u * v;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total;
       o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = o / v;
    const int64_t l = o - i * v;
    const auto* base = A + i * su + l;
    C s = C(0);
    for (int64_t j = 0; j < nk; ++j) s = fma(promote<SD, C>(base[j * sk]), promote<SD, C>(x[j]), s);
    y[o] = epilogue<SD, C>(s, alpha, beta, has_beta != 0, y + o);
  }
}

// ------------------------------------------------------------ dispatch ----
static int g_sms = 0;
static int sm_count() {
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

static int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

static unsigned grid_for(int64_t work_items, int64_t per_block, int waves_cap) {
  int64_t need = cdiv(work_items, per_block);
  int64_t cap = (int64_t)sm_count() * waves_cap;
  if (need > cap) need = cap;
  if (need < 1) need = 1;
  return (unsigned)need;
}

// pick G in {32, 16, 8, 4}: the widest group idling at most 1/8 of the
// vector slots of a row, else the one idling the fewest
static int pick_row_group(int64_t nkv) {
  int best = 32;
  int64_t best_waste = -1;
  for (int G : {32, 16, 8, 4}) {
    const int64_t waste = cdiv(nkv, G) * G - nkv;
    if (waste * 8 <= nkv) return G;
    if (best_waste < 0 || waste < best_waste) {
      best = G;
      best_waste = waste;
    }
  }
  return best;
}

int regime_of(const void* A, int storage, int64_t u, int64_t nk, int64_t v) {
  if (u < 0 || nk < 1 || v < 1) return -1;
  const int sb = dtype_bytes(storage);
  if (sb <= 0) return -1;
  const int VEC = 16 / sb;
  const bool aligned = (reinterpret_cast<uintptr_t>(A) & 15) == 0;
  if (v == 1) {
    if (!aligned || nk % VEC != 0) return REG_GENERIC;
    return (nk / VEC >= 8) ? REG_ROWS : REG_ROWS_SHORT;
  }
  if (!aligned || v % VEC != 0) return REG_GENERIC;
  return (v / VEC >= 32) ? REG_COLS : REG_SLABS;
}

template <int SD, typename C, int G>
static void launch_rows(const void* A, const void* x, void* y, int64_t u, int64_t nk, C al, C be,
                        int hb, cudaStream_t st) {
  using T = typename St<SD>::T;
  constexpr int UNR = 4;
  const size_t xs_bytes = (size_t)nk * sizeof(C);
  const int64_t rows_per_block = (kThreads / 32) * (32 / G);
  const unsigned grid = grid_for(u, rows_per_block, 32);
  if (xs_bytes <= 96 * 1024) {
    auto kern = k_rows<SD, C, G, UNR, true>;
    if (xs_bytes > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xs_bytes);
    kern<<<grid, kThreads, xs_bytes, st>>>((const T*)A, (const T*)x, (T*)y, u, nk, al, be, hb);
  } else {
    k_rows<SD, C, G, UNR, false>
        <<<grid, kThreads, 0, st>>>((const T*)A, (const T*)x, (T*)y, u, nk, al, be, hb);
  }
}

template <int SD, typename C>
static int tvc_typed(const void* A, int64_t u, int64_t nk, int64_t v, int64_t su, int64_t sk,
                     const void* x, double alpha, double beta, void* y, cudaStream_t st,
                     int force_generic) {
  using T = typename St<SD>::T;
  constexpr int VEC = VecN<SD>::N;
  const C al = (C)alpha, be = (C)beta;
  const int hb = beta != 0.0;
  if (u == 0 || v == 0) return TV_OK;
  const int reg = force_generic ? REG_GENERIC : regime_of(A, SD, u, nk, v);
  switch (reg) {
    case REG_ROWS: {
      const int G = pick_row_group(nk / VEC);
      if (G == 32) launch_rows<SD, C, 32>(A, x, y, u, nk, al, be, hb, st);
      else if (G == 16) launch_rows<SD, C, 16>(A, x, y, u, nk, al, be, hb, st);
      else if (G == 8) launch_rows<SD, C, 8>(A, x, y, u, nk, al, be, hb, st);
      else launch_rows<SD, C, 4>(A, x, y, u, nk, al, be, hb, st);
      break;
    }
    case REG_ROWS_SHORT: {
      constexpr int UNR = 4;
      const int nkv = (int)(nk / VEC);
      const int64_t rows_per_block = (kThreads / 32) * (32 / nkv) * UNR;
      const unsigned grid = grid_for(u, rows_per_block, 32);
      k_rows_short<SD, C, UNR>
          <<<grid, kThreads, 0, st>>>((const T*)A, (const T*)x, (T*)y, u, (int)nk, al, be, hb);
      break;
    }
    case REG_COLS: {
      constexpr int UNR = 4;
      const int64_t ntile = cdiv(v / VEC, 32);
      const int64_t blocks = u * ntile;
      if (blocks > 0x7fffffffLL) return set_error(TV_EKERNEL, "tv_tvc: view too large for COLS grid");
      k_cols<SD, C, UNR><<<(unsigned)blocks, kThreads, 0, st>>>((const T*)A, (const T*)x, (T*)y, u,
                                                                nk, v, ntile, al, be, hb);
      break;
    }
    case REG_SLABS: {
      constexpr int UNR = 4;
      const unsigned grid = grid_for(u, kThreads / 32, 32);
      k_slabs<SD, C, UNR>
          <<<grid, kThreads, 0, st>>>((const T*)A, (const T*)x, (T*)y, u, nk, (int)v, al, be, hb);
      break;
    }
    default: {
      if (v == 1) {
        const unsigned grid = grid_for(u, kThreads / 32, 32);
        k_generic_rows<SD, C>
            <<<grid, kThreads, 0, st>>>((const T*)A, (const T*)x, (T*)y, u, nk, su, sk, al, be, hb);
      } else {
        const unsigned grid = grid_for(u * v, kThreads, 32);
        k_generic_cols<SD, C><<<grid, kThreads, 0, st>>>((const T*)A, (const T*)x, (T*)y, u, nk, v,
                                                         su, sk, al, be, hb);
      }
    }
  }
  return check_launch("tv_tvc");
}

int tvc_dispatch(const void* A, int storage, int compute, int64_t u, int64_t nk, int64_t v,
                 int64_t su, int64_t sk, const void* x, double alpha, double beta, void* y,
                 void* stream, int force_generic) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (mode_id(storage, compute)) {
    case MODE_F64:
      return tvc_typed<TV_F64, double>(A, u, nk, v, su, sk, x, alpha, beta, y, st, force_generic);
    case MODE_F32:
      return tvc_typed<TV_F32, float>(A, u, nk, v, su, sk, x, alpha, beta, y, st, force_generic);
    case MODE_F32F64:
      return tvc_typed<TV_F32, double>(A, u, nk, v, su, sk, x, alpha, beta, y, st, force_generic);
    case MODE_F16F32:
      return tvc_typed<TV_F16, float>(A, u, nk, v, su, sk, x, alpha, beta, y, st, force_generic);
    case MODE_BF16F32:
      return tvc_typed<TV_BF16, float>(A, u, nk, v, su, sk, x, alpha, beta, y, st, force_generic);
    default:
      return set_error(TV_EMODE, "invalid (storage, compute) pair");
  }
}

}  // namespace tv

extern "C" int tv_tvc(const void* A, int storage, int compute, int64_t u, int64_t nk, int64_t v,
                      const void* x, double alpha, double beta, void* y, void* stream) {
  if (u < 0 || nk < 1 || v < 1)
    return tv::set_error(TV_EKERNEL, "tv_tvc: need u >= 0, nk >= 1, v >= 1");
  if ((u > 0 && (A == nullptr || y == nullptr)) || x == nullptr)
    return tv::set_error(TV_EKERNEL, "tv_tvc: null pointer");
  return tv::tvc_dispatch(A, storage, compute, u, nk, v, nk * v, v, x, alpha, beta, y, stream, 0);
}

extern "C" int tv_tvc_naive(const void* A, int storage, int compute, int64_t u, int64_t nk,
                            int64_t v, const void* x, double alpha, double beta, void* y,
                            void* stream) {
  if (u < 0 || nk < 1 || v < 1)
    return tv::set_error(TV_EKERNEL, "tv_tvc_naive: need u >= 0, nk >= 1, v >= 1");
  if ((u > 0 && (A == nullptr || y == nullptr)) || x == nullptr)
    return tv::set_error(TV_EKERNEL, "tv_tvc_naive: null pointer");
  return tv::tvc_dispatch(A, storage, compute, u, nk, v, nk * v, v, x, alpha, beta, y, stream, 1);
}

extern "C" int tv_tvc_regime(const void* A, int storage, int64_t u, int64_t nk, int64_t v) {
  return tv::regime_of(A, storage, u, nk, v);
}

extern "C" int tv_getvc(int trans, const void* A, int storage, int compute, int64_t m, int64_t n,
                        int64_t lda, const void* x, double alpha, double beta, void* y,
                        void* stream) {
  if (m < 0 || n < 0 || lda < n) return tv::set_error(TV_EKERNEL, "tv_getvc: need lda >= n >= 0");
  if (trans == 0) {  // matvec: y[i] = sum_j A[i*lda + j] x[j]
    if (m == 0) return TV_OK;
    if (n == 0) return tv::set_error(TV_EKERNEL, "tv_getvc: empty contraction");
    return tv::tvc_dispatch(A, storage, compute, m, n, 1, lda, 1, x, alpha, beta, y, stream,
                            lda != n);
  }
  if (trans == 1) {  // vecmat: y[c] = sum_i x[i] A[i*lda + c]
    if (n == 0) return TV_OK;
    if (m == 0) return tv::set_error(TV_EKERNEL, "tv_getvc: empty contraction");
    return tv::tvc_dispatch(A, storage, compute, 1, m, n, 0, lda, x, alpha, beta, y, stream,
                            lda != n);
  }
  return tv::set_error(TV_EKERNEL, "tv_getvc: trans must be 0 (matvec) or 1 (vecmat)");
}
