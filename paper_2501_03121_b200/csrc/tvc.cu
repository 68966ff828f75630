// Native mode-oblivious tensor-vector contraction (TVC) for sm_100a.
//
// Replaces the reference's tvc_native / getvc (pkg/src/tenvec/kernels.py:73-171):
// the order-d tensor is read through its (u, n_k, v) block view
// (tensor.py:85-102) -- u slabs of n_k x v, last index fastest -- so no mode
// ever needs an unfolding copy and every tensor byte is streamed from HBM
// exactly once.  The reference runs one BLAS matvec for k = d-1 and a Python
// loop of u BLAS vecmats otherwise; here one launch covers the whole view and
// the host picks a regime from the view's shape and alignment:
//
//   ROWS        v == 1: G lanes per row (G chosen so each lane keeps UNR loads
//               in flight with few idle slots), x promoted once into shared
//               memory, xor-shuffle row reduction.
//   ROWS_SHORT  v == 1, aligned rows of 1..7 16-byte vectors: lanes tile whole
//               rows (R = 32 / nkv rows per warp step), in-order segmented
//               shuffle sum per row.
//   COLS        v >= 32 units: a CTA = CW 32-lane column stripes x JR row
//               phases of one slab (JR from n_k: 1 for short columns -- no
//               reduction -- up to 8 for long ones), registers accumulate, a
//               fixed-order shared-memory fold finishes when JR > 1.
//   SLABS       1 < v < 32 units: one warp per slab, R = 32 / units rows per
//               step so each warp load is one contiguous run, then a
//               fixed-order fold across rows in shared memory.
//   FLAT /      narrow aligned slabs / short aligned rows streamed as flat
//   FLAT_ROWS   warp runs of 16-byte vectors, lanes mapped to columns by gcd.
//   STAGED      slabs that fit a 48 KB tile (odd extents, short rows): whole-
//               slab tiles moved by ONE TMA bulk copy each (cp.async.bulk on
//               mbarriers, double-buffered), dot products from shared memory.
//   STAGED_LONG larger slabs of <= 4096 columns: row-run tiles, one bulk copy
//               each, column sums kept in registers across a slab's tiles.
//   STAGED_TALL tall narrow unaligned slabs (n_k >= 1024 rows of 2-31
//               elements, few slabs): split-K row chunks, each a run of TMA
//               row tiles; a thread sums whole rows into column registers.
//   split-K     few outputs, long columns (COLS / SLABS / FLAT_U /
//               STAGED_TALL): row chunks write partial sums to a workspace
//               folded in chunk order.
//
// Every regime has an aligned form (one 16-byte ld.global.nc.L1::no_allocate
// per lane, "unit" = 16 bytes) and an unaligned form for rows or slabs that do
// not start on 16 bytes (odd extents such as the paper's 979^3 or 13^8 in
// fp64): scalar loads interleaved so consecutive lanes read consecutive
// elements ("unit" = one element; COLS lanes own VEC columns 32 apart).
//
// All regimes accumulate in the compute type, apply alpha after the dot
// product and beta * y after that (kernels.py:113-118), and demote once on
// store.  beta == 0 never reads y.  The reduction order of every output element
// depends only on (u, n_k, v, strides, dtype): reruns and ranks reproduce
// bits.  There are no tensor cores here: arithmetic intensity is 0.25-1 FLOP/B.

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>

#include "tv_internal.h"
#include "tv_norm.cuh"
#include "tv_types.cuh"

namespace tv {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// Launches of the TVC kernels.  Inside tv_tvc_sweep every mode after the
// first is launched with programmatic stream serialization (the modes are
// independent: same read-only tensor, distinct outputs), so its CTAs fill
// the SMs the previous mode's tail frees; PdlScope keeps completion order.
static thread_local bool t_pdl = false;

template <typename... KArgs, typename... Args>
static void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args... args) {
  count_launch();
  if (!t_pdl) {
    kern<<<grid, block, smem, st>>>(static_cast<KArgs>(args)...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// a lane's load: one 16-byte vector (AL) or one element
template <int SD, typename C, bool AL>
struct Unit {
  using T = typename St<SD>::T;
  static constexpr int N = AL ? VecN<SD>::N : 1;
  using Raw = typename std::conditional<AL, uint4, T>::type;
  static __device__ __forceinline__ Raw load(const T* p) {
    if constexpr (AL) return ld_stream16(p);
    else return ld_stream_elem(p);
  }
  static __device__ __forceinline__ void widen(const Raw& r, C (&out)[N]) {
    if constexpr (AL) unpack<SD, C>(r, out);
    else out[0] = promote<SD, C>(r);
  }
};

// ---------------------------------------------------------------- ROWS ----
// Row `row` starts at A + row * su.  Its body is read as 16-byte vectors
// q = g, g + G, ... (G lanes per row); with PEEL the row may start anywhere
// (odd extents such as 979 or 175 in fp64): the elements before its first
// 16-byte boundary (head) and after its last full vector (tail) are folded by
// scalar loads, so the body still streams as full vectors.
// Every lane issues QB loads per batch (one memory round trip): LONG rows
// loop over batches of QB vectors of one row; short rows (at most QB / RS
// vectors per lane) take ONE batch covering RS row steps, idle slots loading
// a clamped in-range vector so the batch issues without predicates.
// G (chosen on the host) trades the 128-byte-line count of a warp load
// (G >= 8) against the log2(G) shuffle levels each row's sum costs.
// XR (short aligned rows): each lane's x values -- the same for every row --
// are copied from shared memory into registers once, so the fold issues no
// shared-memory loads; the FMA order is unchanged (same bits).  C5's per-rank
// slab at p = 8 (rows of 512 bf16, k = 2): 6.20 -> 6.63 TB/s although the
// 2-byte forms go from 64 to 80 registers (3 CTAs per SM; forcing 4 spills);
// no other ROWS view changes (profiles/r02_rows_ab/rowxr_*.jsonl).
template <int SD, typename C, int G, int RS, int QB, bool XS, bool PEEL, bool LONG, bool XR = false>
__global__ void __launch_bounds__(kThreads)
    k_rows(const typename St<SD>::T* __restrict__ A, const typename St<SD>::T* __restrict__ x,
           typename St<SD>::T* __restrict__ y, int64_t u, int64_t nk, int64_t su, C alpha, C beta,
           int has_beta) {
  PdlScope pdl_scope;
  using T = typename St<SD>::T;
  constexpr int VEC = VecN<SD>::N;
  constexpr int QPL = QB / RS;  // loads per lane per row in one batch
  constexpr int RPW = 32 / G;   // rows per warp step
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* xs = reinterpret_cast<C*>(smem_raw);
  if (XS) {
    for (int64_t i = threadIdx.x; i < nk; i += blockDim.x) xs[i] = promote<SD, C>(x[i]);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int g = lane % G;
  const int rs = lane / G;
  const int64_t warps_total = (int64_t)gridDim.x * kWarps;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  auto xv = [&](int64_t j) -> C { return XS ? xs[j] : promote<SD, C>(__ldg(x + j)); };
  // head length (elements before the first 16-byte boundary) of a row
  auto head_of = [&](const T* rp) -> int64_t {
    if constexpr (!PEEL) return 0;
    const int64_t h = (int64_t)(((16u - (unsigned)(reinterpret_cast<uintptr_t>(rp) & 15u)) & 15u) / sizeof(T));
    return h < nk ? h : nk;
  };
  auto fold_vec = [&](const uint4& raw, int64_t j0, C (&acc)[VEC]) {
    C a[VEC];
    unpack<SD, C>(raw, a);
    if constexpr (XS && !PEEL) {
      // aligned rows: the VEC x values of a vector are contiguous 16-byte
      // aligned words of shared memory -- 16-byte loads, not VEC scalar ones
      constexpr int NX = VEC * (int)sizeof(C) / 16;
      union {
        uint4 u[NX];
        C c[VEC];
      } xw;
#pragma unroll
      for (int q = 0; q < NX; ++q) xw.u[q] = reinterpret_cast<const uint4*>(xs + j0)[q];
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[e] = fma(a[e], xw.c[e], acc[e]);
    } else {
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[e] = fma(a[e], xv(j0 + e), acc[e]);
    }
  };
  // head and tail elements of a peeled row (returned, added to acc[0] after)
  auto fold_edges = [&](const T* rp, int64_t h, int64_t nb) -> C {
    C e = C(0);
    if constexpr (PEEL) {
      for (int64_t j = g; j < h; j += G) e = fma(promote<SD, C>(__ldg(rp + j)), xv(j), e);
      for (int64_t j = h + nb * VEC + g; j < nk; j += G) e = fma(promote<SD, C>(__ldg(rp + j)), xv(j), e);
    }
    return e;
  };
  static_assert(!XR || (XS && !PEEL && !LONG), "register-resident x: short aligned rows only");
  C xr[XR ? QPL : 1][VEC];
  if constexpr (XR) {
    const int64_t nbr = nk / VEC;
#pragma unroll
    for (int t = 0; t < QPL; ++t) {
      const int64_t q = g + (int64_t)t * G;
#pragma unroll
      for (int e = 0; e < VEC; ++e) xr[t][e] = q < nbr ? xs[q * VEC + e] : C(0);
    }
  }
  for (int64_t row0 = gw * RPW * RS; row0 < u; row0 += warps_total * RPW * RS) {
    C acc[RS][VEC];
#pragma unroll
    for (int r2 = 0; r2 < RS; ++r2)
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[r2][e] = C(0);
    if constexpr (LONG) {  // rows of more than QB vectors per lane: batched loop
      const int64_t row = row0 + rs;
      if (row < u) {
        const T* rp = A + row * su;
        const int64_t h = head_of(rp);
        const int64_t nb = (nk - h) / VEC;
        const uint4* body = reinterpret_cast<const uint4*>(rp + h);
        // full batches without predicates, register double-buffered: batch
        // b + 1 is in flight while batch b folds
        int64_t q0 = g;
        const int64_t step = (int64_t)G * QPL;
        if (q0 + (int64_t)(QPL - 1) * G < nb) {
          uint4 cur[QPL];
#pragma unroll
          for (int t = 0; t < QPL; ++t) cur[t] = ld_stream16(body + q0 + (int64_t)t * G);
          for (;;) {
            const int64_t qn = q0 + step;
            const bool more = qn + (int64_t)(QPL - 1) * G < nb;
            uint4 nxt[QPL];
            if (more) {
#pragma unroll
              for (int t = 0; t < QPL; ++t) nxt[t] = ld_stream16(body + qn + (int64_t)t * G);
            }
#pragma unroll
            for (int t = 0; t < QPL; ++t) fold_vec(cur[t], h + (q0 + (int64_t)t * G) * VEC, acc[0]);
            q0 = qn;
            if (!more) break;
#pragma unroll
            for (int t = 0; t < QPL; ++t) cur[t] = nxt[t];
          }
        }
        for (; q0 < nb; q0 += G) fold_vec(ld_stream16(body + q0), h + q0 * VEC, acc[0]);
        if constexpr (PEEL) acc[0][0] += fold_edges(rp, h, nb);
      }
    } else {
      // loads of idle lanes / rows past the end are clamped to an in-range
      // vector (and not folded) so the batch issues without predicates
      uint4 buf[RS][QPL];
#pragma unroll
      for (int r2 = 0; r2 < RS; ++r2) {
        const int64_t row = row0 + (int64_t)r2 * RPW + rs;
        const T* rp = A + (row < u ? row : u - 1) * su;
        const int64_t h = head_of(rp);
        const int64_t nb = (nk - h) / VEC;
        const uint4* body = reinterpret_cast<const uint4*>(rp + h);
        if (!PEEL || nb > 0) {
#pragma unroll
          for (int t = 0; t < QPL; ++t) {
            const int64_t q = g + (int64_t)t * G;
            buf[r2][t] = ld_stream16(body + (q < nb ? q : nb - 1));
          }
        }
      }
#pragma unroll
      for (int r2 = 0; r2 < RS; ++r2) {
        const int64_t row = row0 + (int64_t)r2 * RPW + rs;
        if (row < u) {
          const T* rp = A + row * su;
          const int64_t h = head_of(rp);
          const int64_t nb = (nk - h) / VEC;
#pragma unroll
          for (int t = 0; t < QPL; ++t) {
            const int64_t q = g + (int64_t)t * G;
            if constexpr (XR) {
              if (q < nb) {
                C a[VEC];
                unpack<SD, C>(buf[r2][t], a);
#pragma unroll
                for (int e = 0; e < VEC; ++e) acc[r2][e] = fma(a[e], xr[t][e], acc[r2][e]);
              }
            } else {
              if (q < nb) fold_vec(buf[r2][t], h + q * VEC, acc[r2]);
            }
          }
          if constexpr (PEEL) acc[r2][0] += fold_edges(rp, h, nb);
        }
      }
    }
#pragma unroll
    for (int r2 = 0; r2 < RS; ++r2) {
      const int64_t row = row0 + (int64_t)r2 * RPW + rs;
      C s = acc[r2][0];
#pragma unroll
      for (int e = 1; e < VEC; ++e) s += acc[r2][e];
#pragma unroll
      for (int off = G / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (g == 0 && row < u) y[row] = epilogue<SD, C>(s, alpha, beta, has_beta != 0, y + row);
    }
  }
}

// ---------------------------------------------------------- ROWS_SHORT ----
// aligned rows of nkv in [1, 7] vectors; lanes (r = lane / nkv, c = lane % nkv)
template <int SD, typename C, int UNR>
__global__ void __launch_bounds__(kThreads)
    k_rows_short(const typename St<SD>::T* __restrict__ A, const typename St<SD>::T* __restrict__ x,
                 typename St<SD>::T* __restrict__ y, int64_t u, int nk, int64_t su, C alpha,
                 C beta, int has_beta) {
  PdlScope pdl_scope;
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
  const int64_t warps_total = (int64_t)gridDim.x * kWarps;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int64_t step = (int64_t)R * UNR;
  for (int64_t row0 = gw * step; row0 < u; row0 += warps_total * step) {
    uint4 buf[UNR];
#pragma unroll
    for (int t = 0; t < UNR; ++t) {
      const int64_t row = row0 + (int64_t)t * R + r;
      if (active && row < u) buf[t] = ld_stream16(A + row * su + c * VEC);
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
      for (int i = 1; i < nkv; ++i) s += __shfl_down_sync(0xffffffffu, p, i);
      if (active && c == 0 && row < u)
        y[row] = epilogue<SD, C>(s, alpha, beta, has_beta != 0, y + row);
    }
  }
}

// ---------------------------------------------------------------- COLS ----
// slab i at A + i * su, row j at + j * sk.  Warp (stripe, r) of the CTA sums
// rows j = r, r + JR, ... of its stripe.  Aligned: lane owns one 16-byte
// vector (VEC adjacent columns); unaligned: lane owns VEC columns 32 apart, so
// each of its scalar loads is part of one contiguous 32-element warp access.
template <int SD, typename C, int JR, int UNR, bool AL, bool SPLIT = false, bool DB = false>
__global__ void __launch_bounds__(kThreads)
    k_cols(const typename St<SD>::T* __restrict__ A, const typename St<SD>::T* __restrict__ x,
           typename St<SD>::T* __restrict__ y, int64_t u, int64_t nk_all, int64_t v, int64_t su,
           int64_t sk, int64_t ntile, C alpha, C beta, int has_beta, int64_t rpc,
           C* __restrict__ ws) {
  PdlScope pdl_scope;
  using T = typename St<SD>::T;
  constexpr int VEC = VecN<SD>::N;
  constexpr int CW = kWarps / JR;
  __shared__ C red[JR > 1 ? JR : 1][CW][32][VEC + (sizeof(C) == 8 ? 0 : 1)];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int stripe = w % CW;
  const int r = w / CW;
  const int64_t i = blockIdx.x / ntile;
  const int64_t tile = blockIdx.x - i * ntile;
  const int64_t sbase = (tile * CW + stripe) * 32;  // first unit of this warp's stripe
  // column of accumulator e
  auto col_of = [&](int e) -> int64_t {
    return AL ? (sbase + lane) * VEC + e : sbase * VEC + (int64_t)e * 32 + lane;
  };
  const bool any = AL ? (sbase + lane) * VEC < v : sbase * VEC + lane < v;
  // row chunk blockIdx.y: rows [jb, nk) (one chunk = the whole column when
  // gridDim.y == 1); with ws the chunk's partial sums go there, no epilogue
  // (SPLIT = false compiles the whole-column form: jb = 0, nk = nk_all)
  const int64_t jb = SPLIT ? (int64_t)blockIdx.y * rpc : 0;
  const int64_t nk = SPLIT ? (jb + rpc < nk_all ? jb + rpc : nk_all) : nk_all;
  const T* base = A + i * su;
  C acc[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) acc[e] = C(0);
  if (any) {
    // full batches of UNR rows without predicates (all loads issue back to
    // back), then the remaining rows one at a time
    int64_t j0 = jb + r;
    if constexpr (AL) {
      const T* cb = base + (sbase + lane) * VEC;
      auto fold = [&](const uint4& raw, int64_t j) {
        const C xj = promote<SD, C>(__ldg(x + j));
        C a[VEC];
        unpack<SD, C>(raw, a);
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[e] = fma(a[e], xj, acc[e]);
      };
      // long columns (JR > 1): register double buffer, batch b + 1 in flight
      // while batch b folds; short ones keep the lighter single-buffer loop
      // (occupancy matters more there)
      const int64_t step = (int64_t)JR * UNR;
      if constexpr (JR == 1) {
        for (; j0 + (int64_t)(UNR - 1) * JR < nk; j0 += step) {
          uint4 buf[UNR];
#pragma unroll
          for (int t = 0; t < UNR; ++t) buf[t] = ld_stream16(cb + (j0 + (int64_t)t * JR) * sk);
#pragma unroll
          for (int t = 0; t < UNR; ++t) fold(buf[t], j0 + (int64_t)t * JR);
        }
      } else if (j0 + (int64_t)(UNR - 1) * JR < nk) {
        uint4 cur[UNR];
#pragma unroll
        for (int t = 0; t < UNR; ++t) cur[t] = ld_stream16(cb + (j0 + (int64_t)t * JR) * sk);
        for (;;) {
          const int64_t jn = j0 + step;
          const bool more = jn + (int64_t)(UNR - 1) * JR < nk;
          uint4 nxt[UNR];
          if (more) {
#pragma unroll
            for (int t = 0; t < UNR; ++t) nxt[t] = ld_stream16(cb + (jn + (int64_t)t * JR) * sk);
          }
#pragma unroll
          for (int t = 0; t < UNR; ++t) fold(cur[t], j0 + (int64_t)t * JR);
          j0 = jn;
          if (!more) break;
#pragma unroll
          for (int t = 0; t < UNR; ++t) cur[t] = nxt[t];
        }
      }
      for (; j0 < nk; j0 += JR) fold(ld_stream16(cb + j0 * sk), j0);
    } else {
      // predicated batches (measured faster for scalar columns than split loops)
      bool ok[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) ok[e] = col_of(e) < v;
      if constexpr (DB) {
        // long columns of few stripes (paper d = 2 k = 0: 3.2 CTAs per SM):
        // a register double buffer keeps batch b + 1 in flight while batch
        // b folds -- twice the bytes in flight per warp
        const T* cb = base + sbase * VEC + lane;
        const int64_t step = (int64_t)JR * UNR;
        auto ldb = [&](T (&b)[UNR][VEC], int64_t jj) {
#pragma unroll
          for (int t = 0; t < UNR; ++t)
#pragma unroll
            for (int e = 0; e < VEC; ++e)
              if (ok[e]) b[t][e] = ld_stream_elem(cb + (jj + (int64_t)t * JR) * sk + e * 32);
        };
        auto fld = [&](const T (&b)[UNR][VEC], int64_t jj) {
#pragma unroll
          for (int t = 0; t < UNR; ++t) {
            const C xj = promote<SD, C>(__ldg(x + jj + (int64_t)t * JR));
#pragma unroll
            for (int e = 0; e < VEC; ++e)
              if (ok[e]) acc[e] = fma(promote<SD, C>(b[t][e]), xj, acc[e]);
          }
        };
        if (j0 + (int64_t)(UNR - 1) * JR < nk) {
          T cur[UNR][VEC], nxt[UNR][VEC];
          ldb(cur, j0);
          for (;;) {
            const int64_t jn = j0 + step;
            const bool more = jn + (int64_t)(UNR - 1) * JR < nk;
            if (more) ldb(nxt, jn);
            fld(cur, j0);
            j0 = jn;
            if (!more) break;
#pragma unroll
            for (int t = 0; t < UNR; ++t)
#pragma unroll
              for (int e = 0; e < VEC; ++e) cur[t][e] = nxt[t][e];
          }
        }
      }
      for (; j0 < nk; j0 += (int64_t)JR * UNR) {
        T buf[UNR][VEC];
#pragma unroll
        for (int t = 0; t < UNR; ++t) {
          const int64_t j = j0 + (int64_t)t * JR;
#pragma unroll
          for (int e = 0; e < VEC; ++e)
            if (j < nk && ok[e]) buf[t][e] = ld_stream_elem(base + j * sk + col_of(e));
        }
#pragma unroll
        for (int t = 0; t < UNR; ++t) {
          const int64_t j = j0 + (int64_t)t * JR;
          if (j < nk) {
            const C xj = promote<SD, C>(__ldg(x + j));
#pragma unroll
            for (int e = 0; e < VEC; ++e)
              if (ok[e]) acc[e] = fma(promote<SD, C>(buf[t][e]), xj, acc[e]);
          }
        }
      }
    }
  }
  const int64_t wrow = (i * gridDim.y + blockIdx.y) * v;  // partial row in ws
  if constexpr (JR == 1) {
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const int64_t c = col_of(e);
      if (c < v) {
        if (SPLIT && ws != nullptr) {
          ws[wrow + c] = acc[e];
        } else {
          const int64_t o = i * v + c;
          y[o] = epilogue<SD, C>(acc[e], alpha, beta, has_beta != 0, y + o);
        }
      }
    }
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e) red[r][stripe][lane][e] = acc[e];
    __syncthreads();
    if (r == 0) {
      const int64_t jr = nk - jb < JR ? nk - jb : JR;
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const int64_t c = col_of(e);
        if (c < v) {
          C s = red[0][stripe][lane][e];
          for (int k = 1; k < jr; ++k) s += red[k][stripe][lane][e];
          if (SPLIT && ws != nullptr) {
            ws[wrow + c] = s;
          } else {
            const int64_t o = i * v + c;
            y[o] = epilogue<SD, C>(s, alpha, beta, has_beta != 0, y + o);
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------- FLAT ----
// Narrow aligned slabs (vv = v / VEC in [1, 31] 16-byte vectors per row, odd
// part P of vv in {1, 3, 5, 7}): a warp streams its slab as one flat run of
// nk * vv vectors, lane l reading vector w = l + 32 t at step t -- every warp
// load is 512 contiguous bytes and no lane idles (SLABS leaves 32 mod vv
// lanes idle, 25 % for the C3 / C4 widths).  Lane l's vectors cycle through P
// columns, (l + 32 t) mod vv, so it keeps P accumulator vectors (slot t mod
// P); a fixed-order shared-memory fold over the 32 / gcd(32, vv) lanes that
// visited a column finishes the slab.  Row / column advance incrementally
// (no division in the stream).
__host__ __device__ __forceinline__ int gcd_small(int a, int b) {
  while (b) {
    const int t = a % b;
    a = b;
    b = t;
  }
  return a;
}

template <int SD, typename C, int P, int K>
__global__ void __launch_bounds__(kThreads)
    k_flat(const typename St<SD>::T* __restrict__ A, const typename St<SD>::T* __restrict__ x,
           typename St<SD>::T* __restrict__ y, int64_t u, int nk, int v, C alpha, C beta,
           int has_beta) {
  PdlScope pdl_scope;
  constexpr int VEC = VecN<SD>::N;
  constexpr int B = P * K;  // steps per batch (a multiple of P: slots are compile-time)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C* xs = reinterpret_cast<C*>(smem_raw);
  C(*red)[32][P][VEC] = reinterpret_cast<C(*)[32][P][VEC]>(
      smem_raw + ((nk * (int)sizeof(C) + 15) / 16) * 16);
  for (int i = threadIdx.x; i < nk; i += blockDim.x) xs[i] = promote<SD, C>(x[i]);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int vv = v / VEC;
  const int L = nk * vv;               // vectors per slab
  const int q32 = 32 / vv, r32 = 32 % vv;
  const int64_t warps_total = (int64_t)gridDim.x * kWarps;
  for (int64_t i = (int64_t)blockIdx.x * kWarps + w; i < u; i += warps_total) {
    const uint4* base = reinterpret_cast<const uint4*>(A + i * (int64_t)nk * v);
    C acc[P][VEC];
#pragma unroll
    for (int p = 0; p < P; ++p)
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[p][e] = C(0);
    int row = lane / vv, col = lane - (lane / vv) * vv;  // of vector w = lane
    int wv = lane;
    for (int t0 = 0; t0 * 32 < L; t0 += B) {
      uint4 buf[B];
#pragma unroll
      for (int tt = 0; tt < B; ++tt) {
        const int wi = wv + 32 * tt;
        buf[tt] = ld_stream16(base + (wi < L ? wi : L - 1));  // clamped: no predicate
      }
#pragma unroll
      for (int tt = 0; tt < B; ++tt) {
        if (wv < L) {
          C a[VEC];
          unpack<SD, C>(buf[tt], a);
          const C xr = xs[row];
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc[tt % P][e] = fma(a[e], xr, acc[tt % P][e]);
        }
        wv += 32;
        col += r32;
        row += q32;
        if (col >= vv) {
          col -= vv;
          ++row;
        }
      }
    }
    // lane l visits each of the P columns congruent to l mod g = gcd(32, vv)
    // exactly once, so column c gathers the 32 / g lanes l = c mod g + m g:
    // store slot p of lane l at (c = (l + 32 p) mod vv, m = l / g) and fold
    // m = 0, 1, ... in order (red is [32 / g][vv] slots of VEC, 32 P in all)
    const int g = gcd_small(32, vv);
    C(*slot)[VEC] = reinterpret_cast<C(*)[VEC]>(&red[w][0][0][0]);
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int c = (lane + 32 * p) % vv;
#pragma unroll
      for (int e = 0; e < VEC; ++e) slot[(lane / g) * vv + c][e] = acc[p][e];
    }
    __syncwarp();
    if (lane < vv) {
      C s[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) s[e] = slot[lane][e];
      for (int m = 1; m < 32 / g; ++m)
#pragma unroll
        for (int e = 0; e < VEC; ++e) s[e] += slot[m * vv + lane][e];
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const int64_t o = i * v + (int64_t)lane * VEC + e;
        y[o] = epilogue<SD, C>(s[e], alpha, beta, has_beta != 0, y + o);
      }
    }
    __syncwarp();
  }
}

// -------------------------------------------------------------- FLAT_U ----
// Tall narrow slabs whose rows are NOT 16-byte multiples (v = 7 fp64, v = 12
// bf16 ...) or are too tall for FLAT's shared-memory x: every (slab, row
// chunk) is one warp streaming its rows as a flat run of 16-byte vectors.
// A "group" of G = 32 P VEC elements (P warp loads, one per lane each) is a
// whole number RG = G / v of rows, so lane l's element (s, k) -- offset
// (32 s + l) VEC + k in every group -- always sits at the same (row, column)
// of its group: the lane keeps P x VEC accumulators, reads x at two rows per
// vector, and at the end the warp folds its G partial sums into column sums
// through shared memory in row order (a fixed order: reruns reproduce bits).
// Row chunks of rpc rows (a multiple of RG, so chunks start 16-byte aligned)
// split the long columns; their sums go to the split-K workspace.
template <int SD, typename C, int P>
__global__ void __launch_bounds__(kThreads)
    k_flat_u(const typename St<SD>::T* __restrict__ A, const typename St<SD>::T* __restrict__ x,
             typename St<SD>::T* __restrict__ y, int64_t u, int64_t nk, int v, int64_t su, C alpha, C beta,
             int has_beta, int64_t nch, int64_t rpc, C* __restrict__ ws) {
  PdlScope pdl_scope;
  using T = typename St<SD>::T;
  constexpr int VEC = VecN<SD>::N;
  constexpr int G = 32 * P * VEC;
  constexpr int UG = P >= 4 ? 1 : 4 / P;  // groups per batch: >= 4 loads in flight per lane
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  C* red = reinterpret_cast<C*>(smem_raw) + (size_t)w * G;  // this warp's RG x v partial sums
  const int RG = G / v;
  // where this lane's elements sit in a group: first element's row / column,
  // and the element k from which a vector's elements belong to the next row
  int r_s[P], kb_s[P];
#pragma unroll
  for (int s = 0; s < P; ++s) {
    const int off = (32 * s + lane) * VEC;
    r_s[s] = off / v;
    kb_s[s] = v - (off - r_s[s] * v);
  }
  const int64_t items = u * nch;
  const int64_t warps_total = (int64_t)gridDim.x * kWarps;
  for (int64_t it = (int64_t)blockIdx.x * kWarps + w; it < items; it += warps_total) {
    const int64_t i = it / nch;
    const int64_t ch = it - i * nch;
    const int64_t r0 = ch * rpc;
    const int64_t r1 = r0 + rpc < nk ? r0 + rpc : nk;
    const T* base = A + i * su + r0 * v;  // 16-byte aligned: r0 is a multiple of RG
    const int64_t ng = (r1 - r0) / RG;
    C acc[P][VEC];
#pragma unroll
    for (int s = 0; s < P; ++s)
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[s][e] = C(0);
    auto fold = [&](const uint4& raw, int s, int64_t row0) {
      C a[VEC];
      unpack<SD, C>(raw, a);
      const int64_t rr = row0 + r_s[s];
      const C x0 = promote<SD, C>(__ldg(x + rr));
      const C x1 = kb_s[s] < VEC ? promote<SD, C>(__ldg(x + rr + 1)) : x0;
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[s][e] = fma(a[e], e < kb_s[s] ? x0 : x1, acc[s][e]);
    };
    int64_t g = 0;
    for (; g + UG <= ng; g += UG) {
      uint4 buf[UG][P];
#pragma unroll
      for (int q = 0; q < UG; ++q)
#pragma unroll
        for (int s = 0; s < P; ++s)
          buf[q][s] = ld_stream16(reinterpret_cast<const uint4*>(base + (g + q) * G) + 32 * s + lane);
#pragma unroll
      for (int q = 0; q < UG; ++q)
#pragma unroll
        for (int s = 0; s < P; ++s) fold(buf[q][s], s, r0 + (g + q) * RG);
    }
    for (; g < ng; ++g) {
#pragma unroll
      for (int s = 0; s < P; ++s)
        fold(ld_stream16(reinterpret_cast<const uint4*>(base + g * G) + 32 * s + lane), s, r0 + g * RG);
    }
    // a partial last group (rows r0 + ng RG .. r1): element by element
    const int64_t tail_rows = (r1 - r0) - ng * RG;
    if (tail_rows > 0) {
      const T* tb = base + ng * G;
      const int64_t row0 = r0 + ng * RG;
#pragma unroll
      for (int s = 0; s < P; ++s)
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const int row = r_s[s] + (e >= kb_s[s] ? 1 : 0);
          if (row < tail_rows) {
            const C a = promote<SD, C>(ld_stream_elem(tb + (32 * s + lane) * VEC + e));
            acc[s][e] = fma(a, promote<SD, C>(__ldg(x + row0 + row)), acc[s][e]);
          }
        }
    }
    // element (s, e) of the group is (row r, column c): park it at red[r v + c]
    // (a bijection over the group), then column c sums its RG rows in order
#pragma unroll
    for (int s = 0; s < P; ++s)
#pragma unroll
      for (int e = 0; e < VEC; ++e) red[(32 * s + lane) * VEC + e] = acc[s][e];
    __syncwarp();
    for (int c = lane; c < v; c += 32) {
      C sum = red[c];
      for (int r = 1; r < RG; ++r) sum += red[r * v + c];
      if (nch > 1) {
        ws[(i * nch + ch) * v + c] = sum;
      } else {
        const int64_t o = i * v + c;
        y[o] = epilogue<SD, C>(sum, alpha, beta, has_beta != 0, y + o);
      }
    }
    __syncwarp();
  }
}

// ----------------------------------------------------------- FLAT_ROWS ----
// Short aligned rows (v == 1, nkv 16-byte vectors per row, odd part S of nkv
// in {1, 3, 5, 7}): the warp streams a block of 32 S vectors (= 32 / g whole
// rows, g = nkv / S) as S flat 512-byte loads, every lane busy; each lane
// dots its vector with its x piece, parks the partial in shared memory, and
// lane r then sums row r's nkv partials in order.  Replaces per-row shuffle
// trees and the idle lanes of power-of-two lane groups on rows like C3's 3, 6
// or 12 vectors.  K blocks per batch keep K * S loads in flight per lane.
template <int SD, typename C, int S, int K>
__global__ void __launch_bounds__(kThreads)
    k_flat_rows(const typename St<SD>::T* __restrict__ A, const typename St<SD>::T* __restrict__ x,
                typename St<SD>::T* __restrict__ y, int64_t u, int nk, C alpha, C beta,
                int has_beta) {
  PdlScope pdl_scope;
  constexpr int VEC = VecN<SD>::N;
  __shared__ C xs[32 * 8];  // nk <= 32 vectors of <= 8 elements
  __shared__ C part[kWarps][K][32 * S];
  for (int i = threadIdx.x; i < nk; i += blockDim.x) xs[i] = promote<SD, C>(x[i]);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int nkv = nk / VEC;
  const int rb = 32 * S / nkv;  // rows per block
  int piece[S];                 // x piece of this lane's vector at step t
#pragma unroll
  for (int t = 0; t < S; ++t) piece[t] = (lane + 32 * t) % nkv;
  const uint4* base = reinterpret_cast<const uint4*>(A);
  const int64_t total = u * nkv;  // vectors
  const int64_t nblocks = (u + rb - 1) / rb;
  const int64_t warps_total = (int64_t)gridDim.x * kWarps;
  for (int64_t b0 = ((int64_t)blockIdx.x * kWarps + w) * K; b0 < nblocks; b0 += warps_total * K) {
    uint4 buf[K][S];
#pragma unroll
    for (int kb = 0; kb < K; ++kb)
#pragma unroll
      for (int t = 0; t < S; ++t) {
        const int64_t wv = (b0 + kb) * 32 * S + lane + 32 * t;
        buf[kb][t] = ld_stream16(base + (wv < total ? wv : total - 1));  // clamped
      }
#pragma unroll
    for (int kb = 0; kb < K; ++kb)
#pragma unroll
      for (int t = 0; t < S; ++t) {
        C a[VEC];
        unpack<SD, C>(buf[kb][t], a);
        C p = a[0] * xs[piece[t] * VEC];
#pragma unroll
        for (int e = 1; e < VEC; ++e) p = fma(a[e], xs[piece[t] * VEC + e], p);
        part[w][kb][lane + 32 * t] = p;
      }
    __syncwarp();
#pragma unroll
    for (int kb = 0; kb < K; ++kb) {
      const int64_t row = (b0 + kb) * rb + lane;
      if (lane < rb && row < u) {
        C s = part[w][kb][lane * nkv];
        for (int j = 1; j < nkv; ++j) s += part[w][kb][lane * nkv + j];
        y[row] = epilogue<SD, C>(s, alpha, beta, has_beta != 0, y + row);
      }
    }
    __syncwarp();
  }
}

// --------------------------------------------------------------- SLABS ----
// one warp per slab; `units` = v / VEC (aligned) or v (unaligned) in [1, 31];
// lanes (r = lane / units, c = lane % units), R = 32 / units rows per step.
template <int SD, typename C, int UNR, bool AL>
__global__ void __launch_bounds__(kThreads)
    k_slabs(const typename St<SD>::T* __restrict__ A, const typename St<SD>::T* __restrict__ x,
            typename St<SD>::T* __restrict__ y, int64_t u, int64_t nk, int v, int64_t su,
            int64_t sk, C alpha, C beta, int has_beta, int64_t nch, int64_t rpc,
            C* __restrict__ ws) {
  PdlScope pdl_scope;
  using U = Unit<SD, C, AL>;
  constexpr int N = U::N;
  __shared__ C red[kWarps][32][N + (sizeof(C) == 8 ? 0 : 1)];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int units = v / N;
  const int R = 32 / units;
  const int r = lane / units;
  const int c = lane - r * units;
  const bool active = r < R;
  const int64_t warps_total = (int64_t)gridDim.x * kWarps;
  const int64_t gw = (int64_t)blockIdx.x * kWarps + w;
  // a warp unit = (slab i, row chunk ch); nch == 1: whole slabs, no partials
  for (int64_t unit = gw; unit < u * nch; unit += warps_total) {
    const int64_t i = unit / nch;
    const int64_t jb = (unit - i * nch) * rpc;
    const int64_t je = jb + rpc < nk ? jb + rpc : nk;
    const auto* base = A + i * su + c * N;
    C acc[N];
#pragma unroll
    for (int e = 0; e < N; ++e) acc[e] = C(0);
    // predicated batches (measured faster here than split full/remainder loops)
    for (int64_t j0 = jb + r; j0 < je; j0 += (int64_t)R * UNR) {
      typename U::Raw buf[UNR];
#pragma unroll
      for (int t = 0; t < UNR; ++t) {
        const int64_t j = j0 + (int64_t)t * R;
        if (active && j < je) buf[t] = U::load(base + j * sk);
      }
#pragma unroll
      for (int t = 0; t < UNR; ++t) {
        const int64_t j = j0 + (int64_t)t * R;
        if (active && j < je) {
          const C xj = promote<SD, C>(__ldg(x + j));
          C a[N];
          U::widen(buf[t], a);
#pragma unroll
          for (int e = 0; e < N; ++e) acc[e] = fma(a[e], xj, acc[e]);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < N; ++e) red[w][lane][e] = acc[e];
    __syncwarp();
    if (lane < units) {
      const int64_t rr = je - jb < R ? je - jb : R;
#pragma unroll
      for (int e = 0; e < N; ++e) {
        C s = red[w][lane][e];
        for (int k = 1; k < rr; ++k) s += red[w][lane + k * units][e];
        if (ws != nullptr) {
          ws[unit * v + (int64_t)lane * N + e] = s;  // the chunk's partial sum
        } else {
          const int64_t o = i * v + (int64_t)lane * N + e;
          y[o] = epilogue<SD, C>(s, alpha, beta, has_beta != 0, y + o);
        }
      }
    }
    __syncwarp();
  }
}

// -------------------------------------------------------------- STAGED ----
// Slabs that fit one tile, aligned or not: whole-slab tiles of the flat
// buffer are copied global -> shared by ONE TMA bulk copy each (aligned-down
// 16-byte start; the < 16-byte ragged end of the buffer by scalar loads),
// double-buffered per CTA on two mbarriers, so HBM sees pure contiguous
// streaming whatever n_k and v are and the SM issues no load instructions
// for the tile (the cp.async form was issue-bound at 4.1-5.8 TB/s); the dot
// products are then read from shared memory.  Output o of a tile = (slab
// o / v, column o % v); G lanes share an output (j = g, g + G, ...) and
// combine with an xor shuffle.  For v == 1, G lanes read consecutive words.
constexpr int kStageBytes = 49152;
constexpr int kStagedRowBytes = 512;     // aligned v == 1 rows up to this size are staged
constexpr int kStagedRowBytesU = 2048;  // unaligned ones
// stage size (bytes per tile buffer); TENVEC_B200_STAGE_BYTES overrides it for A/B runs
static int stage_bytes() {
  static const int b = [] {
    const char* e = getenv("TENVEC_B200_STAGE_BYTES");
    const int r = e ? atoi(e) : kStageBytes;
    return r < 4096 ? 4096 : (r > 65536 ? 65536 : r / 16 * 16);
  }();
  return b;
}
static int stage_count() {  // TENVEC_B200_STAGES: tiles per CTA ring (2..4)
  static const int n = [] {
    const char* e = getenv("TENVEC_B200_STAGES");
    const int r = e ? atoi(e) : 2;
    return r < 2 ? 2 : (r > 4 ? 4 : r);
  }();
  return n;
}
static int staged_row_bytes() {
  static const int b = [] {
    const char* e = getenv("TENVEC_B200_STAGE_ROW");
    return e ? atoi(e) : kStagedRowBytesU;
  }();
  return b;
}

// TMA 1-D bulk copies completing on an mbarrier (one elected thread issues a
// whole tile; every thread waits on the barrier's phase)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "TV_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TV_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int SD, typename C, bool VROW>
__global__ void __launch_bounds__(kThreads)
    k_staged(const typename St<SD>::T* __restrict__ A, const typename St<SD>::T* __restrict__ x,
             typename St<SD>::T* __restrict__ y, int64_t u, int nk, int v, int spt, int64_t ntiles,
             int G, int sbytes, int nst, C alpha, C beta, int has_beta) {
  PdlScope pdl_scope;
  using T = typename St<SD>::T;
  constexpr int SB = sizeof(T);
  constexpr int VEC = VecN<SD>::N;
  constexpr int NA = VROW ? VEC : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int xs_pad = (nk * (int)sizeof(C) + 15) / 16 * 16;
  C* xs = reinterpret_cast<C*>(smem_raw);
  unsigned char* const stage0 = smem_raw + xs_pad;
  auto stage = [&](int k) { return stage0 + k * (sbytes + 16); };
  C* red = reinterpret_cast<C*>(smem_raw + xs_pad + nst * (sbytes + 16));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + xs_pad + nst * (sbytes + 16) +
                                               (kThreads * sizeof(C) + 7) / 8 * 8);
  for (int i = threadIdx.x; i < nk; i += blockDim.x) xs[i] = promote<SD, C>(x[i]);
  if (threadIdx.x == 0) {
    for (int k = 0; k < nst; ++k) mbar_init(&bars[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const int L = nk * v;
  const unsigned char* gbase = reinterpret_cast<const unsigned char*>(A);
  const int64_t total_bytes = u * (int64_t)L * SB;
  const int64_t bulk_end = total_bytes & ~(int64_t)15;  // TMA moves whole 16-byte units
  // tile -> [a0, a1): 16-byte aligned bulk range; the < 16-byte ragged end of
  // the buffer (last tile only) is copied by scalar loads after the wait
  auto issue = [&](int64_t tile, int k) {
    const int64_t b0 = tile * spt * (int64_t)L * SB;
    const int64_t s1 = (tile + 1) * spt < u ? (tile + 1) * spt : u;
    const int64_t a0 = b0 & ~(int64_t)15;
    const int64_t e16 = (s1 * (int64_t)L * SB + 15) & ~(int64_t)15;
    const int64_t a1 = e16 < bulk_end ? e16 : bulk_end;
    const unsigned nb = a1 > a0 ? (unsigned)(a1 - a0) : 0u;
    mbar_expect_tx(&bars[k], nb);
    if (nb) bulk_g2s(stage(k), gbase + a0, nb, &bars[k]);
  };

  // thread = (gi, oi): output oi of each pass of `per` outputs, j-slice gi of G
  const int per = kThreads / G;
  const int gi = threadIdx.x / per;
  const int oi = threadIdx.x - gi * per;
  // units of a "row" (output's j range): 16-byte chunks when VROW, else elements
  const int nunits = VROW ? nk / VEC : nk;
  // nst-stage ring: tiles blockIdx.x + i * gridDim.x, i = 0 .. nst - 2, are in
  // flight before the first wait; stage `cur` holds the current tile
  int64_t tile = blockIdx.x;
  if (threadIdx.x == 0)
    for (int k = 0; k < nst - 1; ++k)
      if (tile + k * (int64_t)gridDim.x < ntiles) issue(tile + k * (int64_t)gridDim.x, k);
  int cur = 0;
  unsigned phase = 0;
  for (; tile < ntiles; tile += gridDim.x) {
    const int64_t ahead = tile + (nst - 1) * (int64_t)gridDim.x;
    if (threadIdx.x == 0 && ahead < ntiles) {
      // stage cur - 1 was released by the trailing __syncthreads of the
      // previous iteration; order those generic-proxy reads before the TMA write
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      issue(ahead, cur == 0 ? nst - 1 : cur - 1);
    }
    mbar_wait(&bars[cur], phase);
    unsigned char* const sp0 = stage(cur);
    if (tile == ntiles - 1 && (total_bytes & 15)) {  // block-uniform: ragged buffer end
      const int64_t a0 = (tile * spt * (int64_t)L * SB) & ~(int64_t)15;
      for (int64_t b = bulk_end + threadIdx.x; b < total_bytes; b += blockDim.x) sp0[b - a0] = gbase[b];
      __syncthreads();
    }
    if (++cur == nst) {
      cur = 0;
      phase ^= 1u;
    }
    const int64_t s0 = tile * spt;
    const int ns = (int)(spt < u - s0 ? spt : u - s0);
    const T* t = reinterpret_cast<const T*>(sp0 + ((s0 * (int64_t)L * SB) & 15));
    const int outs = ns * v;
    for (int ob = 0; ob < outs; ob += per) {  // block-uniform trip count
      const int o = ob + oi;
      C acc[NA];
#pragma unroll
      for (int e = 0; e < NA; ++e) acc[e] = C(0);
      if (o < outs && gi < G) {  // kThreads % G threads idle
        const int s = o / v;
        const int l = o - s * v;
        if constexpr (VROW) {
          // v == 1, 16-byte rows: rotate the start chunk by the row index when
          // the row has an even chunk count so a quarter-warp hits 8 banks
          const uint4* rp = reinterpret_cast<const uint4*>(t + s * nk);
          const int rot = (nunits & 1) ? 0 : s;
          for (int i = gi; i < nunits; i += G) {
            int q = i + rot % nunits;
            q = q >= nunits ? q - nunits : q;
            C a[VEC];
            unpack<SD, C>(rp[q], a);
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc[e] = fma(a[e], xs[q * VEC + e], acc[e]);
          }
        } else if (v == 1) {
          const T* rp = t + s * nk;
          const int rot = (nk & 1) ? 0 : s % nk;
          for (int i = gi; i < nk; i += G) {
            int j = i + rot;
            j = j >= nk ? j - nk : j;
            acc[0] = fma(promote<SD, C>(rp[j]), xs[j], acc[0]);
          }
        } else {
          // four interleaved partial sums: the shared-memory loads of four
          // rows are in flight together instead of one serial FMA chain
          // (C3 p = 8 k = 3: 48 rows per thread)
          const T* sp = t + s * L + l;
          C a4[4] = {C(0), C(0), C(0), C(0)};
          int j = gi;
          for (; j + 3 * G < nk; j += 4 * G) {
#pragma unroll
            for (int q = 0; q < 4; ++q) a4[q] = fma(promote<SD, C>(sp[(j + q * G) * v]), xs[j + q * G], a4[q]);
          }
          for (; j < nk; j += G) a4[0] = fma(promote<SD, C>(sp[j * v]), xs[j], a4[0]);
          acc[0] = (a4[0] + a4[1]) + (a4[2] + a4[3]);
        }
      }
      C sum = acc[0];
#pragma unroll
      for (int e = 1; e < NA; ++e) sum += acc[e];
      if (G > 1) {
        red[threadIdx.x] = sum;
        __syncthreads();
        if (gi == 0 && o < outs) {
          for (int k = 1; k < G; ++k) sum += red[k * per + oi];
          const int64_t oy = s0 * v + o;
          y[oy] = epilogue<SD, C>(sum, alpha, beta, has_beta != 0, y + oy);
        }
        __syncthreads();
      } else if (o < outs) {
        const int64_t oy = s0 * v + o;
        y[oy] = epilogue<SD, C>(sum, alpha, beta, has_beta != 0, y + oy);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------- STAGED_LONG ----
// Slabs larger than a tile with at most kLongCols columns (unaligned wide
// views, e.g. paper d = 7 k = 4: 19 x 361 fp64 slabs of 55 KB).  A slab's
// rows are contiguous, so a run of R rows of one slab is ONE contiguous byte
// range: each tile is a single TMA bulk copy (as in STAGED), a CTA walks the
// tiles of its slabs in order, and thread (gi, c) keeps the partial sums of
// columns c, c + per, ... (M of them) in registers across the slab's tiles;
// the G row groups (narrow slabs) fold through shared memory at slab end.
constexpr int kLongCols = 16 * kThreads;

template <int SD, typename C, int M>
__global__ void __launch_bounds__(kThreads)
    k_staged_long(const typename St<SD>::T* __restrict__ A, const typename St<SD>::T* __restrict__ x,
                  typename St<SD>::T* __restrict__ y, int64_t u, int nk, int v, int tps, int G,
                  int sbytes, C alpha, C beta, int has_beta) {
  PdlScope pdl_scope;
  using T = typename St<SD>::T;
  constexpr int SB = sizeof(T);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int xs_pad = (nk * (int)sizeof(C) + 15) / 16 * 16;
  C* xs = reinterpret_cast<C*>(smem_raw);
  unsigned char* const stage0 = smem_raw + xs_pad;
  C* red = reinterpret_cast<C*>(smem_raw + xs_pad + 2 * (sbytes + 16));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + xs_pad + 2 * (sbytes + 16) +
                                               (kThreads * sizeof(C) + 7) / 8 * 8);
  for (int i = threadIdx.x; i < nk; i += blockDim.x) xs[i] = promote<SD, C>(x[i]);
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const unsigned char* gbase = reinterpret_cast<const unsigned char*>(A);
  const int64_t row_bytes = (int64_t)v * SB;
  const int64_t total_bytes = u * nk * row_bytes;
  const int64_t bulk_end = total_bytes & ~(int64_t)15;
  const int64_t my_slabs = blockIdx.x < u ? (u - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t my_tiles = my_slabs * tps;
  // a slab's nk rows over its tps tiles: the first (nk % tps) tiles take one
  // row more.  Cursors advance incrementally (no divisions per tile): (slab,
  // tile q, first row j0) of the tile being summed and, on thread 0, of the
  // tile being fetched.
  const int rbase = nk / tps, rrem = nk % tps;
  const int per = kThreads / G;
  const int gi = threadIdx.x / per;
  const int c = threadIdx.x - gi * per;
  C acc[M];
#pragma unroll
  for (int m = 0; m < M; ++m) acc[m] = C(0);

  int64_t f_slab = blockIdx.x;  // fetch cursor (thread 0)
  int f_q = 0, f_j0 = 0;
  auto fetch = [&](int k) {
    const int f_j1 = f_j0 + rbase + (f_q < rrem ? 1 : 0);
    const int64_t b0 = (f_slab * nk + f_j0) * row_bytes;
    const int64_t a0 = b0 & ~(int64_t)15;
    const int64_t e16 = (b0 + (f_j1 - f_j0) * row_bytes + 15) & ~(int64_t)15;
    const int64_t a1 = e16 < bulk_end ? e16 : bulk_end;
    const unsigned nb = a1 > a0 ? (unsigned)(a1 - a0) : 0u;
    unsigned char* dst = stage0 + k * (sbytes + 16);
    mbar_expect_tx(&bars[k], nb);
    if (nb) bulk_g2s(dst, gbase + a0, nb, &bars[k]);
    if (++f_q == tps) {
      f_q = 0;
      f_j0 = 0;
      f_slab += gridDim.x;
    } else {
      f_j0 = f_j1;
    }
  };
  if (threadIdx.x == 0 && my_tiles > 0) fetch(0);

  int64_t slab = blockIdx.x;  // sum cursor (every thread)
  int q = 0, j0 = 0;
  for (int64_t t = 0; t < my_tiles; ++t) {
    const int k = (int)(t & 1);
    if (threadIdx.x == 0 && t + 1 < my_tiles) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      fetch(k ^ 1);
    }
    const int j1 = j0 + rbase + (q < rrem ? 1 : 0);
    const int64_t b0 = (slab * nk + j0) * row_bytes;
    unsigned char* const sp = stage0 + k * (sbytes + 16);
    mbar_wait(&bars[k], (unsigned)(t >> 1) & 1u);
    if (b0 + (j1 - j0) * row_bytes > bulk_end) {  // block-uniform: the buffer's ragged end
      const int64_t a0 = b0 & ~(int64_t)15;
      for (int64_t b = (bulk_end > a0 ? bulk_end : a0) + threadIdx.x; b < total_bytes; b += blockDim.x)
        sp[b - a0] = gbase[b];
      __syncthreads();
    }
    const T* tile = reinterpret_cast<const T*>(sp + (b0 & 15));
    if (gi < G) {
      for (int r = gi; r < j1 - j0; r += G) {
        const T* rp = tile + r * v + c;
        const C xj = xs[j0 + r];
#pragma unroll
        for (int m = 0; m < M; ++m)
          if (c + m * per < v) acc[m] = fma(promote<SD, C>(rp[m * per]), xj, acc[m]);
      }
    }
    if (j1 == nk) {  // slab done: fold the row groups, write its v outputs
      if (G > 1) {
#pragma unroll
        for (int m = 0; m < M; ++m) {
          red[threadIdx.x] = acc[m];
          __syncthreads();
          if (gi == 0 && c + m * per < v)
            for (int g2 = 1; g2 < G; ++g2) acc[m] += red[g2 * per + c];
          __syncthreads();
        }
      }
      if (gi == 0) {
#pragma unroll
        for (int m = 0; m < M; ++m) {
          if (c + m * per < v) {
            const int64_t o = slab * v + c + m * per;
            y[o] = epilogue<SD, C>(acc[m], alpha, beta, has_beta != 0, y + o);
          }
        }
      }
#pragma unroll
      for (int m = 0; m < M; ++m) acc[m] = C(0);
    }
    if (++q == tps) {
      q = 0;
      j0 = 0;
      slab += gridDim.x;
    } else {
      j0 = j1;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------- STAGED_TALL ----
// Tall narrow slabs whose rows are not 16-byte multiples (n_k >= 1024 rows of
// 2-31 elements, few slabs: [3000001, 7], [8, 1e6, 12] ...): the scalar
// loads of SLABS_U put 2-8 bytes per lane in flight and ran latency-bound
// at 0.8-2.7 TB/s.  Here a slab's rows are cut into chunks (split-K); a
// persistent CTA walks the row tiles of its chunks in order, each tile ONE
// TMA bulk copy of whole rows (aligned-down start, the buffer's ragged end by
// scalar loads) on a two-stage mbarrier ring, as in STAGED_LONG; thread t sums
// rows t, t + 256, ... of every tile into MAXV column accumulators (x read once
// per row), and at chunk end the CTA folds them -- a fixed xor tree per warp,
// then the 8 warps in order -- into the chunk's partial sums.
constexpr int kTallRowsPerThread = 16;  // rows per tile <= 16 * kThreads

#ifndef TV_TALL_OCC
#define TV_TALL_OCC 2
#endif
template <int SD, typename C, int MAXV>
__global__ void __launch_bounds__(kThreads, TV_TALL_OCC)
    k_staged_tall(const typename St<SD>::T* __restrict__ A, const typename St<SD>::T* __restrict__ x,
                  typename St<SD>::T* __restrict__ y, int64_t u, int64_t nk, int v, int64_t nch, int64_t rpc,
                  int tr, int sbytes, C alpha, C beta, int has_beta, C* __restrict__ ws) {
  PdlScope pdl_scope;
  using T = typename St<SD>::T;
  constexpr int SB = sizeof(T);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int stride_b = sbytes + 32 + (MAXV * SB + 15) / 16 * 16;
  unsigned char* const stage0 = smem_raw;
  C* red = reinterpret_cast<C*>(smem_raw + 2 * stride_b);  // [kWarps][MAXV]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + 2 * stride_b + (kWarps * MAXV * sizeof(C) + 7) / 8 * 8);
  // the last row's over-read (columns past v) never sees uninitialised bytes
  for (int i = threadIdx.x; i < 2 * stride_b / 16; i += kThreads)
    reinterpret_cast<uint4*>(stage0)[i] = make_uint4(0u, 0u, 0u, 0u);
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();

  const unsigned char* gbase = reinterpret_cast<const unsigned char*>(A);
  const int64_t row_bytes = (int64_t)v * SB;
  const int64_t total_bytes = u * nk * row_bytes;
  const int64_t bulk_end = total_bytes & ~(int64_t)15;
  const int64_t units = u * nch;
  // cursors (unit, first row j0 of the tile); a unit is (slab unit / nch,
  // rows [(unit % nch) * rpc, +rpc) clipped to nk)
  auto unit_end = [&](int64_t unit) {
    const int64_t e = (unit % nch + 1) * rpc;
    return e < nk ? e : nk;
  };
  int64_t f_unit = blockIdx.x, f_j0 = (f_unit % nch) * rpc;  // fetch cursor (thread 0)
  auto fetch = [&](int k) {
    const int64_t je = unit_end(f_unit);
    const int64_t j1 = f_j0 + tr < je ? f_j0 + tr : je;
    const int64_t b0 = ((f_unit / nch) * nk + f_j0) * row_bytes;
    const int64_t a0 = b0 & ~(int64_t)15;
    const int64_t e16 = (b0 + (j1 - f_j0) * row_bytes + 15) & ~(int64_t)15;
    const int64_t a1 = e16 < bulk_end ? e16 : bulk_end;
    const unsigned nb = a1 > a0 ? (unsigned)(a1 - a0) : 0u;
    mbar_expect_tx(&bars[k], nb);
    if (nb) bulk_g2s(stage0 + k * stride_b, gbase + a0, nb, &bars[k]);
    if (j1 == je) {
      f_unit += gridDim.x;
      f_j0 = (f_unit % nch) * rpc;
    } else {
      f_j0 = j1;
    }
  };
  if (threadIdx.x == 0 && blockIdx.x < units) fetch(0);

  C acc[MAXV];
#pragma unroll
  for (int m = 0; m < MAXV; ++m) acc[m] = C(0);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t unit = blockIdx.x, j0 = (unit % nch) * rpc;
  for (int64_t t = 0; unit < units; ++t) {
    const int k = (int)(t & 1);
    const int64_t je = unit_end(unit);
    const int64_t j1 = j0 + tr < je ? j0 + tr : je;
    if (threadIdx.x == 0 && (j1 < je || unit + gridDim.x < units)) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      fetch(k ^ 1);
    }
    const int64_t slab = unit / nch;
    const int64_t b0 = (slab * nk + j0) * row_bytes;
    unsigned char* const sp = stage0 + k * stride_b;
    mbar_wait(&bars[k], (unsigned)(t >> 1) & 1u);
    if (b0 + (j1 - j0) * row_bytes > bulk_end) {  // block-uniform: the buffer's ragged end
      const int64_t a0 = b0 & ~(int64_t)15;
      for (int64_t b = (bulk_end > a0 ? bulk_end : a0) + threadIdx.x; b < total_bytes; b += blockDim.x)
        sp[b - a0] = gbase[b];
      __syncthreads();
    }
    const T* tile = reinterpret_cast<const T*>(sp + (b0 & 15));
    const int rows = (int)(j1 - j0);
    // x of this thread's rows first (independent loads, one latency per
    // tile), then MAXV columns per row with no predicates: the columns past v
    // read the next row's elements (or the stage's zero pad) into
    // accumulators that are never folded
    C xr[kTallRowsPerThread];
#pragma unroll
    for (int i = 0; i < kTallRowsPerThread; ++i) {
      const int r = threadIdx.x + i * kThreads;
      xr[i] = r < rows ? promote<SD, C>(__ldg(x + j0 + r)) : C(0);
    }
#pragma unroll
    for (int i = 0; i < kTallRowsPerThread; ++i) {
      const int r = threadIdx.x + i * kThreads;
      if (r < rows) {
        if constexpr (SB == 2) {
          // 2-byte elements: the row as 32-bit words from the stage base,
          // re-paired by a funnel shift when it starts on an odd element
          const int e0 = (int)((b0 & 15) >> 1) + r * v;
          const uint32_t* wp = reinterpret_cast<const uint32_t*>(sp) + (e0 >> 1);
          const unsigned sh = (unsigned)(e0 & 1) * 16u;
          uint32_t wv[MAXV / 2 + 1];
#pragma unroll
          for (int q = 0; q <= MAXV / 2; ++q) wv[q] = wp[q];
#pragma unroll
          for (int q = 0; q < MAXV / 2; ++q) {
            const uint32_t pr = __funnelshift_r(wv[q], wv[q + 1], sh);
            acc[2 * q] = fma(promote<SD, C>((T)(pr & 0xffffu)), xr[i], acc[2 * q]);
            acc[2 * q + 1] = fma(promote<SD, C>((T)(pr >> 16)), xr[i], acc[2 * q + 1]);
          }
        } else {
          const T* rp = tile + r * v;
#pragma unroll
          for (int m = 0; m < MAXV; ++m) acc[m] = fma(promote<SD, C>(rp[m]), xr[i], acc[m]);
        }
      }
    }
    if (j1 == je) {  // chunk done: fold the CTA's row sums, column by column
#pragma unroll
      for (int m = 0; m < MAXV; ++m) {
        if (m < v) {
          C s = acc[m];
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
          if (lane == 0) red[w * MAXV + m] = s;
        }
        acc[m] = C(0);
      }
      __syncthreads();
      if (threadIdx.x < v) {
        C s = red[threadIdx.x];
#pragma unroll
        for (int ww = 1; ww < kWarps; ++ww) s += red[ww * MAXV + threadIdx.x];
        if (ws != nullptr) {
          ws[unit * v + threadIdx.x] = s;
        } else {
          const int64_t o = slab * v + threadIdx.x;
          y[o] = epilogue<SD, C>(s, alpha, beta, has_beta != 0, y + o);
        }
      }
      unit += gridDim.x;
      j0 = (unit % nch) * rpc;
    } else {
      j0 = j1;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------- TVC + NORMALIZE ----
// The last contraction of a dHOPM3 iteration (the carried 2-mode tensor
// contracted to the iteration's vector, hopm.py:295-319) with the vector
// normalisation folded into the kernel epilogue (kernels.py:242-254): CTAs of
// kNormThreads compute the outputs, the LAST CTA to finish (ticket counter,
// reset on exit) runs the tv_normalize tree over y -- the same bits as
// tv_normalize on the same y, one launch instead of a TVC, a copy and a norm.
// Meant for the small final products (<= kTvcNormMax elements): v == 1 ->
// a warp per row (16-byte loads when aligned); v > 1 -> a CTA per (slab,
// 32-column block), its 32 warps split n_k and fold in phase order.
constexpr int64_t kTvcNormMax = 1LL << 22;

template <int SD, typename C, bool AL>
__global__ void __launch_bounds__(kNormThreads)
    k_tvc_norm(const typename St<SD>::T* __restrict__ A, const typename St<SD>::T* __restrict__ x,
               typename St<SD>::T* __restrict__ y, int64_t u, int64_t nk, int64_t v, int64_t ncb,
               double* __restrict__ norm_out, int32_t* __restrict__ status, unsigned* counter) {
  PdlScope pdl_scope;
  using T = typename St<SD>::T;
  constexpr int VEC = VecN<SD>::N;
  constexpr int NW = kNormThreads / 32;
  __shared__ C red[NW][33];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (v == 1) {
    for (int64_t row = (int64_t)blockIdx.x * NW + w; row < u; row += (int64_t)gridDim.x * NW) {
      const T* rp = A + row * nk;
      C acc = C(0);
      if constexpr (AL) {
        for (int64_t q = lane; q < nk / VEC; q += 32) {
          C a[VEC];
          unpack<SD, C>(ld_stream16(rp + q * VEC), a);
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc = fma(a[e], promote<SD, C>(x[q * VEC + e]), acc);
        }
      } else {
        for (int64_t j = lane; j < nk; j += 32) acc = fma(promote<SD, C>(rp[j]), promote<SD, C>(x[j]), acc);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (lane == 0) y[row] = epilogue<SD, C>(acc, C(1), C(0), false, y + row);
    }
  } else {
    const int64_t items = u * ncb;
    for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
      const int64_t i = item / ncb;
      const int64_t l = (item - i * ncb) * 32 + lane;
      C acc = C(0);
      if (l < v) {
        const T* cp = A + i * nk * v + l;
        for (int64_t j = w; j < nk; j += NW) acc = fma(promote<SD, C>(cp[j * v]), promote<SD, C>(x[j]), acc);
      }
      red[w][lane] = acc;
      __syncthreads();
      if (w == 0 && l < v) {
        C s = red[0][lane];
        const int ph = nk < NW ? (int)nk : NW;
        for (int q = 1; q < ph; ++q) s += red[q][lane];
        y[i * v + l] = epilogue<SD, C>(s, C(1), C(0), false, y + i * v + l);
      }
      __syncthreads();
    }
  }
  // the last CTA to arrive normalises the whole vector
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  norm_block<SD, C, true>(y, u * v, norm_out, status, 1);
  if (threadIdx.x == 0) *counter = 0u;
}

// --------------------------------------------------------------- NAIVE ----
// the "looped" cross-check (tv_tvc_naive): plain scalar loops, element
// (i, j, l) at A[i * su + j * sk + l].  v == 1: one warp per row.
template <int SD, typename C>
__global__ void __launch_bounds__(kThreads)
    k_naive_rows(const typename St<SD>::T* __restrict__ A, const typename St<SD>::T* __restrict__ x,
                 typename St<SD>::T* __restrict__ y, int64_t u, int64_t nk, int64_t su, int64_t sk,
                 C alpha, C beta, int has_beta) {
  PdlScope pdl_scope;
  const int lane = threadIdx.x & 31;
  const int64_t warps_total = (int64_t)gridDim.x * kWarps;
  for (int64_t i = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); i < u; i += warps_total) {
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
    k_naive_cols(const typename St<SD>::T* __restrict__ A, const typename St<SD>::T* __restrict__ x,
                 typename St<SD>::T* __restrict__ y, int64_t u, int64_t nk, int64_t v, int64_t su,
                 int64_t sk, C alpha, C beta, int has_beta) {
  PdlScope pdl_scope;
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


// Lanes per row (units = 16-byte vectors).  A warp load costs one L1
// wavefront per 128-byte line it touches, so each row segment should be
// >= 128 bytes (G >= 8); every extra lane costs a shuffle level per row.
// Measured on B200 (C3/C4 short rows, C2 long rows): rows of <= 8 vectors
// take pow2ceil(units) lanes (adjacent rows stay contiguous), up to 32
// vectors 8 lanes, up to 64 vectors 16, longer rows the full warp.
static int pick_row_group(int64_t nunits, int sb, bool peel) {
  if (nunits <= 8) {
    int G = 1;
    while (G < nunits) G <<= 1;
    return G;
  }
  if (nunits <= 32) return 8;
  if (peel) return nunits <= 64 ? 16 : 32;
  // aligned rows, measured per row length on >= 1 GB views
  // (profiles/r02_rows_ab/rowg_len.txt): 64 vectors -> 32 lanes (fp64 5.55
  // -> 6.4, bf16 6.06 -> 6.5 TB/s, fp32 equal); 128 -> 8 lanes for 4- and
  // 8-byte storage (16 vectors per lane: the double-buffered long-row loop;
  // fp64 5.86 -> 6.69, fp32 6.02 -> 6.72; bf16 equal, kept at 32); 129-256 ->
  // 16 (fp64 6.29 -> 6.71, fp32 6.37 -> 6.75, bf16 5.70 -> 6.13); longer: 32
  if (nunits <= 64) return 32;
  if (nunits <= 128) return sb >= 4 ? 8 : 32;
  if (nunits <= 256) return 16;
  return 32;
}

// row phases of the COLS kernel: enough rows per warp for deep load
// pipelines, as many 32-lane stripes per CTA as the slab is wide, and at
// least 4 CTAs per SM so small views still fill the GPU
static int pick_col_phases(int64_t nk, int64_t stripes, int64_t u, int sb = 0) {
  static const int jr_env = [] {  // TENVEC_B200_COL_JR: row phases, for A/B runs
    const char* e = getenv("TENVEC_B200_COL_JR");
    return e ? atoi(e) : 0;
  }();
  if (jr_env == 1 || jr_env == 2 || jr_env == 4 || jr_env == 8) return jr_env;
  // one fp64 slab with plenty of stripes (C2 k = 0, C4 k = 0): whole columns
  // per warp measured faster than row phases (7.35 vs 7.24 TB/s, 7.20 vs
  // 7.10; profiles/r01_cols_jr_ab/) -- not for narrower types or few stripes
  if (sb == 8 && u == 1 && cdiv(stripes, kWarps) >= 16LL * sm_count()) return 1;
  int jr = nk >= 1024 ? 8 : nk >= 512 ? 4 : nk >= 256 ? 2 : 1;
  int cw_max = 1;
  while (cw_max < kWarps && cw_max * 2 <= stripes) cw_max *= 2;
  if (kWarps / jr > cw_max) jr = kWarps / cw_max;
  static const int want_env = [] {  // TENVEC_B200_COL_WANT: target CTAs per SM, for A/B runs
    const char* e = getenv("TENVEC_B200_COL_WANT");
    return e ? atoi(e) : 0;
  }();
  // at least one CTA per SM; more row phases only when the column blocks
  // cannot cover the SMs (C1 256^3 k = 0/1: 256 blocks of 2 phases stream at
  // 28.7 us vs 30.7 for 1024 blocks of 8, which need 1.7 waves at 4 per SM;
  // larger views are unaffected -- profiles/r02_cols_want_ab/)
  const int64_t want = (want_env > 0 ? want_env : 1) * (int64_t)sm_count();
  while (jr < kWarps && jr < nk && u * cdiv(stripes, kWarps / jr) < want) jr *= 2;
  return jr;
}

// TENVEC_B200_FORCE=<regime number> / tv_set_regime_override pin a regime
// wherever it is valid (kernel A/B measurements, regime coverage tests)
static std::atomic<int> g_forced{-2};
static int forced_regime() {
  int f = g_forced.load(std::memory_order_relaxed);
  if (f == -2) {
    const char* e = getenv("TENVEC_B200_FORCE");
    int want = e ? atoi(e) : -1;
    int expect = -2;
    g_forced.compare_exchange_strong(expect, want);
    f = g_forced.load(std::memory_order_relaxed);
  }
  return f;
}

// FLAT_U geometry: P = the warp loads per group (a group of 32 P VEC
// elements is a whole number of rows), 0 when the width is not supported:
// at most 128 bytes of accumulators per lane (P VEC values of the widest
// compute type the storage can have), so P <= 8 for fp64 and <= 4 otherwise
static int flat_u_period(int64_t v, int vec) {
  if (v < 2 || v >= 32 || v + 1 < vec) return 0;  // a 16-byte vector spans at most two rows
  const int d = (int)((32LL * vec) % v);
  const int P = d == 0 ? 1 : (int)(v / gcd_small((int)v, d));
  // 128 bytes of accumulators per lane: 4-byte storage may accumulate in
  // fp64 (f32f64); larger budgets for 2-byte storage compiled to 255
  // registers with spills
  const int cbytes = vec <= 4 ? 8 : 4;
  return (P <= 8 && P * vec * cbytes <= 128) ? P : 0;
}

// row chunks of a FLAT_U launch: enough (slab, chunk) warps for the GPU,
// chunks a whole number of groups
static void flat_u_split(int64_t u, int64_t nk, int64_t v, int vec, int P, int64_t* nch, int64_t* rpc) {
  const int64_t rg = 32LL * P * vec / v;
  const int64_t want = cdiv(32LL * sm_count(), u);
  int64_t n = std::max<int64_t>(1, std::min<int64_t>(want, nk / (8 * rg)));
  int64_t r = cdiv(cdiv(nk, n), rg) * rg;
  *rpc = r;
  *nch = cdiv(nk, r);
}

static int regime_strided(const void* A, int sb, int64_t u, int64_t nk, int64_t v, int64_t su,
                          int64_t sk) {
  const int VEC = 16 / sb;
  const bool base_al = (reinterpret_cast<uintptr_t>(A) & 15) == 0;
  const bool su_al = u <= 1 || (su * sb) % 16 == 0;
  const bool contiguous = su == nk * v && sk == v;
  const bool al_rows = base_al && su_al && nk % VEC == 0;
  const bool al_cols = base_al && su_al && (sk * sb) % 16 == 0 && v % VEC == 0;
  const int stb = stage_bytes();
  const bool stageable = base_al && contiguous && u > 1 && nk * v * sb + 16 <= stb;
  // STAGED_LONG: >= 8 slabs per co-resident CTA (2 per SM) keeps the tail
  // short; rows of > kThreads / 2 columns (narrower ones make long serial
  // column sums).  Measured: paper d = 4 k = 2 (175 columns) 6.8 vs COLS_U
  // 5.8 TB/s; on aligned views it beats COLS only for short columns of
  // fp32/fp64 (n_k <= 128: +1-2 %; n_k = 2048 or bf16 lose)
  const bool long_ok = base_al && contiguous && v > kThreads / 2 && v <= kLongCols &&
                       v * sb <= stb && nk * 8 <= 96 * 1024 && u >= 16LL * sm_count() &&
                       nk * v * sb + 16 > stb;
  const bool long_al_ok = long_ok && al_cols && nk <= 128 && sb >= 4 && v >= kThreads;
  // FLAT: aligned narrow contiguous slabs whose width's odd part is 1 or 3
  // and gcd(32, width) >= 2 (C3 / C4 widths 24, 12, 6 vectors; width 3 folds
  // 32 lanes per column and measured slower than SLABS), slabs of at least
  // one warp load
  const int64_t vvu = v / VEC;
  const int gg = vvu > 0 ? gcd_small(32, (int)std::min<int64_t>(vvu, 32)) : 1;
  const int64_t oddp = vvu / gg;
  const bool flat_ok = al_cols && contiguous && vvu >= 1 && vvu < 32 && (oddp == 1 || oddp == 3) &&
                       gg >= 2 && nk * vvu >= 32 && nk * 8 <= 96 * 1024;  // x lives in smem
  // FLAT_ROWS: short aligned contiguous rows of <= 32 vectors, odd part <= 7
  const int64_t nkv = nk / VEC;
  const int64_t rodd = nkv > 0 ? nkv / gcd_small(32, (int)std::min<int64_t>(nkv, 32)) : 0;
  const bool flat_rows_ok = v == 1 && al_rows && contiguous && nkv >= 1 && nkv <= 32 &&
                            (rodd == 1 || rodd == 3 || rodd == 5 || rodd == 7);
  // FLAT_U: contiguous slabs starting on 16 bytes, narrow rows of any
  // alignment whose group period is supported
  const bool flat_u_ok = base_al && contiguous && su_al && v > 1 && flat_u_period(v, VEC) > 0 &&
                         (int64_t)kWarps * 32 * flat_u_period(v, VEC) * VEC * 8 <= 96 * 1024;
  // STAGED_TALL: contiguous narrow slabs (2-31 elements) from a 16-byte base
  const bool tall_ok = base_al && contiguous && v > 1 && v < 32 && v * sb <= stb;
  // a forced regime the view cannot take falls through to the heuristics
  const int forced = forced_regime();
  if (forced > 0) {
    const bool ok = (forced == REG_ROWS && v == 1 && al_rows) ||
                    (forced == REG_ROWS_SHORT && v == 1 && al_rows && nk / VEC <= 8) ||
                    (forced == REG_ROWS_U && v == 1) || (forced == REG_COLS && v > 1 && al_cols) ||
                    (forced == REG_SLABS && v > 1 && al_cols && v / VEC < 32) ||
                    (forced == REG_COLS_U && v > 1) || (forced == REG_SLABS_U && v > 1 && v < 32) ||
                    (forced == REG_STAGED && stageable) || (forced == REG_FLAT && flat_ok) ||
                    (forced == REG_FLAT_ROWS && flat_rows_ok) || (forced == REG_FLAT_U && flat_u_ok) ||
                    (forced == REG_STAGED_TALL && tall_ok) ||
                    (forced == REG_STAGED_LONG && base_al && contiguous && v > 1 && v <= kLongCols &&
                     v * sb <= stb && u > 1 && nk * 8 <= 96 * 1024);
    if (ok) return forced;
  }
  // measured on B200 (profiles/r01_regime_ab.txt): aligned views always stream
  // best straight from HBM -- rows of any length through ROWS (G lanes per
  // row, batched row steps), wide slabs through COLS, narrow ones through
  // SLABS.  Views whose rows/slabs are NOT 16-byte multiples and small enough
  // go through STAGED (contiguous cp.async tiles), which beats scalar loads
  // 2-4x there; larger unaligned views use the peeled / scalar forms.
  // tall views -- few slabs, long columns -- are split-K SLABS: every other
  // narrow or row regime gets about u warps, too few for 148 SMs (a single
  // dot product would run on one warp)
  if (u < 16LL * sm_count() && nk >= 8192 && v == 1) return REG_SLABS_U;
  if (u < 16LL * sm_count() && nk >= 1024 && v > 1 && (al_cols ? v / VEC < 32 : v < 32)) {
    static const int fu_env = [] {  // TENVEC_B200_FLAT_U=0: keep SLABS for tall views, for A/B runs
      const char* e = getenv("TENVEC_B200_FLAT_U");
      return e ? atoi(e) : 1;
    }();
    // FLAT_U beats the scalar 2-byte loads of SLABS_U (C5-like bf16 / f16
    // narrow rows: [8, 1e6, 12] bf16 1.02 -> 2.32 TB/s); for 4- and 8-byte
    // storage and aligned rows SLABS / SLABS_U measured as fast or faster
    // (profiles/r02_flat_u_ab/)
    static const int st_env = [] {  // TENVEC_B200_STAGED_TALL=0: the previous choice, for A/B runs
      const char* e = getenv("TENVEC_B200_STAGED_TALL");
      return e ? atoi(e) : 1;
    }();
    if (tall_ok && st_env != 0 && !al_cols) return REG_STAGED_TALL;
    if (flat_u_ok && fu_env != 0 && sb == 2 && !al_cols) return REG_FLAT_U;
    return al_cols ? REG_SLABS : REG_SLABS_U;
  }
  if (v == 1) {
    // rows of 3, 5, 6, 7 vectors idle 25-60 % of ROWS' power-of-two lane
    // groups; streamed flat they measured 6.2-6.35 vs 4.6-5.9 TB/s.  fp64
    // rows up to 32 vectors too (their shuffle trees cost twice: C4's 48-
    // element rows 5.8 vs 5.5 TB/s)
    // short rows (<= 512 B aligned, <= 2 KB unaligned) stream best as
    // contiguous TMA tiles: 6.7-6.8 TB/s vs 5.8-6.6 (FLAT_ROWS / ROWS) and
    // 4.8 (ROWS_U, 175-element fp64 rows)
    if (stageable && nk * sb <= (al_rows ? kStagedRowBytes : staged_row_bytes())) return REG_STAGED;
    if (flat_rows_ok && (nkv & (nkv - 1)) != 0 && (nkv <= 8 || sb == 8)) return REG_FLAT_ROWS;
    if (al_rows) return REG_ROWS;
    return REG_ROWS_U;
  }
  // small aligned slabs with short columns (n_k <= 32) leave COLS/SLABS warps
  // too little work per slab: staged tiles win there (paper d = 9, 10 tensors)
  if (al_cols && stageable && nk <= 32 && nk * v * sb <= stb / 2) return REG_STAGED;
  if (long_al_ok) return REG_STAGED_LONG;
  // narrow aligned slabs FLAT cannot fold (odd part of the width 5, 7, ...,
  // or width 3 vectors): staged tiles when a slab fits one (C3 p = 8 k = 3,
  // 3-vector slabs: 6.8 vs SLABS 5.8 TB/s, profiles/r01_staged_ab/)
  // 6-vector slabs (gcd 2: 16 lanes per column fold) stream faster staged
  // (C3 p = 4 k = 3: 7.0 vs FLAT 6.7 TB/s); wider gcds keep FLAT
  if (al_cols && flat_ok && gg < 4 && stageable) return REG_STAGED;
  if (al_cols) return (v / VEC >= 32) ? REG_COLS : (flat_ok ? REG_FLAT : (stageable ? REG_STAGED : REG_SLABS));
  if (stageable) return REG_STAGED;  // any unaligned slab that fits one tile
  // larger unaligned slabs of <= kLongCols columns, many of them: row-run tiles
  if (long_ok) return REG_STAGED_LONG;
  return v >= 32 ? REG_COLS_U : REG_SLABS_U;
}

int regime_of(const void* A, int storage, int64_t u, int64_t nk, int64_t v) {
  if (u < 0 || nk < 1 || v < 1) return -1;
  const int sb = dtype_bytes(storage);
  if (sb <= 0) return -1;
  return regime_strided(A, sb, u, nk, v, nk * v, v);
}

constexpr int kRowBatch = 4;  // 16-byte loads per lane per batch
// long aligned rows (batched loop, register double buffer): 6 loads per
// lane per batch measured 1.5 % faster than 4 on C2 k = 2 (7.42 vs 7.31
// TB/s, profiles/r01_rows_ab/rq*; 8 no better); peeled rows keep 4 (paper
// d = 3 k = 2: 6.6 vs 6.9)
constexpr int kRowBatchLong = 6;

template <int SD, typename C, int G, int RS, bool PEEL, bool LONG>
static void launch_rows(const void* A, const void* x, void* y, int64_t u, int64_t nk, int64_t su,
                        C al, C be, int hb, cudaStream_t st) {
  using T = typename St<SD>::T;
  const size_t xs_bytes = (size_t)nk * sizeof(C);
  const int64_t rows_per_block = (int64_t)kWarps * (32 / G) * RS;
  const unsigned grid = grid_for(u, rows_per_block, 32);
  static const int xr_env = [] {  // TENVEC_B200_ROW_XR=0: x from shared memory, for A/B runs
    const char* e = getenv("TENVEC_B200_ROW_XR");
    return e ? atoi(e) : 1;
  }();
  constexpr int QPLS = kRowBatch / RS;
  constexpr bool kXR = !LONG && !PEEL && QPLS * VecN<SD>::N * sizeof(C) <= 128;
  if (kXR && xr_env != 0 && xs_bytes <= 96 * 1024) {
    auto kern = k_rows<SD, C, G, RS, kRowBatch, true, PEEL, LONG, kXR>;
    if (xs_bytes > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xs_bytes);
    launch_k(kern, grid, kThreads, xs_bytes, st, (const T*)A, (const T*)x, (T*)y, u, nk, su, al, be, hb);
  } else if (xs_bytes <= 96 * 1024) {
    auto kern = k_rows<SD, C, G, RS, (LONG && !PEEL) ? kRowBatchLong : kRowBatch, true, PEEL, LONG>;
    if (xs_bytes > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xs_bytes);
    launch_k(kern, grid, kThreads, xs_bytes, st, (const T*)A, (const T*)x, (T*)y, u, nk, su, al, be, hb);
  } else if constexpr (G == 32 && RS == 1 && LONG) {
    // rows longer than the shared-memory copy of x: x through L1
    launch_k(k_rows<SD, C, 32, 1, kRowBatch, false, PEEL, true>, grid, kThreads, 0, st, (const T*)A, (const T*)x, (T*)y, u, nk, su, al, be, hb);
  }
}

template <int SD, typename C, int G, bool PEEL>
static void rows_by_steps(int RS, bool lng, const void* A, const void* x, void* y, int64_t u,
                          int64_t nk, int64_t su, C al, C be, int hb, cudaStream_t st) {
  if (lng) launch_rows<SD, C, G, 1, PEEL, true>(A, x, y, u, nk, su, al, be, hb, st);
  else if (RS == 4) launch_rows<SD, C, G, 4, PEEL, false>(A, x, y, u, nk, su, al, be, hb, st);
  else if (RS == 2) launch_rows<SD, C, G, 2, PEEL, false>(A, x, y, u, nk, su, al, be, hb, st);
  else launch_rows<SD, C, G, 1, PEEL, false>(A, x, y, u, nk, su, al, be, hb, st);
}

template <int SD, typename C, bool PEEL>
static void launch_rows_auto(const void* A, const void* x, void* y, int64_t u, int64_t nk,
                             int64_t su, C al, C be, int hb, cudaStream_t st) {
  constexpr int VEC = VecN<SD>::N;
  const int64_t nunits = std::max<int64_t>(1, nk / VEC);
  int G = pick_row_group(nunits, (int)sizeof(typename St<SD>::T), PEEL);
  static const int g_env = [] {  // TENVEC_B200_ROW_G: lanes per row, for A/B runs
    const char* e = getenv("TENVEC_B200_ROW_G");
    return e ? atoi(e) : 0;
  }();
  if (g_env == 1 || g_env == 2 || g_env == 4 || g_env == 8 || g_env == 16 || g_env == 32) G = g_env;
  const int64_t qpl = cdiv(nunits, G);
  bool lng = qpl > kRowBatch;
  int RS = lng ? 1 : (qpl * 4 <= kRowBatch ? 4 : qpl * 2 <= kRowBatch ? 2 : 1);
  if ((size_t)nk * sizeof(C) > 96 * 1024) G = 32, RS = 1, lng = true;  // x stays in L1, not smem
  switch (G) {
    case 32: rows_by_steps<SD, C, 32, PEEL>(RS, lng, A, x, y, u, nk, su, al, be, hb, st); break;
    case 16: rows_by_steps<SD, C, 16, PEEL>(RS, lng, A, x, y, u, nk, su, al, be, hb, st); break;
    case 8: rows_by_steps<SD, C, 8, PEEL>(RS, lng, A, x, y, u, nk, su, al, be, hb, st); break;
    case 4: rows_by_steps<SD, C, 4, PEEL>(RS, lng, A, x, y, u, nk, su, al, be, hb, st); break;
    case 2: rows_by_steps<SD, C, 2, PEEL>(RS, lng, A, x, y, u, nk, su, al, be, hb, st); break;
    default: rows_by_steps<SD, C, 1, PEEL>(RS, lng, A, x, y, u, nk, su, al, be, hb, st); break;
  }
}

// ------------------------------------------------------------- SPLIT-K ----
// Few, long outputs (u x column blocks too small to fill 148 SMs, n_k large:
// tall-skinny views, single dot products, paper d = 2 k = 0): the rows are
// cut into nch chunks, each chunk's partial sums go to a workspace in the
// compute type, and k_split_fold adds the chunks of every output in chunk
// order (deterministic) and applies the epilogue.
template <int SD, typename C>
__global__ void __launch_bounds__(256)
    k_split_fold_cta(const C* __restrict__ ws, int64_t nch, int64_t n, int64_t v,
                     typename St<SD>::T* __restrict__ y, C alpha, C beta, int has_beta) {
  // few outputs, thousands of chunks: a CTA per output, thread t sums chunks
  // t, t + 256, ... in order (loads 4 deep), then a fixed pairwise tree
  __shared__ C red[256];
  const int t = threadIdx.x;
  for (int64_t o = blockIdx.x; o < n; o += gridDim.x) {
    const int64_t i = o / v;
    const C* p = ws + i * nch * v + (o - i * v);
    C s = C(0);
    int64_t ch = t;
    for (; ch + 3 * 256 < nch; ch += 4 * 256) {
      C b[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) b[k] = p[(ch + k * 256) * v];
#pragma unroll
      for (int k = 0; k < 4; ++k) s += b[k];
    }
    for (; ch < nch; ch += 256) s += p[ch * v];
    red[t] = s;
    __syncthreads();
#pragma unroll
    for (int h = 128; h > 0; h >>= 1) {
      if (t < h) red[t] += red[t + h];
      __syncthreads();
    }
    if (t == 0) y[o] = epilogue<SD, C>(red[0], alpha, beta, has_beta != 0, y + o);
    __syncthreads();
  }
}

template <int SD, typename C, bool WARP>
__global__ void __launch_bounds__(256)
    k_split_fold(const C* __restrict__ ws, int64_t nch, int64_t n, int64_t v,
                 typename St<SD>::T* __restrict__ y, C alpha, C beta, int has_beta) {
  if constexpr (WARP) {
    // many chunks: a warp per output, lane l sums chunks l, l + 32, ... in
    // order, then a fixed xor tree -- the same order on every call
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t o = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); o < n; o += warps) {
      const int64_t i = o / v;
      const C* p = ws + i * nch * v + (o - i * v);
      C s = C(0);
      // loads batched 8 deep (the adds keep their order): a few outputs of
      // thousands of chunks were a chain of dependent loads (4 M x 8 fp64:
      // 63 us for the fold vs 53 us for the contraction)
      int64_t ch = lane;
      for (; ch + 7 * 32 < nch; ch += 8 * 32) {
        C b[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) b[t] = p[(ch + t * 32) * v];
#pragma unroll
        for (int t = 0; t < 8; ++t) s += b[t];
      }
      for (; ch < nch; ch += 32) s += p[ch * v];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (lane == 0) y[o] = epilogue<SD, C>(s, alpha, beta, has_beta != 0, y + o);
    }
  } else {
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i = o / v;
      const C* p = ws + i * nch * v + (o - i * v);
      C s = p[0];
      int64_t ch = 1;
      for (; ch + 7 < nch; ch += 8) {
        C b[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) b[t] = p[(ch + t) * v];
#pragma unroll
        for (int t = 0; t < 8; ++t) s += b[t];
      }
      for (; ch < nch; ++ch) s += p[ch * v];
      y[o] = epilogue<SD, C>(s, alpha, beta, has_beta != 0, y + o);
    }
  }
}

// Split-K workspace: caller-provided (tv_tvc_ws / tv_getvc_ws, sized by
// tv_tvc_workspace_bytes) or, for the plain entry points only, a stream-ordered
// allocation.  Never a silent fallback to the unsplit kernel: the chunking
// fixes the summation order, so a view always splits the same way.
struct Ws {
  void* p;
  int64_t bytes;
  bool given;
};

// chunk counts of the split-K forms (1 = no split); pure functions of the
// view so tv_tvc_workspace_bytes can size the workspace ahead of the launch
static int64_t cols_split(int64_t blocks, int64_t nk) {
  if (!(blocks < 2LL * sm_count() && nk >= 512)) return 1;
  const int64_t nch = std::min<int64_t>(cdiv(8LL * sm_count(), blocks), nk / 128);
  return nch > 1 ? cdiv(nk, cdiv(nk, nch)) : 1;
}

static int64_t slabs_split(int64_t u, int64_t nk) {
  static const int64_t per_sm = [] {  // TENVEC_B200_SLAB_SPLIT: warp units per SM, for A/B runs
    const char* e = getenv("TENVEC_B200_SLAB_SPLIT");
    const int r = e ? atoi(e) : 32;
    return (int64_t)(r < 8 ? 8 : (r > 256 ? 256 : r));
  }();
  if (!(u < 32LL * sm_count() && nk >= 256)) return 1;
  const int64_t nch = std::min<int64_t>(cdiv(per_sm * sm_count(), u), nk / 64);
  return nch > 1 ? cdiv(nk, cdiv(nk, nch)) : 1;
}

template <typename C>
static C* split_ws(const Ws& ws, int64_t elems, cudaStream_t st, int* rc) {
  const size_t need = (size_t)elems * sizeof(C);
  if (ws.given) {
    if (ws.p == nullptr || ws.bytes < (int64_t)need || (reinterpret_cast<uintptr_t>(ws.p) & 15)) {
      *rc = set_error(TV_EKERNEL, "tv_tvc: split-K workspace missing, misaligned or smaller than "
                                  "tv_tvc_workspace_bytes");
      return nullptr;
    }
    return static_cast<C*>(ws.p);
  }
  void* p = nullptr;
  if (cudaMallocAsync(&p, need, st) != cudaSuccess) {
    cudaGetLastError();
    *rc = set_error(TV_ECUDA, "tv_tvc: split-K workspace allocation failed (pass one to tv_tvc_ws)");
    return nullptr;
  }
  return static_cast<C*>(p);
}

template <int SD, typename C>
static void split_finish(C* ws, const Ws& given, int64_t nch, int64_t u, int64_t v, void* y, C al, C be,
                         int hb, cudaStream_t st) {
  using T = typename St<SD>::T;
  const int64_t n = u * v;
  if (nch >= 1024 && n <= 2LL * sm_count()) {
    count_launch();
    k_split_fold_cta<SD, C><<<(unsigned)n, 256, 0, st>>>(ws, nch, n, v, (T*)y, al, be, hb);
  } else if (nch >= 32) {
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 8), 8LL * sm_count()));
    count_launch();
    k_split_fold<SD, C, true><<<g, 256, 0, st>>>(ws, nch, n, v, (T*)y, al, be, hb);
  } else {
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 8LL * sm_count()));
    count_launch();
    k_split_fold<SD, C, false><<<g, 256, 0, st>>>(ws, nch, n, v, (T*)y, al, be, hb);
  }
  if (!given.given) cudaFreeAsync(ws, st);
}

template <int SD, typename C>
static void launch_staged(const void* A, const void* x, void* y, int64_t u, int64_t nk, int64_t v,
                          C al, C be, int hb, cudaStream_t st) {
  using T = typename St<SD>::T;
  constexpr int VEC = VecN<SD>::N;
  const int64_t slab_bytes = nk * v * (int64_t)sizeof(T);
  const int sbytes = stage_bytes();
  // slabs per tile: as many as fit, trimmed so the tile's outputs fill whole
  // passes of kThreads threads (269 outputs would run a 13-thread 2nd pass)
  const bool vrow = v == 1 && (slab_bytes % 16) == 0;
  const int64_t units = vrow ? nk / VEC : nk;
  // idle threads split each output's j range (G need not be a power of two)
  auto g_of = [&](int64_t s) {
    return (int)std::max<int64_t>(1, std::min<int64_t>({kThreads / (s * v), units / 2, 32}));
  };
  auto eff = [&](int64_t s) {  // busy fraction of the thread passes over a tile
    const int64_t per = kThreads / g_of(s);
    return (double)(s * v) / (double)(cdiv(s * v, per) * per);
  };
  int64_t spt64 = std::max<int64_t>(1, std::min<int64_t>(sbytes / slab_bytes, u));
  if (spt64 * v >= kThreads) {
    const int64_t trim = std::max<int64_t>(1, (spt64 * v / kThreads) * kThreads / v);
    if (eff(trim) > eff(spt64) + 1e-9) spt64 = trim;
  }
  const int spt = (int)spt64;
  const int64_t ntiles = cdiv(u, spt);
  const int G = g_of(spt64);
  const int nst = stage_count();
  const size_t smem = (size_t)cdiv(nk * (int64_t)sizeof(C), 16) * 16 + nst * (sbytes + 16) +
                      (kThreads * sizeof(C) + 7) / 8 * 8 + nst * sizeof(uint64_t);
  // persistent grid: as many CTAs as are co-resident, tiles strided over them
  const int per_sm = std::max(1, std::min(8, (int)(228 * 1024 / (smem + 1024))));
  const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)per_sm * sm_count());
  if (vrow) {
    auto kern = k_staged<SD, C, true>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_k(kern, grid, kThreads, smem, st, (const T*)A, (const T*)x, (T*)y, u, (int)nk, (int)v, spt,
                                       ntiles, G, sbytes, nst, al, be, hb);
  } else {
    auto kern = k_staged<SD, C, false>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_k(kern, grid, kThreads, smem, st, (const T*)A, (const T*)x, (T*)y, u, (int)nk, (int)v, spt,
                                       ntiles, G, sbytes, nst, al, be, hb);
  }
}

template <int SD, typename C>
static void launch_staged_long(const void* A, const void* x, void* y, int64_t u, int64_t nk,
                               int64_t v, C al, C be, int hb, cudaStream_t st) {
  using T = typename St<SD>::T;
  const int sbytes = stage_bytes();
  const int64_t row_bytes = v * (int64_t)sizeof(T);
  const int64_t rmax = std::max<int64_t>(1, sbytes / row_bytes);
  const int tps = (int)cdiv(nk, rmax);  // tiles per slab
  const int R = (int)cdiv(nk, tps);
  // row groups: all threads busy (two groups of 128 columns for 128 < v < 256)
  const int G = v >= kThreads ? 1
                : v > kThreads / 2 ? 2
                                   : (int)std::max<int64_t>(1, std::min<int64_t>({kThreads / v, R, 32}));
  const int M = (int)cdiv(v, kThreads / G);
  const size_t smem = (size_t)cdiv(nk * (int64_t)sizeof(C), 16) * 16 + 2 * (sbytes + 16) +
                      (kThreads * sizeof(C) + 7) / 8 * 8 + 2 * sizeof(uint64_t);
  const int per_sm = std::max(1, std::min(8, (int)(228 * 1024 / (smem + 1024))));
  const unsigned grid = (unsigned)std::min<int64_t>(u, (int64_t)per_sm * sm_count());
  auto go = [&](auto kern) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_k(kern, grid, kThreads, smem, st, (const T*)A, (const T*)x, (T*)y, u, (int)nk, (int)v, tps, G, sbytes,
                                       al, be, hb);
  };
  if (M <= 1) go(k_staged_long<SD, C, 1>);
  else if (M <= 2) go(k_staged_long<SD, C, 2>);
  else if (M <= 4) go(k_staged_long<SD, C, 4>);
  else if (M <= 8) go(k_staged_long<SD, C, 8>);
  else go(k_staged_long<SD, C, 16>);
}

// STAGED_TALL geometry: rows per tile, chunks per slab and rows per chunk
// (a pure function of the view, so tv_tvc_workspace_bytes can size it)
static void staged_tall_split(int64_t u, int64_t nk, int64_t v, int sb, int* tr, int64_t* nch, int64_t* rpc) {
  const int64_t rmax = std::max<int64_t>(1, std::min<int64_t>(stage_bytes() / (v * sb), 16LL * kThreads));
  const int64_t want = cdiv(8LL * sm_count(), u);  // ~4 chunks per co-resident CTA
  int64_t n = std::max<int64_t>(1, std::min<int64_t>(want, cdiv(nk, rmax)));
  const int64_t r = cdiv(nk, n);
  *tr = (int)std::min<int64_t>(rmax, r);
  *rpc = r;
  *nch = cdiv(nk, r);
}

template <int SD, typename C>
static int launch_staged_tall(const void* A, const void* x, void* y, int64_t u, int64_t nk, int64_t v, C al,
                              C be, int hb, const Ws& wsa, cudaStream_t st) {
  using T = typename St<SD>::T;
  int tr = 1;
  int64_t nch = 1, rpc = nk;
  staged_tall_split(u, nk, v, (int)sizeof(T), &tr, &nch, &rpc);
  int rc = TV_OK;
  C* ws = nullptr;
  if (nch > 1 && (ws = split_ws<C>(wsa, u * nch * v, st, &rc)) == nullptr) return rc;
  const int sbytes = stage_bytes();
  const int maxv = v <= 4 ? 4 : v <= 8 ? 8 : v <= 12 ? 12 : v <= 16 ? 16 : v <= 24 ? 24 : 32;
  const size_t stride_b = (size_t)sbytes + 32 + ((size_t)maxv * sizeof(T) + 15) / 16 * 16;
  const size_t smem = 2 * stride_b + ((size_t)kWarps * maxv * sizeof(C) + 7) / 8 * 8 + 2 * sizeof(uint64_t);
  // co-resident CTAs per SM: registers (__launch_bounds__(256, 2): up to 128
  // per thread) allow 2, shared memory 2 at the default 48 KB stages (a third
  // CTA per SM with 32 KB stages ran as a second wave: 3.75 -> 3.07 TB/s)
  const int64_t per_sm = std::max<int64_t>(1, std::min<int64_t>(TV_TALL_OCC, (int64_t)(227 * 1024) / (int64_t)(smem + 1024)));
  const unsigned grid = (unsigned)std::min<int64_t>(u * nch, per_sm * sm_count());
  auto go = [&](auto kern) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_k(kern, grid, kThreads, smem, st, (const T*)A, (const T*)x, (T*)y, u, nk, (int)v, nch, rpc, tr,
             sbytes, al, be, hb, ws);
  };
  switch (maxv) {
    case 4: go(k_staged_tall<SD, C, 4>); break;
    case 8: go(k_staged_tall<SD, C, 8>); break;
    case 12: go(k_staged_tall<SD, C, 12>); break;
    case 16: go(k_staged_tall<SD, C, 16>); break;
    case 24: go(k_staged_tall<SD, C, 24>); break;
    default: go(k_staged_tall<SD, C, 32>); break;
  }
  if (ws != nullptr) split_finish<SD, C>(ws, wsa, nch, u, v, y, al, be, hb, st);
  return TV_OK;
}

// column blocks of a COLS launch (row phases JR from the view)
template <int SD, bool AL>
static int64_t cols_blocks(int64_t u, int64_t nk, int64_t v, int* jr_out, int64_t* ntile_out) {
  using T = typename St<SD>::T;
  constexpr int VEC = VecN<SD>::N;
  const int64_t stripes = cdiv(v, 32 * VEC);
  const int JR = pick_col_phases(nk, stripes, u, AL ? (int)sizeof(T) : 0);
  const int64_t ntile = cdiv(stripes, kWarps / JR);
  if (jr_out) *jr_out = JR;
  if (ntile_out) *ntile_out = ntile;
  return u * ntile;
}

template <int SD, typename C, bool AL>
static int launch_cols(const void* A, const void* x, void* y, int64_t u, int64_t nk, int64_t v,
                       int64_t su, int64_t sk, C al, C be, int hb, const Ws& wsa, cudaStream_t st) {
  using T = typename St<SD>::T;
  constexpr int VEC = VecN<SD>::N;
  constexpr int UA_UNR = VEC >= 8 ? 2 : 4;  // scalar loads in flight: UNR * VEC (8 measured slower)
  int JR = 1;
  int64_t ntile = 1;
  const int64_t blocks = cols_blocks<SD, AL>(u, nk, v, &JR, &ntile);
  if (blocks > 0x7fffffffLL) return set_error(TV_EKERNEL, "tv_tvc: view too large for COLS grid");
  const T* At = (const T*)A;
  const T* xt = (const T*)x;
  T* yt = (T*)y;
  // split-K when the column blocks cannot fill the GPU (< 2 per SM; at 3.2
  // per SM, paper d = 2 k = 0, splitting measured slower: 5.6 vs 5.9 TB/s)
  const int64_t nch = cols_split(blocks, nk);
  C* ws = nullptr;
  if (nch > 1) {
    int rc = TV_OK;
    if ((ws = split_ws<C>(wsa, u * nch * v, st, &rc)) == nullptr) return rc;
  }
  const int64_t rpc = cdiv(nk, nch);
  const dim3 b((unsigned)blocks, (unsigned)nch);
  auto done = [&]() {
    if (ws != nullptr) split_finish<SD, C>(ws, wsa, nch, u, v, y, al, be, hb, st);
    return TV_OK;
  };
  // unaligned, fp32/fp64: 3-row batches measured better for 4 row phases
  // (paper d = 3: 7.1-7.2 vs 6.6-6.8 TB/s) and for n_k <= 16 (d = 8: 6.4 vs
  // 6.1); 4 elsewhere (d = 2 k = 0 with 8 phases: 5.9 vs 5.1)
  // the split-capable instantiation runs when splitting, and also for the
  // unaligned single-phase form, where it compiles to 40 instead of 48
  // registers and measured 3-6 % faster (paper d = 4..8, profiles/r01_cols_u_ab/)
  const bool sp = nch > 1;
  auto go = [&](auto kern) {
    launch_k(kern, b, kThreads, 0, st, At, xt, yt, u, nk, v, su, sk, ntile, al, be, hb, rpc, ws);
    return done();
  };
  if (!AL && VEC <= 4 && (JR == 4 || (JR == 1 && nk <= 16))) {
    if (JR == 4)
      return sp ? go(k_cols<SD, C, 4, 3, false, true>) : go(k_cols<SD, C, 4, 3, false, false>);
    return go(k_cols<SD, C, 1, 3, false, true>);
  }
  static const int db_env = [] {  // TENVEC_B200_COLS_U_DB=0: single-buffered COLS_U, for A/B runs
    const char* e = getenv("TENVEC_B200_COLS_U_DB");
    return e ? atoi(e) : 1;
  }();
  if (!AL && JR == 8 && db_env != 0)
    return sp ? go(k_cols<SD, C, 8, UA_UNR, false, true, true>) : go(k_cols<SD, C, 8, UA_UNR, false, false, true>);
  switch (JR) {
    case 1: return (sp || !AL) ? go(k_cols<SD, C, 1, AL ? 8 : UA_UNR, AL, true>) : go(k_cols<SD, C, 1, AL ? 8 : UA_UNR, AL, false>);
    case 2: return sp ? go(k_cols<SD, C, 2, AL ? 8 : UA_UNR, AL, true>) : go(k_cols<SD, C, 2, AL ? 8 : UA_UNR, AL, false>);
    case 4: return sp ? go(k_cols<SD, C, 4, AL ? 4 : UA_UNR, AL, true>) : go(k_cols<SD, C, 4, AL ? 4 : UA_UNR, AL, false>);
    default: return sp ? go(k_cols<SD, C, 8, AL ? 4 : UA_UNR, AL, true>) : go(k_cols<SD, C, 8, AL ? 4 : UA_UNR, AL, false>);
  }
}

// split-K workspace bytes tv_tvc needs for this view (0: no split)
template <int SD, typename C>
static int64_t ws_bytes_typed(const void* A, int64_t u, int64_t nk, int64_t v, int64_t su, int64_t sk) {
  using T = typename St<SD>::T;
  if (u == 0 || v == 0) return 0;
  int64_t nch = 1;
  switch (regime_strided(A, (int)sizeof(T), u, nk, v, su, sk)) {
    case REG_COLS: nch = cols_split(cols_blocks<SD, true>(u, nk, v, nullptr, nullptr), nk); break;
    case REG_COLS_U: nch = cols_split(cols_blocks<SD, false>(u, nk, v, nullptr, nullptr), nk); break;
    case REG_SLABS:
    case REG_SLABS_U: nch = slabs_split(u, nk); break;
    case REG_FLAT_U: {
      int64_t rpc = nk;
      flat_u_split(u, nk, v, (int)VecN<SD>::N, flat_u_period(v, (int)VecN<SD>::N), &nch, &rpc);
      break;
    }
    case REG_STAGED_TALL: {
      int tr = 1;
      int64_t rpc = nk;
      staged_tall_split(u, nk, v, (int)sizeof(T), &tr, &nch, &rpc);
      break;
    }
    default: break;
  }
  return nch > 1 ? u * nch * v * (int64_t)sizeof(C) : 0;
}

template <int SD, typename C>
static int tvc_typed(const void* A, int64_t u, int64_t nk, int64_t v, int64_t su, int64_t sk,
                     const void* x, double alpha, double beta, void* y, const Ws& wsa, cudaStream_t st,
                     int naive) {
  using T = typename St<SD>::T;
  constexpr int VEC = VecN<SD>::N;
  const C al = (C)alpha, be = (C)beta;
  const int hb = beta != 0.0;
  if (u == 0 || v == 0) return TV_OK;
  const int reg = naive ? REG_GENERIC : regime_strided(A, (int)sizeof(T), u, nk, v, su, sk);
  int rc = TV_OK;
  switch (reg) {
    case REG_ROWS:
      launch_rows_auto<SD, C, false>(A, x, y, u, nk, su, al, be, hb, st);
      break;
    case REG_ROWS_U:
      launch_rows_auto<SD, C, true>(A, x, y, u, nk, su, al, be, hb, st);
      break;
    case REG_STAGED:
      launch_staged<SD, C>(A, x, y, u, nk, v, al, be, hb, st);
      break;
    case REG_STAGED_LONG:
      launch_staged_long<SD, C>(A, x, y, u, nk, v, al, be, hb, st);
      break;
    case REG_STAGED_TALL:
      rc = launch_staged_tall<SD, C>(A, x, y, u, nk, v, al, be, hb, wsa, st);
      break;
    case REG_ROWS_SHORT: {
      constexpr int UNR = 4;
      const int nkv = (int)(nk / VEC);
      const int64_t rows_per_block = kWarps * (32 / nkv) * UNR;
      const unsigned grid = grid_for(u, rows_per_block, 32);
      launch_k(k_rows_short<SD, C, UNR>, grid, kThreads, 0, st, (const T*)A, (const T*)x, (T*)y, u, (int)nk, su, al, be, hb);
      break;
    }
    case REG_COLS:
      rc = launch_cols<SD, C, true>(A, x, y, u, nk, v, su, sk, al, be, hb, wsa, st);
      break;
    case REG_COLS_U:
      rc = launch_cols<SD, C, false>(A, x, y, u, nk, v, su, sk, al, be, hb, wsa, st);
      break;
    case REG_FLAT_ROWS: {
      const int nkv = (int)(nk / VEC);
      const int S = nkv / gcd_small(32, nkv);
      const int rb = 32 * S / nkv;
      const int64_t nblocks = cdiv(u, rb);
      const T* At = (const T*)A;
      const T* xt = (const T*)x;
      T* yt = (T*)y;
      const int ik = (int)nk;
      switch (S) {
        case 1: launch_k(k_flat_rows<SD, C, 1, 8>, grid_for(nblocks, kWarps * 8, 32), kThreads, 0, st, At, xt, yt, u, ik, al, be, hb); break;
        case 3: launch_k(k_flat_rows<SD, C, 3, 2>, grid_for(nblocks, kWarps * 2, 32), kThreads, 0, st, At, xt, yt, u, ik, al, be, hb); break;
        case 5: launch_k(k_flat_rows<SD, C, 5, 1>, grid_for(nblocks, kWarps, 32), kThreads, 0, st, At, xt, yt, u, ik, al, be, hb); break;
        default: launch_k(k_flat_rows<SD, C, 7, 1>, grid_for(nblocks, kWarps, 32), kThreads, 0, st, At, xt, yt, u, ik, al, be, hb); break;
      }
      break;
    }
    case REG_FLAT: {
      const int vv = (int)(v / VEC);
      const int P = vv / gcd_small(32, vv);
      const size_t smem = (size_t)cdiv(nk * (int64_t)sizeof(C), 16) * 16 +
                          (size_t)kWarps * 32 * P * VEC * sizeof(C);
      const unsigned grid = grid_for(u, kWarps, 32);
      auto go = [&](auto kern) {
        if (smem > 48 * 1024)
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        launch_k(kern, grid, kThreads, smem, st, (const T*)A, (const T*)x, (T*)y, u, (int)nk, (int)v, al,
                                           be, hb);
      };
      if (P == 1) go(k_flat<SD, C, 1, 8>);
      else go(k_flat<SD, C, 3, 2>);
      break;
    }
    case REG_FLAT_U: {
      const int P = flat_u_period(v, VEC);
      int64_t nch = 1, rpc = nk;
      flat_u_split(u, nk, v, VEC, P, &nch, &rpc);
      C* ws = nullptr;
      if (nch > 1 && (ws = split_ws<C>(wsa, u * nch * v, st, &rc)) == nullptr) return rc;
      const size_t smem = (size_t)kWarps * 32 * P * VEC * sizeof(C);
      const unsigned grid = grid_for(u * nch, kWarps, 32);
      auto go = [&](auto kern) {
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        launch_k(kern, grid, kThreads, smem, st, (const T*)A, (const T*)x, (T*)y, u, nk, (int)v, su, al, be, hb,
                 nch, rpc, ws);
      };
      switch (P) {
        case 1: go(k_flat_u<SD, C, 1>); break;
        case 2: go(k_flat_u<SD, C, 2>); break;
        case 3: go(k_flat_u<SD, C, 3>); break;
        case 4: go(k_flat_u<SD, C, 4>); break;
        case 5: if constexpr (VEC <= 2) go(k_flat_u<SD, C, 5>); break;
        case 6: if constexpr (VEC <= 2) go(k_flat_u<SD, C, 6>); break;
        case 7: if constexpr (VEC <= 2) go(k_flat_u<SD, C, 7>); break;
        default: if constexpr (VEC <= 2) go(k_flat_u<SD, C, 8>); break;
      }
      if (ws != nullptr) split_finish<SD, C>(ws, wsa, nch, u, v, y, al, be, hb, st);
      break;
    }
    case REG_SLABS:
    case REG_SLABS_U: {
      // split-K when there are too few slabs for the GPU's warps
      const int64_t nch = slabs_split(u, nk);
      C* ws = nullptr;
      if (nch > 1 && (ws = split_ws<C>(wsa, u * nch * v, st, &rc)) == nullptr) return rc;
      const int64_t rpc = cdiv(nk, nch);
      const unsigned grid = grid_for(u * nch, kWarps, 32);
      static const int unr_env = [] {  // TENVEC_B200_SLAB_UNR=2: twice the batch depth, for A/B runs
        const char* e = getenv("TENVEC_B200_SLAB_UNR");
        return e ? atoi(e) : 1;
      }();
      if (reg == REG_SLABS) {
        if (unr_env == 2)
          launch_k(k_slabs<SD, C, 8, true>, grid, kThreads, 0, st, (const T*)A, (const T*)x, (T*)y, u, nk, (int)v,
                   su, sk, al, be, hb, nch, rpc, ws);
        else
          launch_k(k_slabs<SD, C, 4, true>, grid, kThreads, 0, st, (const T*)A, (const T*)x, (T*)y, u, nk, (int)v,
                   su, sk, al, be, hb, nch, rpc, ws);
      } else {
        if (unr_env == 2)
          launch_k(k_slabs<SD, C, 16, false>, grid, kThreads, 0, st, (const T*)A, (const T*)x, (T*)y, u, nk,
                   (int)v, su, sk, al, be, hb, nch, rpc, ws);
        else
          launch_k(k_slabs<SD, C, 8, false>, grid, kThreads, 0, st, (const T*)A, (const T*)x, (T*)y, u, nk,
                   (int)v, su, sk, al, be, hb, nch, rpc, ws);
      }
      if (ws != nullptr) split_finish<SD, C>(ws, wsa, nch, u, v, y, al, be, hb, st);
      break;
    }
    default: {
      if (v == 1) {
        const unsigned grid = grid_for(u, kWarps, 32);
        launch_k(k_naive_rows<SD, C>, grid, kThreads, 0, st, (const T*)A, (const T*)x, (T*)y, u, nk, su, sk, al, be, hb);
      } else {
        const unsigned grid = grid_for(u * v, kThreads, 32);
        launch_k(k_naive_cols<SD, C>, grid, kThreads, 0, st, (const T*)A, (const T*)x, (T*)y, u, nk, v,
                                                       su, sk, al, be, hb);
      }
    }
  }
  if (rc != TV_OK) return rc;
  return check_launch("tv_tvc");
}

template <int SD, typename C>
static int tvc_norm_typed(const void* A, int64_t u, int64_t nk, int64_t v, const void* x, void* y,
                          double* norm_out, int32_t* status, unsigned* counter, cudaStream_t st) {
  using T = typename St<SD>::T;
  constexpr int VEC = VecN<SD>::N;
  constexpr int NW = kNormThreads / 32;
  const int64_t ncb = cdiv(v, 32);
  const int64_t work = v == 1 ? cdiv(u, NW) : u * ncb;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(work, 2LL * sm_count()));
  const bool al = v == 1 && (reinterpret_cast<uintptr_t>(A) & 15) == 0 && nk % VEC == 0;
  if (al)
    launch_k(k_tvc_norm<SD, C, true>, grid, kNormThreads, 0, st, (const T*)A, (const T*)x, (T*)y, u, nk, v, ncb,
                                                           norm_out, status, counter);
  else
    launch_k(k_tvc_norm<SD, C, false>, grid, kNormThreads, 0, st, (const T*)A, (const T*)x, (T*)y, u, nk, v, ncb,
                                                            norm_out, status, counter);
  return check_launch("tv_tvc_normalize");
}

int tvc_dispatch(const void* A, int storage, int compute, int64_t u, int64_t nk, int64_t v,
                 int64_t su, int64_t sk, const void* x, double alpha, double beta, void* y,
                 void* stream, int naive, void* ws, int64_t ws_bytes, int ws_given) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const Ws w{ws, ws_bytes, ws_given != 0};
  switch (mode_id(storage, compute)) {
    case MODE_F64:
      return tvc_typed<TV_F64, double>(A, u, nk, v, su, sk, x, alpha, beta, y, w, st, naive);
    case MODE_F32:
      return tvc_typed<TV_F32, float>(A, u, nk, v, su, sk, x, alpha, beta, y, w, st, naive);
    case MODE_F32F64:
      return tvc_typed<TV_F32, double>(A, u, nk, v, su, sk, x, alpha, beta, y, w, st, naive);
    case MODE_F16F32:
      return tvc_typed<TV_F16, float>(A, u, nk, v, su, sk, x, alpha, beta, y, w, st, naive);
    case MODE_BF16F32:
      return tvc_typed<TV_BF16, float>(A, u, nk, v, su, sk, x, alpha, beta, y, w, st, naive);
    default:
      return set_error(TV_EMODE, "invalid (storage, compute) pair");
  }
}

const void* anchor_tvc() { return reinterpret_cast<const void*>(&k_naive_rows<TV_F64, double>); }

int64_t ws_bytes_dispatch(const void* A, int storage, int compute, int64_t u, int64_t nk, int64_t v,
                          int64_t su, int64_t sk) {
  switch (mode_id(storage, compute)) {
    case MODE_F64: return ws_bytes_typed<TV_F64, double>(A, u, nk, v, su, sk);
    case MODE_F32: return ws_bytes_typed<TV_F32, float>(A, u, nk, v, su, sk);
    case MODE_F32F64: return ws_bytes_typed<TV_F32, double>(A, u, nk, v, su, sk);
    case MODE_F16F32: return ws_bytes_typed<TV_F16, float>(A, u, nk, v, su, sk);
    case MODE_BF16F32: return ws_bytes_typed<TV_BF16, float>(A, u, nk, v, su, sk);
    default: return -1;
  }
}

}  // namespace tv

extern "C" int tv_tvc(const void* A, int storage, int compute, int64_t u, int64_t nk, int64_t v,
                      const void* x, double alpha, double beta, void* y, void* stream) {
  if (u < 0 || nk < 1 || v < 1)
    return tv::set_error(TV_EKERNEL, "tv_tvc: need u >= 0, nk >= 1, v >= 1");
  if ((u > 0 && (A == nullptr || y == nullptr)) || x == nullptr)
    return tv::set_error(TV_EKERNEL, "tv_tvc: null pointer");
  return tv::tvc_dispatch(A, storage, compute, u, nk, v, nk * v, v, x, alpha, beta, y, stream, 0,
                          nullptr, 0, 0);
}

extern "C" int tv_tvc_ws(const void* A, int storage, int compute, int64_t u, int64_t nk, int64_t v,
                         const void* x, double alpha, double beta, void* y, void* ws, int64_t ws_bytes,
                         void* stream) {
  if (u < 0 || nk < 1 || v < 1)
    return tv::set_error(TV_EKERNEL, "tv_tvc: need u >= 0, nk >= 1, v >= 1");
  if ((u > 0 && (A == nullptr || y == nullptr)) || x == nullptr)
    return tv::set_error(TV_EKERNEL, "tv_tvc: null pointer");
  return tv::tvc_dispatch(A, storage, compute, u, nk, v, nk * v, v, x, alpha, beta, y, stream, 0,
                          ws, ws_bytes, 1);
}

// ---------------------------------------------------------------- sweep ----
// The mode sweep of the paper's dTVC benchmarks: y_k = A x_k x_k for every
// mode k of one order-d tensor, independent outputs.  One regime launch per
// mode (exactly tv_tvc_ws's, so every y_k has tv_tvc's bits); modes after the
// first launch with programmatic stream serialization so a mode's ramp
// overlaps the previous mode's tail on small tensors.  Each mode's split-K
// workspace gets its own 256-byte-aligned slice (modes may overlap).
namespace {
struct SweepView {
  int64_t u, nk, v;
};

int sweep_views(int d, const int64_t* ext, SweepView* out) {
  if (d < 1 || d > 64 || ext == nullptr) return tv::set_error(TV_EKERNEL, "tv_tvc_sweep: need 1 <= d <= 64");
  for (int k = 0; k < d; ++k)
    if (ext[k] < 1) return tv::set_error(TV_EKERNEL, "tv_tvc_sweep: extents must be >= 1");
  for (int k = 0; k < d; ++k) {
    int64_t u = 1, v = 1;
    for (int i = 0; i < k; ++i) u *= ext[i];
    for (int i = k + 1; i < d; ++i) v *= ext[i];
    out[k] = {u, ext[k], v};
  }
  return TV_OK;
}

int64_t align256(int64_t b) { return (b + 255) & ~int64_t(255); }
}  // namespace

extern "C" int64_t tv_tvc_sweep_workspace_bytes(const void* A, int storage, int compute, int d,
                                                const int64_t* ext) {
  SweepView vw[64];
  if (sweep_views(d, ext, vw) != TV_OK) return -1;
  int64_t total = 0;
  for (int k = 0; k < d; ++k) {
    const int64_t b = tv::ws_bytes_dispatch(A, storage, compute, vw[k].u, vw[k].nk, vw[k].v,
                                            vw[k].nk * vw[k].v, vw[k].v);
    if (b < 0) return -1;
    total += align256(b);
  }
  return total;
}

extern "C" int tv_tvc_sweep(const void* A, int storage, int compute, int d, const int64_t* ext,
                            const void* const* xs, void* const* ys, void* ws, int64_t ws_bytes, void* stream) {
  SweepView vw[64];
  int rc = sweep_views(d, ext, vw);
  if (rc != TV_OK) return rc;
  if (A == nullptr || xs == nullptr || ys == nullptr) return tv::set_error(TV_EKERNEL, "tv_tvc_sweep: null pointer");
  char* wp = static_cast<char*>(ws);
  int64_t left = ws_bytes;
  for (int k = 0; k < d && rc == TV_OK; ++k) {
    if (xs[k] == nullptr || ys[k] == nullptr) {
      rc = tv::set_error(TV_EKERNEL, "tv_tvc_sweep: null vector or output");
      break;
    }
    const SweepView& w = vw[k];
    const int64_t need = align256(tv::ws_bytes_dispatch(A, storage, compute, w.u, w.nk, w.v, w.nk * w.v, w.v));
    if (need > left) {
      rc = tv::set_error(TV_EKERNEL, "tv_tvc_sweep: workspace smaller than tv_tvc_sweep_workspace_bytes");
      break;
    }
    tv::t_pdl = k > 0;
    rc = tv::tvc_dispatch(A, storage, compute, w.u, w.nk, w.v, w.nk * w.v, w.v, xs[k], 1.0, 0.0, ys[k], stream, 0,
                          need ? wp : nullptr, need, 1);
    wp += need;
    left -= need;
  }
  tv::t_pdl = false;
  return rc;
}

extern "C" int64_t tv_tvc_workspace_bytes(const void* A, int storage, int compute, int64_t u, int64_t nk,
                                          int64_t v) {
  if (u < 0 || nk < 1 || v < 1) return -1;
  return tv::ws_bytes_dispatch(A, storage, compute, u, nk, v, nk * v, v);
}

extern "C" int tv_tvc_naive(const void* A, int storage, int compute, int64_t u, int64_t nk,
                            int64_t v, const void* x, double alpha, double beta, void* y,
                            void* stream) {
  if (u < 0 || nk < 1 || v < 1)
    return tv::set_error(TV_EKERNEL, "tv_tvc_naive: need u >= 0, nk >= 1, v >= 1");
  if ((u > 0 && (A == nullptr || y == nullptr)) || x == nullptr)
    return tv::set_error(TV_EKERNEL, "tv_tvc_naive: null pointer");
  return tv::tvc_dispatch(A, storage, compute, u, nk, v, nk * v, v, x, alpha, beta, y, stream, 1,
                          nullptr, 0, 0);
}

extern "C" int tv_tvc_normalize(const void* A, int storage, int compute, int64_t u, int64_t nk,
                                int64_t v, const void* x, void* y, double* norm_out,
                                int32_t* status_out, unsigned* counter, void* stream) {
  using namespace tv;
  if (u < 1 || nk < 1 || v < 1) return set_error(TV_EKERNEL, "tv_tvc_normalize: need u, nk, v >= 1");
  if (!A || !x || !y || !norm_out || !counter) return set_error(TV_EKERNEL, "tv_tvc_normalize: null pointer");
  if (u * v > kTvcNormMax || u * nk * v > 64 * kTvcNormMax)
    return set_error(TV_EKERNEL, "tv_tvc_normalize: view too large (use tv_tvc + tv_normalize)");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (mode_id(storage, compute)) {
    case MODE_F64: return tvc_norm_typed<TV_F64, double>(A, u, nk, v, x, y, norm_out, status_out, counter, st);
    case MODE_F32: return tvc_norm_typed<TV_F32, float>(A, u, nk, v, x, y, norm_out, status_out, counter, st);
    case MODE_F32F64: return tvc_norm_typed<TV_F32, double>(A, u, nk, v, x, y, norm_out, status_out, counter, st);
    case MODE_F16F32: return tvc_norm_typed<TV_F16, float>(A, u, nk, v, x, y, norm_out, status_out, counter, st);
    case MODE_BF16F32: return tvc_norm_typed<TV_BF16, float>(A, u, nk, v, x, y, norm_out, status_out, counter, st);
    default: return set_error(TV_EMODE, "invalid (storage, compute) pair");
  }
}

extern "C" int tv_tvc_regime(const void* A, int storage, int64_t u, int64_t nk, int64_t v) {
  return tv::regime_of(A, storage, u, nk, v);
}

extern "C" int tv_set_regime_override(int regime) {
  const int prev = tv::forced_regime();
  tv::g_forced.store(regime > 0 ? regime : -1, std::memory_order_relaxed);
  return prev;
}

static int getvc_impl(int trans, const void* A, int storage, int compute, int64_t m, int64_t n,
                      int64_t lda, const void* x, double alpha, double beta, void* y, void* stream,
                      void* ws, int64_t ws_bytes, int given) {
  if (m < 0 || n < 0 || lda < n) return tv::set_error(TV_EKERNEL, "tv_getvc: need lda >= n >= 0");
  if (trans == 0) {  // matvec: y[i] = sum_j A[i*lda + j] x[j]
    if (m == 0) return TV_OK;
    if (n == 0) return tv::set_error(TV_EKERNEL, "tv_getvc: empty contraction");
    return tv::tvc_dispatch(A, storage, compute, m, n, 1, lda, 1, x, alpha, beta, y, stream, 0, ws,
                            ws_bytes, given);
  }
  if (trans == 1) {  // vecmat: y[c] = sum_i x[i] A[i*lda + c]
    if (n == 0) return TV_OK;
    if (m == 0) return tv::set_error(TV_EKERNEL, "tv_getvc: empty contraction");
    return tv::tvc_dispatch(A, storage, compute, 1, m, n, 0, lda, x, alpha, beta, y, stream, 0, ws,
                            ws_bytes, given);
  }
  return tv::set_error(TV_EKERNEL, "tv_getvc: trans must be 0 (matvec) or 1 (vecmat)");
}

extern "C" int tv_getvc(int trans, const void* A, int storage, int compute, int64_t m, int64_t n,
                        int64_t lda, const void* x, double alpha, double beta, void* y,
                        void* stream) {
  return getvc_impl(trans, A, storage, compute, m, n, lda, x, alpha, beta, y, stream, nullptr, 0, 0);
}

extern "C" int tv_getvc_ws(int trans, const void* A, int storage, int compute, int64_t m, int64_t n,
                           int64_t lda, const void* x, double alpha, double beta, void* y, void* ws,
                           int64_t ws_bytes, void* stream) {
  return getvc_impl(trans, A, storage, compute, m, n, lda, x, alpha, beta, y, stream, ws, ws_bytes, 1);
}

extern "C" int64_t tv_getvc_workspace_bytes(int trans, const void* A, int storage, int compute, int64_t m,
                                            int64_t n, int64_t lda) {
  if (m < 0 || n < 0 || lda < n) return -1;
  if (trans == 0) return m == 0 || n == 0 ? 0 : tv::ws_bytes_dispatch(A, storage, compute, m, n, 1, lda, 1);
  if (trans == 1) return m == 0 || n == 0 ? 0 : tv::ws_bytes_dispatch(A, storage, compute, 1, m, n, 0, lda);
  return -1;
}
