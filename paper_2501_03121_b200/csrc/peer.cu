// Device-side rendezvous of the one-process-per-GPU transports (RankGroup's
// "fused" and "p2p" algorithms) over peer memory.
//
// The reference's collectives meet in a host rendezvous slot with a timeout
// that names the ranks that never arrived (pkg/src/tenvec/comm.py:202-235).
// Here every rank owns a peer-mapped buffer (torch symmetric memory across
// GPUs, or plain device buffers when p thread-ranks share one GPU) whose
// first TV_PEER_HEADER bytes hold an arrival word per rank.  A barrier is one
// single-CTA kernel in stream order: it posts this rank's epoch into every
// peer's word for this rank (release, system scope) and waits until its own
// words from every peer reach the epoch (acquire, system scope).  It never
// traps: past the timeout it records TV_ECOLL, the epoch and the bit mask of
// the ranks still missing into a device status block and returns; later
// barriers of a failed group post their arrival without waiting, so a dead
// peer costs one timeout, not one per barrier, and the host raises
// CollectiveTimeout(kind, absent) when it reads the status.

#include <cuda.h>
#include <stdint.h>

#include "tv_internal.h"

namespace tv {

struct PeerWords {
  uint32_t* p[TV_MAX_RANKS];
};

__device__ __forceinline__ void st_release_sys(uint32_t* a, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* a) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// status: [0] code (0 ok / TV_ECOLL), [1] failed epoch, [2] absent mask bits
// 0-31, [3] bits 32-63
__global__ void __launch_bounds__(TV_MAX_RANKS)
    k_peer_barrier(PeerWords w, int p, int rank, uint32_t epoch, long long timeout_ns,
                   int32_t* __restrict__ status) {
  __shared__ unsigned missing_lo, missing_hi;
  const int t = threadIdx.x;
  if (t == 0) missing_lo = missing_hi = 0u;
  const bool failed = *reinterpret_cast<volatile int32_t*>(status) != 0;
  // everything this rank wrote before the barrier (earlier kernels on this
  // stream, e.g. partial sums stored into peer slots) is visible system-wide
  // before its arrival word is
  __threadfence_system();
  __syncthreads();
  if (t < p) st_release_sys(w.p[t] + rank, epoch);
  if (failed) return;
  if (t < p) {
    const uint32_t* mine = w.p[rank] + t;
    const uint64_t t0 = globaltimer_ns();
    while ((int32_t)(ld_acquire_sys(mine) - epoch) < 0) {
      if (timeout_ns > 0 && (long long)(globaltimer_ns() - t0) > timeout_ns) {
        if (t < 32) atomicOr(&missing_lo, 1u << t);
        else atomicOr(&missing_hi, 1u << (t - 32));
        break;
      }
      __nanosleep(256);
    }
  }
  __syncthreads();
  if (t == 0 && (missing_lo | missing_hi)) {
    status[1] = (int32_t)epoch;
    status[2] = (int32_t)missing_lo;
    status[3] = (int32_t)missing_hi;
    __threadfence();
    status[0] = TV_ECOLL;
  }
  __threadfence_system();
}

}  // namespace tv

extern "C" int tv_peer_barrier(void* const* peer_bases, int p, int rank, uint32_t epoch,
                               int64_t timeout_ns, int32_t* status, void* stream) {
  using namespace tv;
  if (!peer_bases || !status || p < 1 || p > TV_MAX_RANKS || rank < 0 || rank >= p || epoch == 0)
    return set_error(TV_ECOLL, "tv_peer_barrier: bad arguments");
  PeerWords w{};
  for (int r = 0; r < p; ++r) {
    if (!peer_bases[r] || (reinterpret_cast<uintptr_t>(peer_bases[r]) & 3))
      return set_error(TV_ECOLL, "tv_peer_barrier: null or misaligned peer buffer");
    w.p[r] = static_cast<uint32_t*>(peer_bases[r]);
  }
  k_peer_barrier<<<1, TV_MAX_RANKS, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      w, p, rank, epoch, (long long)timeout_ns, status);
  return launched("tv_peer_barrier");
}

// Lazy module loading (the CUDA 12 default) loads a kernel at its first
// launch, and loading may wait for the kernels already running on the device.
// A kernel first launched while a tv_peer_barrier spins -- on this GPU for a
// side-stream barrier, or for a peer thread-rank sharing the GPU -- would then
// wait for the barrier, which waits for it.  tv_preload loads every kernel of
// every translation unit up front (driver entry points of CUDA >= 12.4, looked
// up at run time: no link against libcuda).
namespace {
using PFuncGetModule = CUresult (*)(CUmodule*, CUfunction);
using PModFnCount = CUresult (*)(unsigned*, CUmodule);
using PModEnum = CUresult (*)(CUfunction*, unsigned, CUmodule);
using PFuncLoad = CUresult (*)(CUfunction);

template <typename F>
F entry(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPointByVersion(name, &fn, 12040, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return reinterpret_cast<F>(fn);
}
}  // namespace

extern "C" int tv_preload(int* loaded) {
  using namespace tv;
  const void* anchors[3] = {anchor_tvc(), anchor_util(), reinterpret_cast<const void*>(&k_peer_barrier)};
  auto get_mod = entry<PFuncGetModule>("cuFuncGetModule");
  auto count = entry<PModFnCount>("cuModuleGetFunctionCount");
  auto enumerate = entry<PModEnum>("cuModuleEnumerateFunctions");
  auto load = entry<PFuncLoad>("cuFuncLoad");
  int n_loaded = 0;
  for (const void* a : anchors) {
    cudaFunction_t f = nullptr;
    if (cudaGetFuncBySymbol(&f, a) != cudaSuccess) return check_launch("tv_preload: cudaGetFuncBySymbol");
    if (!get_mod || !count || !enumerate || !load) {
      // driver without the enumeration API: the anchors at least
      cudaFuncAttributes attr;
      if (cudaFuncGetAttributes(&attr, a) != cudaSuccess) return check_launch("tv_preload");
      ++n_loaded;
      continue;
    }
    CUmodule mod = nullptr;
    unsigned nf = 0;
    if (get_mod(&mod, reinterpret_cast<CUfunction>(f)) != CUDA_SUCCESS || count(&nf, mod) != CUDA_SUCCESS)
      return set_error(TV_ECUDA, "tv_preload: cannot enumerate the module's kernels");
    CUfunction fs[1024];
    if (nf > 1024) return set_error(TV_ECUDA, "tv_preload: more than 1024 kernels in one module");
    if (enumerate(fs, nf, mod) != CUDA_SUCCESS)
      return set_error(TV_ECUDA, "tv_preload: cannot enumerate the module's kernels");
    for (unsigned i = 0; i < nf; ++i) {
      if (load(fs[i]) != CUDA_SUCCESS) return set_error(TV_ECUDA, "tv_preload: cuFuncLoad failed");
      ++n_loaded;
    }
  }
  if (loaded) *loaded = n_loaded;
  return TV_OK;
}
