// The distributed layer as a C-ABI: communicators, the reference-ordered
// allreduce / allgather of comm.py, and the dHOPM3 sweep of hopm.py, so a
// caller without Python (a C/C++ host, or another language over its FFI)
// drives dTVC and dHOPM3 across the GPUs of a box through this library alone.
//
//   tv_comm_*            one NCCL communicator per rank (ncclCommInitRank /
//                        ncclCommInitAll), resolved from the process's
//                        libnccl.so.2 at run time (torch's when loaded)
//   tv_allreduce         comm.py:84-134: the reference's value order -- the
//                        ascending-rank fold or the mixed ring -- bit-equal on
//                        every rank, or ncclAllReduce (TV_AR_NCCL)
//   tv_allgather         comm.py:137-153: rank-order concatenation of unequal
//                        parts (one grouped broadcast per root, no padding)
//   tv_dhopm3_*          hopm.py:229-354: a plan (schedule, three rotating
//                        buffers, workspaces) and one call per sweep; the
//                        same kernels and the same bits as the Python dhopm3
//
// Host code only (the kernels are tv_tvc_ws, tv_rank_fold*, tv_normalize);
// everything is enqueued on the caller's stream.

#include <cuda.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "tv_internal.h"

namespace {

// ----------------------------------------------------------------- NCCL ----
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
  bool ok;
};

NcclApi* nccl() {
  static NcclApi api{};
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's, if loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    bool ok = true;
    auto get = [&](const char* n) {
      void* f = dlsym(h, n);
      ok = ok && f != nullptr;
      return f;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(get("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(get("ncclCommInitRank"));
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(get("ncclCommInitAll"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(get("ncclCommDestroy"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(get("ncclAllGather"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(get("ncclAllReduce"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(get("ncclBroadcast"));
    api.Send = reinterpret_cast<decltype(api.Send)>(get("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(get("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(get("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(get("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(get("ncclGetErrorString"));
    api.ok = ok;
  });
  return api.ok ? &api : nullptr;
}

int nccl_error(ncclResult_t r, const char* what) {
  std::string m = std::string(what) + ": " + (nccl() ? nccl()->GetErrorString(r) : "NCCL unavailable");
  return tv::set_error(TV_ECOLL, m.c_str());
}

#define NCCL_CHECK(call, what)                       \
  do {                                               \
    ncclResult_t r_ = (call);                        \
    if (r_ != ncclSuccess) return nccl_error(r_, what); \
  } while (0)

struct Comm {
  ncclComm_t c;
  int rank, size, dev;
};

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
int64_t a256(int64_t b) { return (b + 255) & ~int64_t(255); }

// -------------------------------------------------------------- allreduce --
// the reference order (comm.py:84-134) from NCCL data movement + the fold
// kernel: small buffers (<= 1 MB over all ranks) gather every rank's buffer
// and fold all ring chunks locally; larger ones exchange ring chunks
// (all-to-all by grouped send/recv), fold chunk `rank`, and gather the
// folded chunks -- a ring allreduce's traffic.
constexpr int64_t kSmallGather = 1 << 20;

int64_t allreduce_ws(int p, int64_t n, int sb, int algo) {
  if (p == 1 || algo == TV_AR_NCCL) return 0;
  if (n * sb * p <= kSmallGather) return a256(p * n * sb);
  const int64_t q = cdiv(n, p);
  return a256(p * q * sb) + a256(q * sb) + a256(p * q * sb);
}

int allreduce_impl(Comm* cm, void* buf, int64_t n, int storage, int compute, int algo, void* ws, int64_t ws_bytes,
                   cudaStream_t st) {
  const int p = cm->size, rank = cm->rank;
  const int sb = tv::dtype_bytes(storage);
  if (sb <= 0 || tv::mode_id(storage, compute) == tv::MODE_INVALID)
    return tv::set_error(TV_EMODE, "tv_allreduce: invalid (storage, compute) pair");
  if (n < 0 || (algo != TV_AR_NCCL && algo != TV_AR_EXACT && algo != TV_AR_MIXED))
    return tv::set_error(TV_ECOLL, "tv_allreduce: bad length or algorithm");
  if (p == 1 || n == 0) return TV_OK;
  NcclApi* N = nccl();
  if (!N) return tv::set_error(TV_ECOLL, "tv_allreduce: libnccl.so.2 not found");
  if (algo == TV_AR_NCCL) {
    if (storage != compute) return tv::set_error(TV_ECOLL, "tv_allreduce: TV_AR_NCCL sums exact-width data only");
    const ncclDataType_t t = storage == TV_F64 ? ncclFloat64 : ncclFloat32;
    NCCL_CHECK(N->AllReduce(buf, buf, (size_t)n, t, ncclSum, cm->c, st), "tv_allreduce");
    return TV_OK;
  }
  const int mixed = algo == TV_AR_MIXED ? 1 : 0;
  if (allreduce_ws(p, n, sb, algo) > ws_bytes || (ws == nullptr && ws_bytes > 0))
    return tv::set_error(TV_ECOLL, "tv_allreduce: workspace smaller than tv_allreduce_workspace_bytes");
  char* w = static_cast<char*>(ws);
  const int64_t q = cdiv(n, p);
  if (n * sb * p <= kSmallGather) {
    NCCL_CHECK(N->AllGather(buf, w, (size_t)(n * sb), ncclUint8, cm->c, st), "tv_allreduce: gather");
    return tv_rank_fold_strided(w, n, p, n, q, 0, storage, compute, mixed, buf, st);
  }
  char* recv = w;
  char* mine = w + a256(p * q * sb);
  char* gathered = mine + a256(q * sb);
  const int64_t my_n = std::max<int64_t>(0, std::min<int64_t>(q, n - rank * q));
  NCCL_CHECK(N->GroupStart(), "tv_allreduce: group");
  for (int r = 0; r < p; ++r) {
    const int64_t cnt = std::max<int64_t>(0, std::min<int64_t>(q, n - r * q));
    if (cnt > 0) NCCL_CHECK(N->Send(static_cast<char*>(buf) + r * q * sb, (size_t)(cnt * sb), ncclUint8, r, cm->c, st),
                            "tv_allreduce: send");
    if (my_n > 0) NCCL_CHECK(N->Recv(recv + r * my_n * sb, (size_t)(my_n * sb), ncclUint8, r, cm->c, st),
                             "tv_allreduce: recv");
  }
  NCCL_CHECK(N->GroupEnd(), "tv_allreduce: group");
  if (my_n > 0) {
    const int rc = tv_rank_fold_strided(recv, my_n, p, my_n, 0, rank, storage, compute, mixed, mine, st);
    if (rc != TV_OK) return rc;
  }
  NCCL_CHECK(N->AllGather(mine, gathered, (size_t)(q * sb), ncclUint8, cm->c, st), "tv_allreduce: gather");
  // chunk c sits at [c q, c q + size_c); only the tail is short
  if (cudaMemcpyAsync(buf, gathered, (size_t)(n * sb), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return tv::check_launch("tv_allreduce: copy");
  return TV_OK;
}

int allgather_impl(Comm* cm, const void* local, void* out, const int64_t* counts, int elem_bytes, cudaStream_t st) {
  NcclApi* N = nccl();
  if (!N) return tv::set_error(TV_ECOLL, "tv_allgather: libnccl.so.2 not found");
  const int p = cm->size;
  int64_t off = 0;
  NCCL_CHECK(N->GroupStart(), "tv_allgather: group");
  for (int r = 0; r < p; ++r) {
    if (counts[r] > 0)
      NCCL_CHECK(N->Broadcast(local, static_cast<char*>(out) + off * elem_bytes, (size_t)(counts[r] * elem_bytes),
                              ncclUint8, r, cm->c, st),
                 "tv_allgather: broadcast");
    off += counts[r];
  }
  NCCL_CHECK(N->GroupEnd(), "tv_allgather: group");
  return TV_OK;
}

// ----------------------------------------------------------------- dHOPM3 --
// The reuse schedule (costmodel.py:138-153): iteration j = 0 contracts
// 1..d-1 from A; j = 1 contracts 0, 2..d-1 from A; j >= 2 starts from the
// carried tensor W (modes 0..j-2 gone) and contracts j-1 then j+1..d-1.  The
// first product of an iteration is W for the next.
struct Step {
  int k;          // original mode contracted
  int64_t u, nk, v;
  bool split;     // contracts the split mode of an undivided slab: local x slice
  int slot;       // output buffer
  bool from_w;    // input is the carried tensor (else the previous product / A)
};

struct Iter {
  std::vector<Step> steps;
  bool fused_norm;  // p == 1: the last TVC normalises in its epilogue
  int64_t out_n;    // elements of the iteration's final product
};

struct Hopm {
  Comm* comm;      // nullptr: one rank
  int p, rank;
  const void* A;
  int storage, compute, sb, d, s;
  std::vector<int64_t> ext, loc;  // global / local extents
  int64_t lo, hi;
  std::vector<Iter> iters;
  void* bufs[3];
  void* ws;  // split-K workspace (max over the schedule) + collective workspace
  int64_t tvc_ws, coll_ws;
  void* gather;  // p * max extent (allreduce of the iteration vectors)
  unsigned* counter;
  int32_t* status;
};

void iteration_modes(int d, int j, std::vector<int>& modes, int& first_contracted) {
  modes.clear();
  first_contracted = 0;
  if (j == 0) {
    for (int k = 1; k < d; ++k) modes.push_back(k);
  } else if (j == 1) {
    modes.push_back(0);
    for (int k = 2; k < d; ++k) modes.push_back(k);
  } else {
    first_contracted = j - 1;  // modes 0..j-2 already folded into W
    modes.push_back(j - 1);
    for (int k = j + 1; k < d; ++k) modes.push_back(k);
  }
}

// (u, nk, v) of contracting original mode k of a tensor whose modes `gone`
// are contracted, local extents loc (the split mode's extent is the slab's)
void view_of(const std::vector<int64_t>& loc, const std::vector<bool>& gone, int k, int64_t& u, int64_t& nk,
             int64_t& v) {
  u = 1;
  v = 1;
  for (int i = 0; i < (int)loc.size(); ++i) {
    if (gone[i]) continue;
    if (i < k) u *= loc[i];
    if (i > k) v *= loc[i];
  }
  nk = loc[k];
}

int build_schedule(Hopm* h) {
  const int d = h->d;
  // the rotation of hopm.py's three buffers: an iteration's first product
  // goes to a buffer other than the carried one, later products alternate
  // between the remaining two
  int w_idx = -1;
  int64_t max_out = 1;
  h->iters.assign(d, Iter{});
  // the slot pattern depends on w_idx at sweep entry; it is periodic after the
  // first sweep, so the schedule is built for a steady-state sweep (entry
  // w_idx = the last sweep's final W slot) by running it twice
  for (int pass = 0; pass < 2; ++pass) {
    for (int j = 0; j < d; ++j) {
      std::vector<int> modes;
      int pre = 0;
      iteration_modes(d, j, modes, pre);
      std::vector<bool> gone(d, false);
      bool partial = false;
      const bool from_w = j >= 2;
      if (from_w) {
        for (int i = 0; i < pre; ++i) gone[i] = true;
        partial = h->s < pre;  // the split mode was contracted into W
      }
      int pool[3];
      if (w_idx < 0) {
        pool[0] = 0, pool[1] = 1, pool[2] = 2;
      } else {
        int c = 0;
        for (int i = 0; i < 3; ++i)
          if (i != w_idx) pool[c++] = i;
        pool[2] = w_idx;
      }
      Iter it;
      it.fused_norm = false;
      int new_w = w_idx;
      for (int t = 0; t < (int)modes.size(); ++t) {
        Step st{};
        st.k = modes[t];
        st.split = st.k == h->s && !partial;
        view_of(h->loc, gone, st.k, st.u, st.nk, st.v);
        st.slot = t == 0 ? pool[0] : pool[1 + (t - 1) % 2];
        st.from_w = from_w && t == 0;
        gone[st.k] = true;
        partial = partial || st.split;
        max_out = std::max(max_out, st.u * st.v);
        if (t == 0) new_w = st.slot;
        it.steps.push_back(st);
        it.out_n = st.u * st.v;
      }
      w_idx = new_w;
      const Step& last = it.steps.back();
      const bool carried = modes.size() == 1 && 1 <= j && j <= d - 2;  // its output is W
      it.fused_norm = h->p == 1 && !carried && last.u * last.v <= (1LL << 22) &&
                      last.u * last.nk * last.v <= 64 * (1LL << 22);
      if (pass == 1) h->iters[j] = it;
    }
  }
  for (int i = 0; i < 3; ++i)
    if (cudaMalloc(&h->bufs[i], (size_t)(max_out * h->sb)) != cudaSuccess)
      return tv::check_launch("tv_dhopm3_plan_create: buffers");
  // split-K workspace: the largest any step of the sweep asks for
  int64_t need = 0;
  for (const Iter& it : h->iters)
    for (size_t t = 0; t < it.steps.size(); ++t) {
      const Step& st = it.steps[t];
      const void* in = t == 0 && !st.from_w ? h->A : h->bufs[0];  // the buffers share one alignment
      need = std::max(need, tv::ws_bytes_dispatch(in, h->storage, h->compute, st.u, st.nk, st.v, st.nk * st.v, st.v));
    }
  h->tvc_ws = a256(need);
  int64_t emax = 1;
  for (int64_t e : h->ext) emax = std::max(emax, e);
  h->coll_ws = h->p > 1 ? a256(h->p * emax * h->sb) : 0;
  if (h->tvc_ws + h->coll_ws > 0 && cudaMalloc(&h->ws, (size_t)(h->tvc_ws + h->coll_ws)) != cudaSuccess)
    return tv::check_launch("tv_dhopm3_plan_create: workspace");
  if (cudaMalloc(&h->counter, 256) != cudaSuccess) return tv::check_launch("tv_dhopm3_plan_create: counter");
  // zero before any stream can use it (the caller's streams may not
  // synchronise with the legacy default stream)
  if (cudaMemset(h->counter, 0, 256) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
    return tv::check_launch("tv_dhopm3_plan_create: counter");
  h->status = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(h->counter) + 128);
  return TV_OK;
}

int dhopm3_sweep(Hopm* h, void* const* x, double* norms, int32_t* status, cudaStream_t st) {
  const int d = h->d;
  int32_t* stat = status ? status : h->status;
  for (int j = 0; j < d; ++j) {
    const Iter& it = h->iters[j];
    const void* cur = nullptr;
    for (size_t t = 0; t < it.steps.size(); ++t) {
      const Step& sp = it.steps[t];
      // the first product reads A, or the carried W: where the previous
      // iteration's first product went
      const void* in = t > 0 ? cur : sp.from_w ? h->bufs[h->iters[j - 1].steps.front().slot] : h->A;
      const char* vec = static_cast<const char*>(x[sp.k]) + (sp.split ? h->lo * h->sb : 0);
      const bool last = t + 1 == it.steps.size();
      if (last && it.fused_norm) {
        const int rc = tv_tvc_normalize(in, h->storage, h->compute, sp.u, sp.nk, sp.v, vec, x[j], norms + j, stat,
                                        h->counter, st);
        if (rc != TV_OK) return rc;
        cur = x[j];
        break;
      }
      const int rc = tv::tvc_dispatch(in, h->storage, h->compute, sp.u, sp.nk, sp.v, sp.nk * sp.v, sp.v, vec, 1.0,
                                      0.0, h->bufs[sp.slot], st, 0, h->tvc_ws ? h->ws : nullptr, h->tvc_ws, 1);
      if (rc != TV_OK) return rc;
      cur = h->bufs[sp.slot];
    }
    if (it.fused_norm) continue;
    // the iteration's one collective (hopm.py:320-329), then the
    // normalisation every rank repeats
    if (h->p == 1) {
      if (cudaMemcpyAsync(x[j], cur, (size_t)(it.out_n * h->sb), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return tv::check_launch("tv_dhopm3_sweep: copy");
      const int rc = tv_normalize(x[j], h->storage, h->compute, h->ext[j], norms + j, stat, st);
      if (rc != TV_OK) return rc;
    } else if (j == h->s) {
      std::vector<int64_t> counts(h->p);
      const int64_t q = cdiv(h->ext[h->s], h->p);
      for (int r = 0; r < h->p; ++r) counts[r] = std::max<int64_t>(0, std::min<int64_t>(q, h->ext[h->s] - r * q));
      int rc = allgather_impl(h->comm, cur, x[j], counts.data(), h->sb, st);
      if (rc != TV_OK) return rc;
      rc = tv_normalize(x[j], h->storage, h->compute, h->ext[j], norms + j, stat, st);
      if (rc != TV_OK) return rc;
    } else {
      // every rank's vector gathered, all ring chunks folded locally in the
      // reference order with the normalisation in the fold's epilogue
      NcclApi* N = nccl();
      const int64_t n = h->ext[j];
      char* g = static_cast<char*>(h->ws) + h->tvc_ws;
      NCCL_CHECK(N->AllGather(cur, g, (size_t)(n * h->sb), ncclUint8, h->comm->c, st), "tv_dhopm3_sweep: gather");
      const int mixed = h->storage != h->compute ? 1 : 0;
      const int rc = tv_rank_fold_normalize(g, n, h->p, n, cdiv(n, h->p), h->storage, h->compute, mixed, x[j],
                                            norms + j, stat, h->counter, st);
      if (rc != TV_OK) return rc;
    }
  }
  return TV_OK;
}

}  // namespace

// =================================================================== C-ABI ==

extern "C" int tv_comm_get_unique_id(void* id_out) {
  NcclApi* N = nccl();
  if (!N) return tv::set_error(TV_ECOLL, "tv_comm_get_unique_id: libnccl.so.2 not found");
  if (!id_out) return tv::set_error(TV_ECOLL, "tv_comm_get_unique_id: null output");
  ncclUniqueId id;
  NCCL_CHECK(N->GetUniqueId(&id), "tv_comm_get_unique_id");
  std::memcpy(id_out, &id, sizeof(id));
  return TV_OK;
}

extern "C" int tv_comm_init_rank(const void* id, int nranks, int rank, void** comm_out) {
  NcclApi* N = nccl();
  if (!N) return tv::set_error(TV_ECOLL, "tv_comm_init_rank: libnccl.so.2 not found");
  if (!id || !comm_out || nranks < 1 || rank < 0 || rank >= nranks || nranks > TV_MAX_RANKS)
    return tv::set_error(TV_ECOLL, "tv_comm_init_rank: bad arguments");
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  Comm* c = new Comm{};
  cudaGetDevice(&c->dev);
  const ncclResult_t r = N->CommInitRank(&c->c, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_error(r, "tv_comm_init_rank");
  }
  c->rank = rank;
  c->size = nranks;
  *comm_out = c;
  return TV_OK;
}

extern "C" int tv_comm_init_all(int ndev, const int* devs, void** comms_out) {
  NcclApi* N = nccl();
  if (!N) return tv::set_error(TV_ECOLL, "tv_comm_init_all: libnccl.so.2 not found");
  if (ndev < 1 || ndev > TV_MAX_RANKS || !devs || !comms_out) return tv::set_error(TV_ECOLL, "tv_comm_init_all: bad arguments");
  std::vector<ncclComm_t> cs(ndev);
  NCCL_CHECK(N->CommInitAll(cs.data(), ndev, devs), "tv_comm_init_all");
  for (int i = 0; i < ndev; ++i) comms_out[i] = new Comm{cs[i], i, ndev, devs[i]};
  return TV_OK;
}

extern "C" int tv_comm_destroy(void* comm) {
  if (!comm) return TV_OK;
  Comm* c = static_cast<Comm*>(comm);
  NcclApi* N = nccl();
  if (N) N->CommDestroy(c->c);
  delete c;
  return TV_OK;
}

extern "C" int tv_comm_rank_size(void* comm, int* rank, int* size) {
  if (!comm) return tv::set_error(TV_ECOLL, "tv_comm_rank_size: null communicator");
  Comm* c = static_cast<Comm*>(comm);
  if (rank) *rank = c->rank;
  if (size) *size = c->size;
  return TV_OK;
}

extern "C" int64_t tv_allreduce_workspace_bytes(void* comm, int64_t n, int storage, int algo) {
  if (!comm || n < 0) return -1;
  const int sb = tv::dtype_bytes(storage);
  if (sb <= 0) return -1;
  return allreduce_ws(static_cast<Comm*>(comm)->size, n, sb, algo);
}

extern "C" int tv_allreduce(void* comm, void* buf, int64_t n, int storage, int compute, int algo, void* ws,
                            int64_t ws_bytes, void* stream) {
  if (!comm || (!buf && n > 0)) return tv::set_error(TV_ECOLL, "tv_allreduce: null communicator or buffer");
  return allreduce_impl(static_cast<Comm*>(comm), buf, n, storage, compute, algo, ws, ws_bytes,
                        reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int tv_allgather(void* comm, const void* local, void* out, const int64_t* counts, int elem_bytes,
                            void* stream) {
  if (!comm || !out || !counts || elem_bytes < 1) return tv::set_error(TV_ECOLL, "tv_allgather: bad arguments");
  return allgather_impl(static_cast<Comm*>(comm), local, out, counts, elem_bytes,
                        reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int tv_dhopm3_plan_destroy(void* plan);

extern "C" int tv_dhopm3_plan_create(void* comm, const void* A, int storage, int compute, int d, const int64_t* ext,
                                     int s, void** plan_out) {
  if (!A || !ext || !plan_out || d < 2 || d > 64 || s < 0 || s >= d)
    return tv::set_error(TV_EKERNEL, "tv_dhopm3_plan_create: bad arguments");
  if (tv::mode_id(storage, compute) == tv::MODE_INVALID)
    return tv::set_error(TV_EMODE, "tv_dhopm3_plan_create: invalid (storage, compute) pair");
  for (int i = 0; i < d; ++i)
    if (ext[i] < 1) return tv::set_error(TV_EKERNEL, "tv_dhopm3_plan_create: extents must be >= 1");
  Hopm* h = new Hopm{};
  h->comm = static_cast<Comm*>(comm);
  h->p = h->comm ? h->comm->size : 1;
  h->rank = h->comm ? h->comm->rank : 0;
  h->A = A;
  h->storage = storage;
  h->compute = compute;
  h->sb = tv::dtype_bytes(storage);
  h->d = d;
  h->s = s;
  h->ext.assign(ext, ext + d);
  // the rank's slab of the split (tensor.py:105-138): ceil(n/p) per rank
  const int64_t q = cdiv(ext[s], h->p);
  if (cdiv(ext[s], q) != h->p) {
    delete h;
    return tv::set_error(TV_ECOLL, "tv_dhopm3_plan_create: the split mode is too short for every rank to own a slab");
  }
  h->lo = h->rank * q;
  h->hi = std::min(ext[s], h->lo + q);
  h->loc = h->ext;
  h->loc[s] = h->hi - h->lo;
  const int rc = build_schedule(h);
  if (rc != TV_OK) {
    tv_dhopm3_plan_destroy(h);  // frees whatever build_schedule allocated
    return rc;
  }
  *plan_out = h;
  return TV_OK;
}

extern "C" int tv_dhopm3_plan_slab(void* plan, int64_t* lo, int64_t* hi) {
  if (!plan) return tv::set_error(TV_EKERNEL, "tv_dhopm3_plan_slab: null plan");
  Hopm* h = static_cast<Hopm*>(plan);
  if (lo) *lo = h->lo;
  if (hi) *hi = h->hi;
  return TV_OK;
}

extern "C" int tv_dhopm3_sweep(void* plan, void* const* x, double* norms_out, int32_t* status_out, void* stream) {
  if (!plan || !x || !norms_out) return tv::set_error(TV_EKERNEL, "tv_dhopm3_sweep: bad arguments");
  Hopm* h = static_cast<Hopm*>(plan);
  if (h->p > 1 && !nccl()) return tv::set_error(TV_ECOLL, "tv_dhopm3_sweep: libnccl.so.2 not found");
  for (int j = 0; j < h->d; ++j)
    if (!x[j]) return tv::set_error(TV_EKERNEL, "tv_dhopm3_sweep: null vector");
  return dhopm3_sweep(h, x, norms_out, status_out, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int tv_dhopm3_plan_destroy(void* plan) {
  if (!plan) return TV_OK;
  Hopm* h = static_cast<Hopm*>(plan);
  for (void* b : h->bufs)
    if (b) cudaFree(b);
  if (h->ws) cudaFree(h->ws);
  if (h->counter) cudaFree(h->counter);
  delete h;
  return TV_OK;
}
