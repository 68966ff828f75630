/*
 * tenvec_b200.h -- C-ABI of libtenvec_b200.so, the B200 (sm_100a) hot path of
 * arXiv 2501.03121 (native TVC, dTVC reductions, dHOPM3 normalisation).
 *
 * Every entry point takes plain device pointers owned by the caller, element
 * counts, and a cudaStream_t passed as void*.  All work is enqueued
 * asynchronously on that stream; nothing synchronises the host.  Device
 * memory: the only allocation is the split-K workspace of tv_tvc / tv_getvc
 * on views with few, long outputs (stream-ordered cudaMallocAsync, freed on
 * the same stream; failure returns TV_ECUDA, never a different kernel).
 * tv_tvc_ws / tv_getvc_ws take that workspace from the caller instead (size
 * from tv_tvc_workspace_bytes / tv_getvc_workspace_bytes) and allocate
 * nothing -- the Python package always uses them.  Return value: TV_OK (0)
 * or an error code; the thread-local tv_last_error() gives the message.
 * There is no CPU fallback: a missing or failing device raises TV_ECUDA.
 *
 * Reference interfaces replaced (paths relative to the reference pkg/src/tenvec):
 *   tv_tvc_sweep    bench.py:209-215    the per-mode tvc loop of a dTVC mode sweep
 *   tv_tvc, tv_tvc_ws kernels.py:126-171 tvc_native (and getvc, kernels.py:73-123,
 *                                       through the (u, n_k, v) block view)
 *   tv_getvc(_ws)   kernels.py:73-123   getvc over a strided m x n view (lda >= n)
 *   tv_convert      precision.py:109-128 promote / demote (bit-exact semantics)
 *   tv_norm2        kernels.py:234-239  norm2
 *   tv_normalize    kernels.py:242-254  normalize
 *   tv_tvc_normalize hopm.py:295-333   the last tvc_native of a power-method iteration
 *                                       + normalize, fused (normalisation in the epilogue)
 *   tv_rank_fold    comm.py:84-100      ring_all_reduce (ascending-rank fold) and
 *                   comm.py:103-134     ring_all_reduce_mixed (chunk c starts at rank c,
 *                                       demote(promote+promote) per hop)
 *   tv_peer_barrier comm.py:202-235     the WorkerGroup rendezvous slot + timeout, as a
 *                                       stream-ordered barrier over peer memory
 *   tv_comm_*       comm.py:168-284    WorkerGroup's ranks, as NCCL communicators
 *   tv_allreduce    comm.py:84-134      ring_all_reduce / ring_all_reduce_mixed across processes
 *   tv_allgather    comm.py:137-153     all_gather
 *   tv_dhopm3_*     hopm.py:229-354     dhopm3 (one sweep per call)
 *   tv_repack       tensor.py:233-272   reassemble (interleave / gather-copy copy pass)
 *   tv_fill         bench.py:62-80      fill_array (ones / ramp; "hash" replaces numpy's
 *                                       integer-random with a counter hash in [1, 97])
 */
#ifndef TENVEC_B200_H
#define TENVEC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* storage / compute element types (precision.py:69-87) */
typedef enum {
  TV_F64 = 0,  /* double                                   */
  TV_F32 = 1,  /* single                                   */
  TV_F16 = 2,  /* IEEE binary16 ("half")                   */
  TV_BF16 = 3  /* brain float, uint16 bit pattern ("brain") */
} tv_dtype;

/* error codes; Python maps 1->KernelError, 2->ModeError, 3->NormalizationError,
 * 4->CollectiveError, 5->CUDA runtime error */
enum {
  TV_OK = 0,
  TV_EKERNEL = 1,
  TV_EMODE = 2,
  TV_ENORM = 3,
  TV_ECOLL = 4,
  TV_ECUDA = 5
};

/* fill kinds for tv_fill */
enum { TV_FILL_ONES = 0, TV_FILL_RAMP = 1, TV_FILL_HASH = 2 };

/* maximum rank count of tv_rank_fold */
#define TV_MAX_RANKS 64

/* Library version string and the kernel regime names (diagnostics). */
const char* tv_version(void);

/* Kernels this library has launched in this process so far (every launch
 * site counts itself; a bench reads it around its timed region). */
unsigned long long tv_launch_count(void);
const char* tv_last_error(void);

/* Y = alpha * (A x_k x) + beta * Y over the rank-local block view
 * A[u][nk][v] (last index fastest, no unfolding copy).  Valid (storage,
 * compute) pairs: (F64,F64) (F32,F32) (F32,F64) (F16,F32) (BF16,F32).
 * beta == 0 never reads y.  y holds u*v storage elements.  Accumulation in
 * the compute type, one demote on store; alpha multiplies the finished dot
 * product and beta*y is added after it (kernels.py:113-119).  The reduction
 * order per output element is fixed by (u, nk, v, dtype): reruns and ranks
 * reproduce bits. */
int tv_tvc(const void* A, int storage, int compute, int64_t u, int64_t nk, int64_t v,
           const void* x, double alpha, double beta, void* y, void* stream);

/* Bytes of split-K workspace tv_tvc needs for this view (0 when the view
 * does not split; -1 on invalid arguments).  A pure function of (A's
 * alignment, storage, compute, u, nk, v) and the device's SM count: a view
 * always splits the same way, so its summation order never depends on
 * memory availability. */
int64_t tv_tvc_workspace_bytes(const void* A, int storage, int compute, int64_t u, int64_t nk, int64_t v);

/* tv_tvc with a caller-provided split-K workspace (16-byte aligned, at least
 * tv_tvc_workspace_bytes; may be NULL when that is 0).  Allocates nothing:
 * safe inside CUDA graph capture; TV_EKERNEL if the workspace is short. */
int tv_tvc_ws(const void* A, int storage, int compute, int64_t u, int64_t nk, int64_t v,
              const void* x, double alpha, double beta, void* y, void* ws, int64_t ws_bytes,
              void* stream);

/* The mode sweep (the unit of the paper's dTVC benchmarks, bench.py:209-215):
 * ys[k] <- A x_k xs[k] for every mode k = 0..d-1 of the contiguous order-d
 * tensor A (extents ext[0..d-1], last fastest), alpha = 1, beta = 0 -- each
 * output bit-identical to tv_tvc_ws on that mode's (u, n_k, v) view.  Modes
 * after the first launch with programmatic stream serialization: outputs
 * must be distinct and must not alias A.  ws: at least
 * tv_tvc_sweep_workspace_bytes (NULL when that is 0); allocates nothing. */
int tv_tvc_sweep(const void* A, int storage, int compute, int d, const int64_t* ext, const void* const* xs,
                 void* const* ys, void* ws, int64_t ws_bytes, void* stream);
int64_t tv_tvc_sweep_workspace_bytes(const void* A, int storage, int compute, int d, const int64_t* ext);

/* The same contraction through the naive scalar kernel only (one thread per
 * output for v > 1, one warp per row for v == 1): the "looped" cross-check of
 * tv_tvc's regime kernels, used by tvc_looped_oracle (kernels.py:174-188). */
int tv_tvc_naive(const void* A, int storage, int compute, int64_t u, int64_t nk, int64_t v,
                 const void* x, double alpha, double beta, void* y, void* stream);

/* The last contraction of a power-method iteration with the vector
 * normalisation folded into the kernel epilogue (north star; hopm.py:295-333:
 * tvc_native of the carried 2-mode tensor, then normalize kernels.py:242-254):
 * y = A x over the contiguous (u, nk, v) view with alpha = 1, beta = 0, then,
 * in the same launch (the last CTA to finish), y <- demote(promote(y)/||y||)
 * with tv_normalize's reduction tree; *norm_out (device double) gets the
 * norm, *status_out (device int32, may be NULL) TV_ENORM on a zero vector
 * (y then left unscaled).  counter: a device uint32 that is 0 on entry and is
 * left 0; one per concurrently running call.  For small final products:
 * u * v <= 2^22 and u * nk * v <= 2^28, else TV_EKERNEL. */
int tv_tvc_normalize(const void* A, int storage, int compute, int64_t u, int64_t nk, int64_t v,
                     const void* x, void* y, double* norm_out, int32_t* status_out,
                     unsigned* counter, void* stream);

/* Which kernel regime tv_tvc would pick for this view: 1 rows, 2 short rows,
 * 3 columns, 4 narrow slabs, and their unaligned (scalar-load) forms 5 rows,
 * 6 columns, 7 slabs, 8 slabs staged through shared memory by TMA bulk
 * copies, 9 flat narrow slabs, 10 flat short rows, 11 larger unaligned slabs
 * as TMA row-run tiles, 12 tall narrow slabs of any row alignment as flat
 * 16-byte runs (0 is the naive kernel,
 * tv_tvc_naive only); -1 on invalid arguments. */
int tv_tvc_regime(const void* A, int storage, int64_t u, int64_t nk, int64_t v);

/* Diagnostic: pin the regime tv_tvc uses wherever the view can take it
 * (regime codes as tv_tvc_regime; <= 0 restores the heuristics).  Returns the
 * previous override (-1 = none).  Initialised from TENVEC_B200_FORCE.  Not in
 * the reference; used by the regime coverage tests and kernel A/B runs. */
int tv_set_regime_override(int regime);

/* getvc over an m x n row-major view with leading dimension lda >= n.
 * trans 0 = matvec (x has n, y has m), 1 = vecmat (x has m, y has n). */
int tv_getvc(int trans, const void* A, int storage, int compute, int64_t m, int64_t n,
             int64_t lda, const void* x, double alpha, double beta, void* y, void* stream);

/* Split-K workspace of tv_getvc for this view, and tv_getvc with it supplied
 * by the caller (as tv_tvc_workspace_bytes / tv_tvc_ws). */
int64_t tv_getvc_workspace_bytes(int trans, const void* A, int storage, int compute, int64_t m, int64_t n,
                                 int64_t lda);
int tv_getvc_ws(int trans, const void* A, int storage, int compute, int64_t m, int64_t n, int64_t lda,
                const void* x, double alpha, double beta, void* y, void* ws, int64_t ws_bytes,
                void* stream);

/* dst[i] = convert(src[i]) with reference semantics: widening is exact,
 * f64->f32 and ->f16 round to nearest even (f16 overflow -> inf), ->bf16
 * rounds to f32 first and truncates the low 16 bits. */
int tv_convert(const void* src, int src_dtype, void* dst, int dst_dtype, int64_t n,
               void* stream);

/* *norm_out (device double) = sqrt(sum promote(x)^2) accumulated in the
 * compute type with a fixed reduction tree (single CTA). */
int tv_norm2(const void* x, int storage, int compute, int64_t n, double* norm_out,
             void* stream);

/* x <- demote(promote(x) / ||x||) in place; *norm_out (device double) gets
 * the norm it had.  A zero norm leaves x untouched and sets *status_out
 * (device int32) to TV_ENORM; status_out may be NULL. */
int tv_normalize(void* x, int storage, int compute, int64_t n, double* norm_out,
                 int32_t* status_out, void* stream);

/* Rank-ordered fold of p device buffers (srcs is a HOST array of p device
 * pointers, p <= TV_MAX_RANKS) into dst (may alias srcs[0]).
 *   mixed == 0: dst[e] = ((s0[e] + s1[e]) + s2[e]) + ...  in the storage type
 *               (exact-width ring_all_reduce, bit-equal to serial_rank_sum)
 *   mixed == 2: dst[e] = demote(((promote(s0[e]) + promote(s1[e])) + ...) in
 *               the compute type (undistribute's partial-sum collapse,
 *               hopm.py:76-84; chunk and start ignored)
 *   mixed == 1: with c = chunk ? e / chunk : 0 and r0 = (start + c) % p,
 *               cur = s_r0[e]; for i in 1..p-1: cur = demote(promote(cur) +
 *               promote(s_{(r0+i)%p}[e]))  (ring_all_reduce_mixed)
 * chunk is ring_chunks' ceil(n/p) for an in-process fold over whole
 * buffers, or 0 with start = c when the buffers hold only chunk c. */
int tv_rank_fold(const void* const* srcs, int p, int64_t n, int64_t chunk, int start,
                 int storage, int compute, int mixed, void* dst, void* stream);

/* Same fold, sources at src + r * src_stride_elems (one contiguous receive
 * buffer after an all-to-all). */
int tv_rank_fold_strided(const void* src, int64_t src_stride_elems, int p, int64_t n,
                         int64_t chunk, int start, int storage, int compute, int mixed,
                         void* dst, void* stream);

/* The reduction of a dHOPM3 iteration's vector with the normalisation in
 * the kernel epilogue (hopm.py:320-330: allreduce, then normalize on every
 * rank): dst = tv_rank_fold_strided(src, stride, p, n, chunk, start = 0)
 * and, in the same launch (the last CTA to finish), dst <- dst / ||dst||
 * with tv_normalize's tree; *norm_out / *status_out as tv_normalize.
 * counter: a device uint32, 0 on entry, left 0. */
int tv_rank_fold_normalize(const void* src, int64_t src_stride_elems, int p, int64_t n,
                           int64_t chunk, int storage, int compute, int mixed, void* dst,
                           double* norm_out, int32_t* status_out, unsigned* counter, void* stream);

/* tv_rank_fold_strided over a RANGE [offset, offset + n) of a ring buffer
 * whose ring chunks have ring_chunk elements (chunk c starts at rank c, the
 * mixed ring of comm.py:103-134; ignored for the exact fold): the owner of a
 * range folds the p partial copies of it that peers wrote into its receive
 * slots (src + r * src_stride_elems), in the reference's per-element order. */
int tv_rank_fold_range(const void* src, int64_t src_stride_elems, int p, int64_t n,
                       int64_t ring_chunk, int64_t offset, int storage, int compute, int mixed,
                       void* dst, void* stream);

/* dst[e] = srcs[e / chunk][e] (srcs a HOST array of p device pointers, e.g.
 * peer buffers of a symmetric-memory group): the gather phase of the
 * peer-memory allreduce, where rank r's buffer holds reduced ring chunk r. */
int tv_rank_select(const void* const* srcs, int p, int64_t n, int64_t chunk, int dtype,
                   void* dst, void* stream);

/* reassemble (tensor.py:233-272): the joint tensor, viewed as (u, ns, v)
 * around the split mode, from p parts split along it -- part r (a HOST
 * array of p device pointers; peer pointers work) is (u, ext_r, v) with
 * ext_r = min(q, ns - r q).  Both assembly strategies end in this one copy
 * pass: "interleave" passes the parts where they lie, "gather-copy" the
 * parts' offsets in one gathered buffer.  Bytes are moved as they are
 * (elem_bytes = 1, 2, 4 or 8), each contiguous run in the widest aligned
 * unit. */
int tv_repack(const void* const* srcs, int p, int64_t u, int64_t ns, int64_t v, int64_t q, int elem_bytes,
              void* dst, void* stream);

/* One part's share of tv_repack: part r's runs from src into the joint
 * tensor at dst (which may be a peer's buffer: the interleave assembly
 * across GPUs pushes every rank's part into every rank's joint copy). */
int tv_repack_part(const void* src, int r, int p, int64_t u, int64_t ns, int64_t v, int64_t q, int elem_bytes,
                   void* dst, void* stream);

/* tv_repack_part into EVERY rank's joint copy at once: dst_mc is the
 * NVSwitch multicast address of the ranks' joint buffers (the same offset in
 * each); each 16-byte unit is stored once (multimem.st) and replicated by
 * the switch.  Needs 16-byte aligned buffers and runs (TV_EKERNEL else). */
int tv_repack_part_multicast(const void* src, int r, int p, int64_t u, int64_t ns, int64_t v, int64_t q,
                             int elem_bytes, void* dst_mc, void* stream);

/* tv_repack_part into ndst joint copies in ONE launch (this rank's and the
 * peers', dsts = a HOST array of device pointers as mapped here): each
 * 16-byte unit is read once and stored to every destination.  Needs 16-byte
 * aligned buffers and runs (TV_EKERNEL else). */
int tv_repack_part_peers(const void* src, int r, int p, int64_t u, int64_t ns, int64_t v, int64_t q,
                         int elem_bytes, void* const* dsts, int ndst, void* stream);

/* Bytes at the start of a peer buffer reserved for the barrier words
 * (uint32 per rank); the transports put their data after it. */
#define TV_PEER_HEADER 4096

/* Stream-ordered barrier of p ranks over peer memory (the device form of the
 * WorkerGroup rendezvous, comm.py:202-235).  peer_bases is a HOST array of
 * the p ranks' peer-buffer bases as mapped in this process (zeroed headers
 * before the first barrier); epoch counts this group's barriers from 1 and
 * must be the same on every rank.  One single-CTA kernel: posts epoch into
 * word [rank] of every peer's header (release, system scope), then waits for
 * word [j] of its own header to reach epoch for every j (acquire).  Past
 * timeout_ns (<= 0: wait forever) it does NOT trap: it writes status[0] =
 * TV_ECOLL, status[1] = epoch, status[2..3] = bit mask of the ranks still
 * missing (device int32[4], zero on entry) and returns; while status[0] is
 * set, later barriers post their arrival without waiting. */
int tv_peer_barrier(void* const* peer_bases, int p, int rank, uint32_t epoch, int64_t timeout_ns,
                    int32_t* status, void* stream);

/* Load every kernel of the library into the current device's context now
 * (CUDA 12 loads kernels lazily, at first launch, and a load may wait for the
 * kernels already running -- including a tv_peer_barrier that waits for this
 * rank: call it before the first barrier).  *loaded (may be NULL) receives
 * the number of kernels loaded. */
int tv_preload(int* loaded);

/* ---- the distributed layer (hopm.py / comm.py without Python) ----------
 * One NCCL communicator per rank, taken from the process's libnccl.so.2 at
 * run time.  Either one process per GPU -- rank 0 calls
 * tv_comm_get_unique_id, ships the 128 bytes to every rank, each calls
 * tv_comm_init_rank with its device current -- or one process for several
 * GPUs (tv_comm_init_all, then one host thread per rank).  Collectives are
 * enqueued on the given stream; every rank must issue the same sequence. */
#define TV_UNIQUE_ID_BYTES 128
int tv_comm_get_unique_id(void* id_out);
int tv_comm_init_rank(const void* id, int nranks, int rank, void** comm_out);
int tv_comm_init_all(int ndev, const int* devs, void** comms_out);
int tv_comm_rank_size(void* comm, int* rank, int* size);
int tv_comm_destroy(void* comm);

/* In-place allreduce of n storage elements (comm.py:84-134):
 *   TV_AR_EXACT  ascending-rank fold in the storage type (ring_all_reduce)
 *   TV_AR_MIXED  the mixed ring: chunk c starts at rank c, every hop
 *                demote(promote + promote) (ring_all_reduce_mixed)
 *   TV_AR_NCCL   ncclAllReduce (f64/f32 only; rank-consistent, not
 *                reference-ordered)
 * EXACT and MIXED give the reference's bits on every rank: NCCL moves the
 * bytes (small buffers: one all-gather; larger: ring-chunk all-to-all, the
 * fold of this rank's chunk, all-gather) and tv_rank_fold adds them.  ws:
 * tv_allreduce_workspace_bytes (allocates nothing). */
#define TV_AR_NCCL 0
#define TV_AR_EXACT 1
#define TV_AR_MIXED 2
int64_t tv_allreduce_workspace_bytes(void* comm, int64_t n, int storage, int algo);
int tv_allreduce(void* comm, void* buf, int64_t n, int storage, int compute, int algo, void* ws,
                 int64_t ws_bytes, void* stream);

/* Rank-order concatenation of counts[r] elements of elem_bytes from every
 * rank into out (comm.py:137-153 all_gather; parts may differ in length). */
int tv_allgather(void* comm, const void* local, void* out, const int64_t* counts, int elem_bytes,
                 void* stream);

/* dHOPM3 (hopm.py:229-354, the reuse schedule of costmodel.py:138-153) on
 * this rank's slab A of the order-d global tensor ext split along mode s
 * over the communicator's ranks (comm NULL: one rank, A the whole tensor).
 * The plan holds the schedule, three rotating product buffers and the
 * workspaces (allocated here, once).  tv_dhopm3_sweep runs one sweep:
 * x[0..d-1] (device, full-length vectors in storage format, identical on
 * every rank) are updated in place, norms_out[j] (device double) gets the
 * norm of iteration j, status_out (device int32, may be NULL) TV_ENORM on a
 * zero vector.  Bit-identical to the Python dhopm3 with a RankGroup.  A
 * must outlive the plan; call with the communicator's device current. */
int tv_dhopm3_plan_create(void* comm, const void* A, int storage, int compute, int d, const int64_t* ext,
                          int s, void** plan_out);
int tv_dhopm3_plan_slab(void* plan, int64_t* lo, int64_t* hi);
int tv_dhopm3_sweep(void* plan, void* const* x, double* norms_out, int32_t* status_out, void* stream);
int tv_dhopm3_plan_destroy(void* plan);

/* Fill the rank-local slab [s_lo, s_hi) along mode s of a global tensor with
 * extents ext[0..d-1] (last mode fastest) from the GLOBAL linear index g:
 * ones -> 1, ramp -> (g mod 97) + 1, hash -> (splitmix64(seed, g) mod 97) + 1. */
int tv_fill(void* A, int dtype, int kind, uint64_t seed, const int64_t* ext, int d, int s,
            int64_t s_lo, int64_t s_hi, void* stream);

/* y <- demote(alpha * promote(x) + beta * promote(y)) elementwise over n
 * storage elements (kernels.py:191-231 axpby): each product and the sum are
 * rounded separately in the compute type; beta == 0 never reads y. */
int tv_axpby(double alpha, const void* x, double beta, void* y, int storage, int compute,
             int64_t n, void* stream);

/* Read-only streaming probe over `bytes` (16-byte aligned) of device memory:
 * the HBM read roofline the TVC kernels are measured against in bench.py.
 * `sink` is a device uint32 that is written only in a practically impossible
 * case (keeps the loads from being optimised away). */
int tv_read_stream(const void* buf, int64_t bytes, void* sink, void* stream);

/* Number of SMs of the current device (grid sizing diagnostics). */
int tv_device_sms(void);

#ifdef __cplusplus
}
#endif

#endif /* TENVEC_B200_H */
