/* dHOPM3 from C through libtenvec_b200.so alone -- no Python, no torch.
 *
 * The reference's power method (hopm.py:229-354) on an order-3 fp64 tensor
 * n^3 filled from its global index (tv_fill "hash", bench.py:62-80's role),
 * split along mode 0 over G GPUs of this process: one host thread per GPU,
 * one NCCL communicator per rank from tv_comm_init_all, each rank generating
 * its own slab and running tv_dhopm3_sweep on it.
 *
 *   cc -O2 -I include examples/dhopm3_capi.c -o dhopm3_capi \
 *      -L paper_2501_03121_b200/_lib -ltenvec_b200 -L /usr/local/cuda/lib64 -lcudart -lpthread
 *   ./dhopm3_capi [gpus=1] [n=256] [sweeps=5]
 *
 * Prints the last sweep's norms (lambda estimates) as %.17g: bit-identical to
 * paper_2501_03121_b200.dhopm3 on the same tensor (tests/test_gpu_capi.py).
 */
#include <cuda_runtime.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>

#include "tenvec_b200.h"

typedef struct {
  int rank, p, sweeps;
  int64_t n;
  void* comm;
  double norms[3];
  int rc;
  char err[256];
} Rank;

#define TRY(call)                                                              \
  do {                                                                         \
    int rc_ = (call);                                                          \
    if (rc_ != TV_OK) {                                                        \
      r->rc = rc_;                                                             \
      snprintf(r->err, sizeof r->err, "%s: %s", #call, tv_last_error());       \
      return NULL;                                                             \
    }                                                                          \
  } while (0)

#define CUDA(call)                                                             \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      r->rc = TV_ECUDA;                                                        \
      snprintf(r->err, sizeof r->err, "%s: %s", #call, cudaGetErrorString(e_)); \
      return NULL;                                                             \
    }                                                                          \
  } while (0)

static void* rank_main(void* arg) {
  Rank* r = (Rank*)arg;
  const int64_t n = r->n;
  const int64_t ext[3] = {n, n, n};
  CUDA(cudaSetDevice(r->rank));
  cudaStream_t st;
  CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  TRY(tv_preload(NULL));
  /* this rank's slab along mode 0: ceil(n / p) indices (tensor.py:105-138) */
  const int64_t q = (n + r->p - 1) / r->p;
  const int64_t lo = r->rank * q, hi = lo + q < n ? lo + q : n;
  double* A;
  CUDA(cudaMalloc((void**)&A, (size_t)((hi - lo) * n * n) * sizeof(double)));
  TRY(tv_fill(A, TV_F64, TV_FILL_HASH, 1, ext, 3, 0, lo, hi, st));
  void* plan;
  TRY(tv_dhopm3_plan_create(r->comm, A, TV_F64, TV_F64, 3, ext, 0, &plan));
  /* start vectors: ones, normalised on the device (hopm.py:168-184) */
  void* x[3];
  double* norms;
  int32_t* status;
  CUDA(cudaMalloc((void**)&norms, 3 * sizeof(double)));
  CUDA(cudaMalloc((void**)&status, sizeof(int32_t)));
  CUDA(cudaMemsetAsync(status, 0, sizeof(int32_t), st));
  double* ones = (double*)malloc((size_t)n * sizeof(double));
  for (int64_t i = 0; i < n; ++i) ones[i] = 1.0;
  for (int j = 0; j < 3; ++j) {
    CUDA(cudaMalloc(&x[j], (size_t)n * sizeof(double)));
    CUDA(cudaMemcpyAsync(x[j], ones, (size_t)n * sizeof(double), cudaMemcpyHostToDevice, st));
    TRY(tv_normalize(x[j], TV_F64, TV_F64, n, norms, status, st));
  }
  for (int sw = 0; sw < r->sweeps; ++sw) TRY(tv_dhopm3_sweep(plan, x, norms, status, st));
  int32_t hstat = 0;
  CUDA(cudaMemcpyAsync(r->norms, norms, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CUDA(cudaMemcpyAsync(&hstat, status, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CUDA(cudaStreamSynchronize(st));
  if (hstat != 0) {
    r->rc = TV_ENORM;
    snprintf(r->err, sizeof r->err, "zero vector");
  }
  TRY(tv_dhopm3_plan_destroy(plan));
  for (int j = 0; j < 3; ++j) cudaFree(x[j]);
  cudaFree(A);
  cudaFree(norms);
  cudaFree(status);
  free(ones);
  return NULL;
}

int main(int argc, char** argv) {
  const int p = argc > 1 ? atoi(argv[1]) : 1;
  const int64_t n = argc > 2 ? atoll(argv[2]) : 256;
  const int sweeps = argc > 3 ? atoi(argv[3]) : 5;
  if (p < 1 || p > TV_MAX_RANKS || n < p || sweeps < 1) {
    fprintf(stderr, "usage: %s [gpus] [n] [sweeps]\n", argv[0]);
    return 2;
  }
  void* comms[TV_MAX_RANKS] = {0};
  if (p > 1) {
    int devs[TV_MAX_RANKS];
    for (int i = 0; i < p; ++i) devs[i] = i;
    if (tv_comm_init_all(p, devs, comms) != TV_OK) {
      fprintf(stderr, "tv_comm_init_all: %s\n", tv_last_error());
      return 1;
    }
  }
  Rank ranks[TV_MAX_RANKS];
  pthread_t th[TV_MAX_RANKS];
  for (int i = 0; i < p; ++i) {
    ranks[i] = (Rank){.rank = i, .p = p, .sweeps = sweeps, .n = n, .comm = comms[i], .rc = 0};
    pthread_create(&th[i], NULL, rank_main, &ranks[i]);
  }
  int bad = 0;
  for (int i = 0; i < p; ++i) {
    pthread_join(th[i], NULL);
    if (ranks[i].rc != TV_OK) {
      fprintf(stderr, "rank %d: %s\n", i, ranks[i].err);
      bad = 1;
    }
  }
  for (int i = 0; i < p; ++i) tv_comm_destroy(comms[i]);
  if (bad) return 1;
  for (int i = 1; i < p; ++i)
    for (int j = 0; j < 3; ++j)
      if (ranks[i].norms[j] != ranks[0].norms[j]) {
        fprintf(stderr, "ranks disagree on norm %d\n", j);
        return 1;
      }
  printf("%s gpus=%d n=%lld sweeps=%d\n", tv_version(), p, (long long)n, sweeps);
  printf("norms %.17g %.17g %.17g\n", ranks[0].norms[0], ranks[0].norms[1], ranks[0].norms[2]);
  return 0;
}
