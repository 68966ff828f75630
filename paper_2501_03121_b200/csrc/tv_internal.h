// Host-side helpers shared by the translation units of libtenvec_b200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tenvec_b200.h"

namespace tv {

// kernel regimes of tv_tvc (reported by tv_tvc_regime)
enum {
  REG_GENERIC = 0,  // the naive kernel (tv_tvc_naive only)
  REG_ROWS = 1,
  REG_ROWS_SHORT = 2,
  REG_COLS = 3,
  REG_SLABS = 4,
  REG_ROWS_U = 5,  // unaligned forms: scalar, lane-interleaved loads
  REG_COLS_U = 6,
  REG_SLABS_U = 7,
  REG_STAGED = 8,  // slabs that fit a tile, staged through shared memory (TMA bulk)
  REG_FLAT = 9,      // narrow aligned slabs streamed as flat warp runs
  REG_FLAT_ROWS = 10,   // short aligned rows streamed as flat warp runs
  REG_STAGED_LONG = 11,  // larger unaligned slabs: row-run tiles by TMA, sums kept across tiles
  REG_FLAT_U = 12,       // tall narrow slabs of any row alignment: flat 16-byte runs, split-K
  REG_STAGED_TALL = 13   // tall narrow unaligned slabs: TMA row tiles, split-K
};

// the five valid (storage, compute) pairs of precision.py:81-87
enum { MODE_INVALID = -1, MODE_F64 = 0, MODE_F32 = 1, MODE_F32F64 = 2, MODE_F16F32 = 3, MODE_BF16F32 = 4 };

inline int mode_id(int storage, int compute) {
  if (storage == TV_F64 && compute == TV_F64) return MODE_F64;
  if (storage == TV_F32 && compute == TV_F32) return MODE_F32;
  if (storage == TV_F32 && compute == TV_F64) return MODE_F32F64;
  if (storage == TV_F16 && compute == TV_F32) return MODE_F16F32;
  if (storage == TV_BF16 && compute == TV_F32) return MODE_BF16F32;
  return MODE_INVALID;
}

inline int dtype_bytes(int dt) {
  switch (dt) {
    case TV_F64: return 8;
    case TV_F32: return 4;
    case TV_F16:
    case TV_BF16: return 2;
    default: return -1;
  }
}

int set_error(int code, const char* msg);
int check_launch(const char* what);
int launched(const char* what);  // check_launch + count one launch
void count_launch();
int regime_of(const void* A, int storage, int64_t u, int64_t nk, int64_t v);
// ws / ws_bytes / ws_given: the split-K workspace (tv_tvc_ws); not given =
// stream-ordered allocation when the view splits
int tvc_dispatch(const void* A, int storage, int compute, int64_t u, int64_t nk, int64_t v,
                 int64_t su, int64_t sk, const void* x, double alpha, double beta, void* y,
                 void* stream, int force_generic, void* ws, int64_t ws_bytes, int ws_given);
// one kernel of each translation unit (tv_preload finds its module)
const void* anchor_tvc();
const void* anchor_util();
int64_t ws_bytes_dispatch(const void* A, int storage, int compute, int64_t u, int64_t nk, int64_t v,
                          int64_t su, int64_t sk);

}  // namespace tv
