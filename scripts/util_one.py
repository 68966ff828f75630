#!/usr/bin/env python
"""Run the non-TVC kernels once each on representative sizes (for ncu):
the in-process rank fold (exact and mixed), normalize, convert, fill.

    python scripts/util_one.py
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    import torch

    import paper_2501_03121_b200 as tv

    n = 1 << 26  # 64 Mi elements per rank buffer
    for _ in range(2):
        # exact fold of 8 fp32 rank buffers (ring_all_reduce, comm.py:84-100)
        bufs = [torch.full((n,), float(r), dtype=torch.float32, device="cuda") for r in range(8)]
        tv.ring_all_reduce(bufs)
        # mixed fold of 8 bf16 buffers (ring_all_reduce_mixed, comm.py:103-134)
        bb = [torch.full((n,), 0x3F80, dtype=torch.int16, device="cuda").view(torch.uint16) for _ in range(8)]
        tv.ring_all_reduce_mixed(bb, tv.BF16F32)
        # promote / demote over 256 Mi fp64 elements
        src = torch.ones(4 * n, dtype=torch.float64, device="cuda")
        tv.demote(src, tv.BF16F32)
        # normalize a 4096-vector (dHOPM3 epilogue)
        v = torch.ones(4096, dtype=torch.float64, device="cuda")
        tv.normalize(v)
        # device fill of a 2 GB slab
        tv.distribute_generated(tv.Shape((1024, 1024, 256)), 0, 1, tv.F64, fill="hash")
        # fused last contraction + normalize of a dHOPM3 iteration (2000 x 2000 fp64)
        w = tv.Tensor(tv.Shape((2000, 2000)), torch.ones(4_000_000, dtype=torch.float64, device="cuda"), tv.F64)
        slot = torch.empty(1, dtype=torch.float64, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
        tv.tvc_normalize_async(w, torch.ones(2000, dtype=torch.float64, device="cuda"), 1,
                               torch.empty(2000, dtype=torch.float64, device="cuda"), slot, None, cnt)
        # axpby over 64 Mi fp32 (kernels.py:191-231)
        xa = torch.ones(n, dtype=torch.float32, device="cuda")
        ya = torch.ones(n, dtype=torch.float32, device="cuda")
        tv.axpby(2.0, xa, 0.5, ya, mode=tv.F32)
        # select-gather of 8 ranges (the peer-memory allreduce's gather phase)
        import ctypes
        from paper_2501_03121_b200 import _lib
        srcs = [torch.full((n,), float(r), dtype=torch.float32, device="cuda") for r in range(8)]
        arr = (ctypes.c_void_p * 8)(*[b.data_ptr() for b in srcs])
        dst = torch.empty(n, dtype=torch.float32, device="cuda")
        _lib.check(_lib.load().tv_rank_select(arr, 8, n, n // 8, _lib.TV_F32, dst.data_ptr(), _lib.stream_ptr()))
        # read-only roofline probe over 2 GB
        sink = torch.zeros(4, dtype=torch.int32, device="cuda")
        big = torch.ones(1 << 31, dtype=torch.uint8, device="cuda")
        _lib.check(_lib.load().tv_read_stream(big.data_ptr(), big.numel(), sink.data_ptr(), _lib.stream_ptr()))
        del bufs, bb, src, w, xa, ya, srcs, dst, big
    torch.cuda.synchronize()
    print("util kernels ok")
    return 0


if __name__ == "__main__":
    sys.exit(main())
