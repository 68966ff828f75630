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
        del bufs, bb, src
    torch.cuda.synchronize()
    print("util kernels ok")
    return 0


if __name__ == "__main__":
    sys.exit(main())
