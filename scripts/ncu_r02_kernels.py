#!/usr/bin/env python
"""The kernels new in round 2, one representative launch each (for an ncu
--set full capture): ROWS with register-resident x (C5's per-rank slab at
p = 8, k = 2), FLAT_U (tall narrow bf16), tv_repack (undistribute of a 1 GB
tensor split over 4 ranks, both strategies) and the compute-type fold of
undistribute's partial sums."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    import torch

    import paper_2501_03121_b200 as tv

    # ROWS + XR: (4096, 4096, 512) bf16, k = 2
    t = tv.distribute_generated(tv.Shape((4096, 4096, 512)), 0, 1, tv.BF16F32, fill="hash", seed=1).parts[0]
    x = torch.full((512,), 0x3F80, dtype=torch.int16, device="cuda").view(torch.uint16)
    for _ in range(2):
        tv.tvc_native(t, x, 2)
    del t
    # FLAT_U: (8, 1e6, 12) bf16, k = 1
    t = tv.distribute_generated(tv.Shape((8, 1_000_000, 12)), 0, 1, tv.BF16F32, fill="hash", seed=1).parts[0]
    x = torch.full((1_000_000,), 0x3F80, dtype=torch.int16, device="cuda").view(torch.uint16)
    for _ in range(2):
        tv.tvc_native(t, x, 1)
    del t
    # repack: 1 GB fp64 tensor split along mode 1 over 4 ranks (in-process)
    dt = tv.distribute_generated(tv.Shape((64, 2048, 1024)), 1, 4, tv.F64, fill="hash", seed=1)
    for strategy in ("interleave", "gather-copy"):
        tv.undistribute(dt, strategy)
    # wide fold: deferred partial sums of a split-mode contraction, collapsed
    part = tv.dtvc(dt, torch.ones(2048, dtype=torch.float64, device="cuda"), 1, defer=True)
    tv.undistribute(part)
    torch.cuda.synchronize()
    print("ok")
    return 0


if __name__ == "__main__":
    sys.exit(main())
