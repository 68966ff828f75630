#!/usr/bin/env python
"""Run tv_tvc a few times on one view (for ncu targeting).

    python scripts/tvc_one.py --shape 96,96,96,96,24 --mode f32 --k 4 [--reps 3]
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", required=True)
    ap.add_argument("--mode", default="f64")
    ap.add_argument("--k", type=int, required=True)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--naive", action="store_true", help="the tv_tvc_naive cross-check kernel instead")
    args = ap.parse_args()
    import torch

    import paper_2501_03121_b200 as tv

    shape = tuple(int(v) for v in args.shape.split(","))
    mode = tv.MODES[args.mode]
    t = tv.distribute_generated(tv.Shape(shape), 0, 1, mode, fill="hash", seed=1).parts[0]
    n = shape[args.k]
    x = torch.ones(n, dtype=mode.torch_storage, device="cuda") if mode.storage != "brain" else \
        torch.full((n,), 0x3F80, dtype=torch.int16, device="cuda").view(torch.uint16)
    out = torch.empty(t.size // n, dtype=mode.torch_storage, device="cuda")
    for _ in range(args.reps):
        if args.naive:
            tv.tvc_looped_oracle(t, x, args.k)
        else:
            tv.tvc_native(t, x, args.k, out=out)
    torch.cuda.synchronize()
    print(args.shape, args.mode, args.k, tv.tvc_regime(t, args.k))
    return 0


if __name__ == "__main__":
    sys.exit(main())
