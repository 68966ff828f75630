#!/usr/bin/env python
"""One tv_tvc call on a generated view, for ncu captures:
    python scripts/one_view.py 8,1000000,12 1 bf16f32 [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    import torch

    import paper_2501_03121_b200 as tv

    shape = tuple(int(s) for s in sys.argv[1].split(","))
    k, mname = int(sys.argv[2]), sys.argv[3]
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    mode = tv.MODES[mname]
    t = tv.distribute_generated(tv.Shape(shape), 0, 1, mode, fill="hash", seed=1).parts[0]
    n = shape[k]
    x = torch.ones(n, dtype=mode.torch_storage, device="cuda") if mode.storage != "brain" else \
        torch.full((n,), 0x3F80, dtype=torch.int16, device="cuda").view(torch.uint16)
    out = torch.empty(t.size // n, dtype=mode.torch_storage, device="cuda")
    for _ in range(reps):
        tv.tvc_native(t, x, k, out=out)
    torch.cuda.synchronize()
    print(tv.tvc_regime(t, k))
    return 0


if __name__ == "__main__":
    sys.exit(main())
