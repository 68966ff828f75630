#!/usr/bin/env python
"""dHOPM3 sweeps per second on small tensors, eager vs graph=True (one GPU)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    import torch

    import paper_2501_03121_b200 as tv

    for shape, name in (((64, 64, 64), "f64"), ((32, 32, 32, 32), "f64"), ((256, 256, 256), "f64"),
                        ((128, 128, 128, 16), "bf16f32")):
        mode = tv.MODES[name]
        dt = tv.distribute_generated(tv.Shape(shape), 0, 1, mode, fill="hash", seed=1)
        x0 = tv.initial_vectors(tv.Shape(shape), mode)
        row = {"shape": list(shape), "mode": name}
        for g in (False, True):
            tv.dhopm3(dt, [v.copy() for v in x0], sweeps=4, graph=g)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sweeps = 50
            tv.dhopm3(dt, [v.copy() for v in x0], sweeps=sweeps, graph=g)
            torch.cuda.synchronize()
            row["graph" if g else "eager"] = round((time.perf_counter() - t0) / sweeps * 1e3, 4)
        row["unit"] = "ms per sweep (wall, 50 sweeps incl. capture)"
        print(json.dumps(row), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
