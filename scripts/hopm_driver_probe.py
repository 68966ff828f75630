#!/usr/bin/env python
"""dHOPM3 ms per sweep on one GPU: the Python driver (eager), its graph
replay, and the C++ plan (tv_dhopm3_sweep) -- host overhead on small tensors."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]


def main() -> int:
    import numpy as np
    import torch

    import paper_2501_03121_b200 as tv
    from capi_checks import c_dhopm3

    for shape in [(32, 32, 32, 32), (64, 64, 64), (96, 96, 96, 96), (256, 256, 256)]:
        dt = tv.distribute_generated(tv.Shape(shape), 0, 1, tv.F64, fill="hash", seed=1)
        x0 = tv.initial_vectors(tv.Shape(shape), tv.F64)
        sweeps = 50
        out = {"shape": shape}
        for name, fn in (("eager", lambda: tv.dhopm3(dt, x0, sweeps=sweeps)),
                         ("graph", lambda: tv.dhopm3(dt, x0, sweeps=sweeps, graph=True)),
                         ("capi", lambda: c_dhopm3(tv, None, dt.parts[0], shape, 0, tv.F64, x0, sweeps))):
            fn()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            out[name + "_ms_per_sweep"] = round((time.perf_counter() - t0) * 1e3 / sweeps, 4)
        print(json.dumps(out), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
