#!/usr/bin/env python
"""Mode-obliviousness sweep: event-timed GB/s of tv_tvc for every mode of a
set of tensors (the paper's Table-1 hypersquares at ~7.5 GB fp64, the
BASELINE configs and their per-rank slabs).  One JSON line per (tensor, k).

    python scripts/tvc_modes_bench.py [--set table1|baseline|all] [--reps 5]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TABLE1 = {2: 30623, 3: 979, 4: 175, 5: 63, 6: 31, 7: 19, 8: 13, 9: 10, 10: 8}

BASELINE = [
    ("C1 256^3", (256,) * 3, "f64"),
    ("C2 2048^3", (2048,) * 3, "f64"),
    ("C3 96^5", (96,) * 5, "f32"),
    ("C3 p=2 slab s=4", (96, 96, 96, 96, 48), "f32"),
    ("C3 p=4 slab s=4", (96, 96, 96, 96, 24), "f32"),
    ("C3 p=8 slab s=4", (96, 96, 96, 96, 12), "f32"),
    ("C3 p=8 slab s=0", (12, 96, 96, 96, 96), "f32"),
    ("C4 p=8 slab s=3", (384, 384, 384, 48), "f64"),
    ("C5 p=8 slab s=2", (4096, 4096, 512), "bf16f32"),
]


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--set", default="all", choices=["table1", "baseline", "all"])
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch

    import paper_2501_03121_b200 as tv

    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
    cases = []
    if args.set in ("table1", "all"):
        cases += [(f"paper d={d}", (n,) * d, "f64") for d, n in TABLE1.items()]
    if args.set in ("baseline", "all"):
        cases += BASELINE
    for name, shape, mname in cases:
        mode = tv.MODES[mname]
        dt = tv.distribute_generated(tv.Shape(shape), 0, 1, mode, fill="hash", seed=1)
        t = dt.parts[0]
        for k in range(len(shape)):
            x = torch.ones(shape[k], dtype=mode.torch_storage, device="cuda") if mode.storage != "brain" \
                else torch.full((shape[k],), 0x3F80, dtype=torch.int16, device="cuda").view(torch.uint16)
            out = torch.empty(t.size // shape[k], dtype=mode.torch_storage, device="cuda")
            for _ in range(2):
                tv.tvc_native(t, x, k, out=out)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                tv.tvc_native(t, x, k, out=out)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.reps
            nbytes = (t.size + shape[k] + t.size // shape[k]) * mode.storage_bytes
            gbs = nbytes / (ms / 1e3) / 1e9
            md = tv.matricize_dims(t.shape, k)
            print(json.dumps({"tensor": name, "shape": list(shape), "mode": mname, "k": k,
                              "uvw": [md.u, md.nk, md.v], "regime": tv.tvc_regime(t, k),
                              "ms": round(ms, 4), "gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}),
                  flush=True)
        del dt, t
        torch.cuda.empty_cache()
    return 0


if __name__ == "__main__":
    sys.exit(main())
