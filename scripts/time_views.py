#!/usr/bin/env python
"""Event-timed GB/s of tv_tvc on generated views (cold: each call reads more
than L2).  Usage: python scripts/time_views.py f64:30623,30623:0 f64:15311,61246:0 ..."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    import torch

    import paper_2501_03121_b200 as tv

    for spec in sys.argv[1:]:
        mname, dims, k = spec.split(":")
        shape, k = tuple(int(s) for s in dims.split(",")), int(k)
        mode = tv.MODES[mname]
        t = tv.distribute_generated(tv.Shape(shape), 0, 1, mode, fill="hash", seed=1).parts[0]
        n = shape[k]
        x = torch.ones(n, dtype=mode.torch_storage, device="cuda") if mode.storage != "brain" else \
            torch.full((n,), 0x3F80, dtype=torch.int16, device="cuda").view(torch.uint16)
        out = torch.empty(t.size // n, dtype=mode.torch_storage, device="cuda")
        for _ in range(2):
            tv.tvc_native(t, x, k, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            tv.tvc_native(t, x, k, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        nbytes = (t.size + n + t.size // n) * mode.storage_bytes
        print(json.dumps({"shape": list(shape), "k": k, "mode": mname, "regime": tv.tvc_regime(t, k),
                          "ms": round(ms, 4), "gbs": round(nbytes / ms / 1e6, 1)}), flush=True)
        del t, out
        torch.cuda.empty_cache()
    return 0


if __name__ == "__main__":
    sys.exit(main())
