#!/usr/bin/env python
"""GB/s of tall-skinny contractions (u small, n_k large, v small): the shapes
whose natural grids are a handful of warps."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    import torch

    import paper_2501_03121_b200 as tv

    cases = [((4_000_000, 8), 0, "f64"), ((1_000_000, 4, 4), 0, "f64"), ((1, 8_000_000, 16), 1, "f32"),
             ((1_000_000, 100), 0, "f64"), ((2, 2_000_000, 24), 1, "f32"), ((3_000_001, 7), 0, "f64"),
             ((400_000, 64), 0, "f64"), ((200_000, 300), 0, "f64"), ((30623, 30623), 0, "f64"),
             ((8, 1_000_000, 12), 1, "bf16f32"), ((8, 1_000_000, 12), 1, "f16f32"),
             ((3_000_001, 7), 0, "bf16f32"), ((2, 2_000_000, 6), 1, "bf16f32"), ((1_000_003, 20), 0, "f16f32")]
    for shape, k, mname in cases:
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
        torch.cuda._sleep(2_000_000)
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
    return 0


if __name__ == "__main__":
    sys.exit(main())
