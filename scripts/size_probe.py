#!/usr/bin/env python
"""Read-only HBM rate vs buffer size, cold L2 (flush before each launch, a
blocking kernel ahead of the start event): the floor that small views such as
C1 (134 MB) can reach.  Prints one JSON line per size."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    import torch

    import bench
    from paper_2501_03121_b200 import _lib

    lib = _lib.load()
    flush = bench.L2Flush(torch.device("cuda"))
    sink = torch.zeros(4, dtype=torch.int32, device="cuda")
    big = torch.ones(1 << 31, dtype=torch.uint8, device="cuda")
    for mb in (16, 32, 64, 134, 256, 512, 1024, 2048):
        nb = (mb << 20) & ~15
        ts = []
        for _ in range(10):
            flush()
            bench._block_stream(torch)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.check(lib.tv_read_stream(big.data_ptr(), nb, sink.data_ptr(), _lib.stream_ptr()))
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        med = ts[len(ts) // 2]
        print(json.dumps({"mb": mb, "us": round(med * 1e3, 2), "gbs": round(nb / (med / 1e3) / 1e9, 1)}),
              flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
