"""C1 (256^3 fp64) per-kernel timing probe: event time of each mode alone
(L2 flushed, blocking kernel ahead), an empty-ish launch, and the read probe."""
import sys, os, json
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import paper_2501_03121_b200 as tv
from paper_2501_03121_b200 import _lib
import bench

lib = _lib.load()
shape = tv.Shape((256, 256, 256))
dt = tv.distribute_generated(shape, 0, 1, tv.F64, fill="hash", seed=1)
A = dt.parts[0]
xs = [torch.ones(256, dtype=torch.float64, device="cuda") for _ in range(3)]
flush = bench.L2Flush(torch.device("cuda"))
def timed(fn, reps=20):
    ts = []
    for _ in range(reps):
        flush(); bench._block_stream(torch)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))
out = {}
for k in range(3):
    out[f"k{k}"] = timed(lambda: tv.tvc_native(A, xs[k], k))
sink = torch.zeros(4, dtype=torch.int32, device="cuda")
small = torch.zeros(1 << 12, dtype=torch.uint8, device="cuda")
out["read_4KB"] = timed(lambda: lib.tv_read_stream(small.data_ptr(), 4096, sink.data_ptr(), _lib.stream_ptr()))
out["read_134MB"] = timed(lambda: lib.tv_read_stream(A.buf.data_ptr(), A.buf.numel() * 8, sink.data_ptr(), _lib.stream_ptr()))
ys = [torch.empty(65536, dtype=torch.float64, device="cuda") for _ in range(3)]
from paper_2501_03121_b200.kernels import launch_sweep
out["sweep3"] = timed(lambda: launch_sweep(A, xs, ys))
out["3 separate"] = timed(lambda: [tv.tvc_native(A, xs[k], k) for k in range(3)])
print(json.dumps({k: round(v, 2) for k, v in out.items()}))
