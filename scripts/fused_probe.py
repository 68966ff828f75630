#!/usr/bin/env python
"""Phase times of the fused split-mode reduction (C2 k = 0 at N GPUs):
local TVC, owner-scatter TVCs, barrier, owner fold, gather.  Max over ranks.
torchrun --nproc-per-node N scripts/fused_probe.py"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    import torch
    import torch.distributed as dist

    import paper_2501_03121_b200 as tv
    from paper_2501_03121_b200 import _lib
    from paper_2501_03121_b200.comm import ring_chunks

    rank, p = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    g = tv.RankGroup(algo="fused")
    dt = tv.distribute_generated(tv.Shape((2048, 2048, 2048)), 0, p, tv.F64, fill="hash", seed=1, group=g)
    part = dt.parts[rank]
    a, b = dt.plan.ranges[rank]
    xv = torch.ones(b - a, dtype=torch.float64, device="cuda")
    nk, v = part.shape.extents[0], 2048 * 2048
    n = v
    q = -(-v // p)
    chunk = q
    sb = 8
    slot_bytes = -(-chunk * sb // 16) * 16
    sym, hdl = g._symmetric((p + 1) * slot_bytes, part.buf.device)
    ptrs = [int(x) for x in hdl.buffer_ptrs]
    lib = _lib.load()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    ring = ring_chunks(n, p)

    def local():
        tv.tvc_native(part, xv, 0, out=out)

    def scatter():
        for j in range(p):
            c = (rank + j) % p
            lo, hi = c * q, min((c + 1) * q, v)
            _lib.check(lib.tv_getvc(1, part.buf.data_ptr() + lo * sb, 0, 0, nk, hi - lo, v, xv.data_ptr(), 1.0,
                                    0.0, ptrs[c] + rank * slot_bytes, _lib.stream_ptr()))

    def barrier():
        hdl.barrier(channel=0)

    def fold():
        _lib.check(lib.tv_rank_fold_range(sym.data_ptr(), slot_bytes // sb, p, chunk, ring[0][1] - ring[0][0],
                                          rank * chunk, 0, 0, 0, sym.data_ptr() + p * slot_bytes,
                                          _lib.stream_ptr()))

    def gather():
        srcs = (ctypes.c_void_p * p)(*[ptrs[c] + p * slot_bytes - c * chunk * sb for c in range(p)])
        _lib.check(lib.tv_rank_select(srcs, p, n, chunk, 0, out.data_ptr(), _lib.stream_ptr()))

    def full():
        g.tvc_reduce_fused(part, xv, 0, tv.F64)

    def timed(fn, reps=10):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda._sleep(2_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / reps * 1e3], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return round(float(t.item()), 1)

    res = {"local_tvc_us": timed(local), "scatter_us": timed(scatter), "barrier_us": timed(barrier),
           "fold_us": timed(fold), "gather_us": timed(gather), "full_us": timed(full)}
    if rank == 0:
        print(json.dumps({"world": p, **res}), flush=True)
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
