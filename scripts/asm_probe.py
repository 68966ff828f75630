#!/usr/bin/env python
"""Time one disjoint output's reassembly (undistribute) per strategy at N GPUs,
event-timed, max over ranks: C3's k = 0 output (96^4 fp32, split on the last
mode).  torchrun --nproc-per-node N scripts/asm_probe.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    import numpy as np
    import torch
    import torch.distributed as dist

    import bench
    import paper_2501_03121_b200 as tv
    from paper_2501_03121_b200 import comm as C

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    wl = bench.WORKLOADS["c3"]
    mode = tv.MODES[wl["mode"]]
    shape = tv.Shape(wl["shape"])
    g = tv.RankGroup()
    dt = tv.distribute_generated(shape, wl["s"], world, mode, fill="hash", seed=1, group=g)
    x = torch.from_numpy(bench.tv_demote_host(np.arange(96) % 7 + 1.0, mode)).cuda()
    res = tv.dtvc(dt, x, 0)
    del dt
    torch.cuda.empty_cache()

    def timed(fn, reps=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / reps], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return round(float(t.item()), 4)

    out = {"n": world, "output_MB": res.parts[rank].size * 4 * world / 1e6}
    for mc_min, one in ((3, True), (0, True), (0, False)):
        C._MULTICAST_MIN, C._PUSH_ONE_LAUNCH = mc_min, one
        key = f"interleave_mcmin{mc_min}_one{int(one)}"
        out[key] = timed(lambda: tv.undistribute(res, "interleave"))
        out[key + "_path"] = g.assembly_path
        got = tv.undistribute(res, "interleave").buf
        ref = tv.undistribute(res, "gather-copy").buf
        out[key + "_same_as_gather_copy"] = bool(torch.equal(got.view(torch.int32), ref.view(torch.int32)))
    out["gather-copy"] = timed(lambda: tv.undistribute(res, "gather-copy"))
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
