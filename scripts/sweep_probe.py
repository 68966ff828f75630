#!/usr/bin/env python
"""Where an N-GPU dTVC sweep's time goes (any BASELINE sweep workload):
event-timed, max over ranks, each phase alone and back to back --
the modes k != s, the split-mode contraction alone (defer) and with its
fused reduction, and the whole sweep (overlap rules as in bench.py).

    torchrun --nproc-per-node N scripts/sweep_probe.py [c3|c2]
"""
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

    wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    mode = tv.MODES[wl["mode"]]
    shape = tv.Shape(wl["shape"])
    s = wl["s"]
    g = tv.RankGroup()
    dt = tv.distribute_generated(shape, s, world, mode, fill="hash", seed=1, group=g)
    xs = [torch.from_numpy(bench.tv_demote_host(np.arange(n) % 7 + 1.0, mode)).cuda() for n in shape.extents]
    d = shape.order

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

    out = {"workload": wl["desc"], "n": world}
    for k in range(d):
        if k != s:
            out[f"k{k}"] = timed(lambda k=k: tv.dtvc(dt, xs[k], k))
    out["others_back_to_back"] = timed(lambda: [tv.dtvc(dt, xs[k], k) for k in range(d) if k != s])
    out[f"k{s}_defer_local_tvc"] = timed(lambda: tv.dtvc(dt, xs[s], s, defer=True))
    out[f"k{s}_fused_reduce"] = timed(lambda: tv.dtvc(dt, xs[s], s))
    out["sweep_serial"] = timed(lambda: tv.dtvc_sweep(dt, xs, overlap=False))
    out["sweep_overlap"] = timed(lambda: tv.dtvc_sweep(dt, xs, overlap=True))
    keep = []
    out["sweep_overlap_results_kept"] = timed(lambda: keep.append(tv.dtvc_sweep(dt, xs, overlap=True)) or
                                              (len(keep) > 2 and keep.pop(0)))
    # per call, this rank
    per = []
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tv.dtvc_sweep(dt, xs, overlap=True)
        e1.record()
        torch.cuda.synchronize()
        per.append(round(e0.elapsed_time(e1), 3))
    allper = [None] * world
    dist.all_gather_object(allper, per)
    out["per_call_per_rank"] = allper
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
