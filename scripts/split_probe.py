#!/usr/bin/env python
"""Where the N-GPU C2 step goes: event-timed dtvc per mode (k = s with and
without its reduction, per transport) on every rank; rank 0 prints the max
over ranks.  torchrun --nproc-per-node N scripts/split_probe.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> int:
    import torch
    import torch.distributed as dist

    import paper_2501_03121_b200 as tv

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    out = {}
    for algo in ("fused", "exact"):
        g = tv.RankGroup(algo=algo)
        shape = tv.Shape((2048, 2048, 2048))
        dt = tv.distribute_generated(shape, 0, world, tv.F64, fill="hash", seed=1, group=g)
        xs = [torch.ones(2048, dtype=torch.float64, device="cuda") for _ in range(3)]

        def timed(fn, reps=5):
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
            t = torch.tensor([e0.elapsed_time(e1) / reps], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return round(float(t.item()), 4)

        out[algo] = {
            "k0_defer": timed(lambda: tv.dtvc(dt, xs[0], 0, defer=True)),
            "k0_reduced": timed(lambda: tv.dtvc(dt, xs[0], 0)),
            "k1": timed(lambda: tv.dtvc(dt, xs[1], 1)),
            "k2": timed(lambda: tv.dtvc(dt, xs[2], 2)),
            "sweep": timed(lambda: tv.dtvc_sweep(dt, xs)),
        }
        del dt
        torch.cuda.empty_cache()
    if rank == 0:
        print(json.dumps({"world": world, "ms": out}), flush=True)
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
