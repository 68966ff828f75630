#!/usr/bin/env python
"""The paper's mixed-precision dHOPM3 comparison (its
Fig. HOPM-mix-prec) on B200s: one dHOPM3 run per precision mode on the SAME
4096^3 tensor (hash fill, integers in [1, 97] scaled by 2^-7 so fp16 outputs
stay finite -- exact in every storage format), split along s = 2 over the N
GPUs of the torchrun job:

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
        scripts/mixed_precision_hopm.py [--shape 4096,4096,4096] [--sweeps 10]

Per mode: event-timed device time of the public dhopm3 call (max over ranks),
the reference cost model's streamed bytes of a sweep (schedule.sweep_bytes) /
time, the speed-up over f64 in time, and the accuracy of the final lambda and
vectors against the f64 run (relative errors; the stated bounds are in
BOUNDS).  One JSON line per mode, then a summary table (rank 0).
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

MODES = ("f64", "f32f64", "f32", "f16f32", "bf16f32")
# stated accuracy bounds after the run, relative to the f64 run: lambda, and
# the max-norm error of the unit direction vectors (storage rounding of a
# unit vector dominates: 2^-24 f32, 2^-11 f16, 2^-8 bf16, times a small factor)
BOUNDS = {"f64": (0.0, 0.0), "f32f64": (1e-6, 1e-6), "f32": (1e-5, 1e-5), "f16f32": (2e-3, 2e-3),
          "bf16f32": (1.6e-2, 1.6e-2)}


def _scale(tv, dt, factor: float) -> None:
    """In place, exactly (a power of two): tv_axpby with y = x, beta = 0."""
    lib = tv._lib.load()
    mode = dt.mode
    for part in dt.parts:
        if part is not None:
            tv._lib.check(lib.tv_axpby(factor, part.buf.data_ptr(), 0.0, part.buf.data_ptr(), mode.tv_storage,
                                       mode.tv_compute, part.size, tv._lib.stream_ptr()), "scale")


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="4096,4096,4096")
    ap.add_argument("--split", type=int, default=2)
    ap.add_argument("--sweeps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--modes", default=",".join(MODES))
    ap.add_argument("--scale-log2", type=int, default=7, help="tensor values scaled by 2^-this (fp16 range)")
    args = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist

    import bench
    import paper_2501_03121_b200 as tv

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    shape = tv.Shape(tuple(int(v) for v in args.shape.split(",")))
    s = args.split
    peak = float(bench._peaks().get("hbm_gbs", 6650.0))
    ref = None
    rows = []
    for name in args.modes.split(","):
        mode = tv.MODES[name]
        group = tv.RankGroup() if world > 1 else None
        dt = tv.distribute_generated(shape, s, world, mode, fill="hash", seed=1, group=group)
        # the fill's integers in [1, 97] scaled by 2^-7 (exact in every format):
        # unscaled, a 4096^3 contraction's outputs (~49 n) overflow fp16
        _scale(tv, dt, 2.0 ** -args.scale_log2)
        x0 = tv.initial_vectors(shape, mode)
        tv.dhopm3(dt, x0, sweeps=args.warmup)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clocks = bench.ClockSampler() if rank == 0 else None
        if clocks:
            clocks.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = tv.dhopm3(dt, x0, sweeps=args.sweeps)
        e1.record()
        torch.cuda.synchronize()
        clk = clocks.stop() if clocks else None
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        job = sum(tv.schedule.sweep_bytes(shape.extents, s, world, mode.storage_bytes))
        value = job * args.sweeps / (ms / 1e3) / 1e9
        vecs = [tv.promote(v, mode).astype(np.float64) for v in res.vectors]
        lam = float(res.norms[-1][-1])
        del dt, res
        gc.collect()
        torch.cuda.empty_cache()
        if name == "f64":
            ref = (lam, vecs, ms)
        line = {"mode": name, "shape": list(shape.extents), "split_mode": s, "n_gpus": world,
                "sweeps": args.sweeps, "ms_per_sweep": round(ms / args.sweeps, 4), "value": round(value, 1),
                "unit": "GB/s", "per_gpu_frac": round(value / world / peak, 4), "lambda": lam, "clocks": clk,
                "storage_bytes": mode.storage_bytes}
        if ref is not None:
            lam_err = abs(lam - ref[0]) / abs(ref[0])
            vec_err = max(float(np.max(np.abs(a - b))) for a, b in zip(vecs, ref[1]))
            lb, vb = BOUNDS[name]
            line.update({"speedup_vs_f64": round(ref[2] / ms, 3), "lambda_rel_err_vs_f64": lam_err,
                         "vector_max_err_vs_f64": vec_err, "bound_lambda": lb, "bound_vector": vb,
                         "within_bound": bool(lam_err <= lb and vec_err <= vb)})
        rows.append(line)
        if rank == 0:
            print(json.dumps(line), flush=True)
    if rank == 0:
        print("| mode | bytes/elem | ms/sweep | GB/s (job) | frac/GPU | speed-up vs f64 | lambda rel err | vec max err |")
        print("|---|---|---|---|---|---|---|---|")
        for r in rows:
            sp = r.get("speedup_vs_f64", "-")
            le = r.get("lambda_rel_err_vs_f64")
            ve = r.get("vector_max_err_vs_f64")
            print(f"| {r['mode']} | {r['storage_bytes']} | {r['ms_per_sweep']} | {r['value']} | {r['per_gpu_frac']} "
                  f"| {sp} | {'-' if le is None else f'{le:.3g}'} | {'-' if ve is None else f'{ve:.3g}'} |")
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
