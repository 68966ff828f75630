"""Debug: back-to-back fused dtvc calls over loopback thread-ranks.
Prints per-call parity, barrier status and timing."""
import faulthandler
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import tenvec_oracle as O  # noqa: E402

import paper_2501_03121_b200 as tv  # noqa: E402
from paper_2501_03121_b200.loopback import LoopbackWorld  # noqa: E402

world = int(os.environ.get("W", "2"))
reps = int(os.environ.get("REPS", "12"))
cases = [((5, world * 3, 6), 1, "f64"), ((5, world * 3, 6), 1, "f32"), ((3 * world + 1, 9, 17), 0, "f16f32"),
         ((2, world * 3, 40), 1, "f64"), ((5, 6, world * 3, 7), 2, "f64")]


progress = {}


def monitor():
    dumped = False
    while True:
        time.sleep(0.5)
        if progress and not dumped and time.time() - min(progress.values()) > 3.0:
            print("=== stall: dumping stacks", {r: round(time.time() - t, 1) for r, t in progress.items()}, flush=True)
            faulthandler.dump_traceback(all_threads=True)
            dumped = True


threading.Thread(target=monitor, daemon=True).start()


def fn(rank, tr):
    g = tv.RankGroup(algo="fused", transport=tr, timeout=float(os.environ.get("TMO", "10")))
    out = []
    for shape, s, name in cases:
        mode = tv.MODES[name]
        full = O.fill_values(shape, "hash", seed=8).reshape(shape)
        host = O.demote(full.reshape(-1), name).reshape(shape)
        x = O.demote((np.arange(shape[s]) % 7) + 1.0, name).copy()
        parts, ranges = O.split(host, s, world)
        _, outs, _ = O.dtvc(parts, ranges, s, x, s, name)
        want = np.ascontiguousarray(outs[0]).reshape(-1)
        dt = tv.distribute_generated(tv.Shape(shape), s, world, mode, fill="hash", seed=8, group=g)
        for i in range(reps):
            progress[rank] = time.time()
            t0 = time.time()
            got = tv.dtvc(dt, x, s).parts[0].to_numpy().reshape(-1)
            dtm = time.time() - t0
            st = g._status.cpu().tolist() if g._status is not None else None
            eq = np.array_equal(got.view(np.uint8), want.view(np.uint8))
            nbad = int(np.sum(np.any(got.view(np.uint8).reshape(got.size, -1) != want.view(np.uint8).reshape(want.size, -1), axis=1)))
            idx = np.nonzero(np.any(got.view(np.uint8).reshape(got.size, -1) != want.view(np.uint8).reshape(want.size, -1), axis=1))[0][:8]
            out.append((shape, name, i, eq, nbad, got.size, idx.tolist(), round(dtm, 3), st, g._peer.epoch))
    progress.pop(rank, None)
    return out


lw = LoopbackWorld(world, timeout=60)
t0 = time.time()
res = lw.run(fn)
for r, rows in enumerate(res):
    for row in rows:
        if not row[3] or row[2] == 0:
            print("rank", r, row, flush=True)
print("total", round(time.time() - t0, 2), "s; bad:", sum(not row[3] for rows in res for row in rows))
