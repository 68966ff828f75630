"""The one-process-per-GPU collective plan of RankGroup, exercised on CPU over
gloo with world sizes 2 and 3: all-to-all of ring chunks, a fold per chunk
(the oracle's, injected in place of the CUDA fold kernel) and the all-gather
must reproduce the reference's ring_all_reduce / ring_all_reduce_mixed values
bit for bit, and all_gather must concatenate uneven slices in rank order."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# small buffers take the all-gather + local fold path, the last two (> 1 MB
# over the group) the all-to-all + fold + all-gather path
CASES = [("f64", 10), ("f32", 7), ("f16f32", 11), ("bf16f32", 13), ("f32f64", 5), ("f64", 1),
         ("f64", 70001), ("bf16f32", 300001)]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_data(mode_name, n, r, O):
    rng = np.random.default_rng(1000 + 17 * r + n)
    return O.demote(rng.uniform(-4, 4, n), mode_name).copy()


def _worker(rank, world, port, q):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import tenvec_oracle as O
        import paper_2501_03121_b200 as tv

        names = {torch.float64: "f64", torch.float32: "f32", torch.float16: "f16f32", torch.uint16: "bf16f32"}

        def host_fold(recv, stride, p, n, dst, *, mixed, mode, start, chunk=0):
            name = mode.name if mode is not None else names[dst.dtype]
            arr = recv.numpy()
            contribs = [arr[r * stride: r * stride + n] for r in range(p)]
            if chunk:  # whole buffers: the reference's full ring fold
                out = O.fold_mixed(contribs, name) if mixed else O.fold_exact(contribs)
            else:
                out = O.fold_chunk(contribs, start, name, mixed)
            dst.view(torch.int16 if dst.dtype == torch.uint16 else dst.dtype).copy_(
                torch.from_numpy(out.view(np.int16) if out.dtype == np.uint16 else out))

        group = tv.RankGroup(fold=host_fold)
        results = []
        for name, n in CASES:
            mode = tv.MODES[name]
            mine = _rank_data(name, n, rank, O)
            buf = torch.from_numpy(mine.copy())
            if mode.mixed:
                group.all_reduce_sum_mixed(rank, buf, mode)
            else:
                group.all_reduce_sum(rank, buf)
            everyone = [_rank_data(name, n, r, O) for r in range(world)]
            want = O.fold_mixed(everyone, name) if mode.mixed else O.fold_exact(everyone)
            results.append(bool(np.array_equal(buf.numpy().view(np.uint8), want.view(np.uint8))))
        # uneven gather: the last rank is short, like a split plan's last slab
        counts = [3] * (world - 1) + [1]
        local = torch.arange(counts[rank], dtype=torch.float64) + 10 * rank
        got = group.all_gather(rank, local, counts)
        want = np.concatenate([np.arange(c, dtype=np.float64) + 10 * r for r, c in enumerate(counts)])
        results.append(bool(np.array_equal(got.numpy(), want)))
        with pytest.raises(tv.CollectiveError):
            group.all_reduce_sum((rank + 1) % world, buf)
        results.append(group.counters[0].collective_calls == len(CASES) + 1)
        q.put((rank, results))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_rank_group_reference_values_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, res = q.get(timeout=240)
        out[r] = res
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert all(out[r]), (r, out[r])


def _failure_worker(rank, world, port, q, scenario):
    import datetime

    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=3))
    import paper_2501_03121_b200 as tv

    try:
        if scenario == "absent":
            g = tv.RankGroup(algo="exact", timeout=2.0)
            if rank == world - 1:
                import time

                time.sleep(9)
                q.put((rank, "slept"))
                return
            try:
                g.all_gather(rank, torch.ones(3, dtype=torch.float64))
                q.put((rank, "no error"))
            except tv.CollectiveTimeout as exc:
                try:
                    g.barrier(rank)
                    again = False
                except tv.CollectiveTimeout as exc2:
                    again = exc2 is exc
                q.put((rank, (exc.kind, exc.absent, again)))
        else:  # mismatched collective kinds under check=True
            g = tv.RankGroup(algo="exact", check=True, timeout=20.0)
            buf = torch.ones(8, dtype=torch.float64)
            try:
                g.all_reduce_sum(rank, buf) if rank == 0 else g.all_gather(rank, buf)
                q.put((rank, "no error"))
            except tv.CollectiveError as exc:
                q.put((rank, (type(exc).__name__, "while others run" in str(exc))))
    finally:
        q.close()
        q.join_thread()  # flush the result before leaving
        os._exit(0)  # skip the teardown handshake with a peer that may be gone


@pytest.mark.parametrize("scenario", ["absent", "mismatch"])
def test_rank_group_failure_semantics_over_gloo(scenario):
    """CollectiveTimeout names the ranks that never issued the collective
    (a ledger in the c10d store) and the group stays failed; with check=True
    a kind mismatch raises CollectiveError on every rank (comm.py:206-235)."""
    world = 3 if scenario == "absent" else 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_failure_worker, args=(r, world, port, q, scenario)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    if scenario == "absent":
        assert out[world - 1] == "slept"
        for r in range(world - 1):
            assert out[r] == ("all_gather", [world - 1], True), out
    else:
        assert out == {0: ("CollectiveError", True), 1: ("CollectiveError", True)}, out
