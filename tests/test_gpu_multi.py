"""One process per GPU over NCCL (RankGroup with the default torch transport):
the shared transport checks of tests/multirank_checks.py -- dtvc with the split
on and off the contraction mode in every transport, the fused split-mode
reduction over peer memory, assembly, the fold-and-normalise and dhopm3 --
against the oracle.  Needs >= 2 visible GPUs (skipped otherwise; run with
`gpurun --gpus 2|4`).  The same checks run on one GPU as thread-ranks in
tests/test_gpu_loopback.py."""

import os
import socket
import sys

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as dist

    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        import multirank_checks
        import tenvec_oracle as O
        import paper_2501_03121_b200 as tv

        ok = multirank_checks.run_checks(rank, world, lambda algo: tv.RankGroup(algo=algo), tv, O)
        ok += _capi(rank, world, tv)
        q.put((rank, ok))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, [("error", repr(exc)[:500], False)]))
    finally:
        dist.destroy_process_group()


def _capi(rank, world, tv):
    """The distributed C-ABI with one NCCL communicator per process (the
    unique id travels over torch.distributed, as any launcher would ship it)."""
    import ctypes

    import torch.distributed as dist

    import capi_checks
    from paper_2501_03121_b200 import _lib

    lib = _lib.load()
    uid = ctypes.create_string_buffer(128)
    if rank == 0:
        _lib.check(lib.tv_comm_get_unique_id(uid), "unique id")
    box = [bytes(uid.raw)]
    dist.broadcast_object_list(box, src=0)
    uid = ctypes.create_string_buffer(box[0], 128)
    comm = ctypes.c_void_p()
    _lib.check(lib.tv_comm_init_rank(uid, world, rank, ctypes.byref(comm)), "comm")
    try:
        r, n = ctypes.c_int(), ctypes.c_int()
        lib.tv_comm_rank_size(comm, ctypes.byref(r), ctypes.byref(n))
        ok = [("capi-comm", r.value == rank and n.value == world)]
        ok += capi_checks.run_capi_checks(rank, world, tv, comm)
    finally:
        torch.cuda.synchronize()
        lib.tv_comm_destroy(comm)
    return ok


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_rank_group_over_nccl_matches_oracle():
    world = min(torch.cuda.device_count(), 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(world):
        r, res = q.get(timeout=900)
        results[r] = res
    for p in procs:
        p.join(timeout=120)
    for r, res in results.items():
        bad = [c for c in res if not c[-1]]
        assert not bad, (r, bad)
