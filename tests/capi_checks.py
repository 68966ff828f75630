"""Checks of the distributed C-ABI (csrc/dist.cu) against the Python layer
it mirrors: tv_dhopm3_plan_create / tv_dhopm3_sweep bit-identical to
``dhopm3`` (hopm.py:229-354), tv_allreduce / tv_allgather identical to
RankGroup's reference-ordered collectives (comm.py:84-153).  Used by
tests/test_gpu_capi.py (one rank, no communicator) and by the NCCL worker of
tests/test_gpu_multi.py (one process per GPU, a tv_comm per rank)."""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from paper_2501_03121_b200 import _lib


def c_dhopm3(tv, comm, part, gshape, s, mode, x0, sweeps):
    """Run `sweeps` sweeps through the C-ABI on this rank's slab; returns
    (host vectors, norms per sweep)."""
    lib = _lib.load()
    d = len(gshape)
    ext = (ctypes.c_int64 * d)(*gshape)
    plan = ctypes.c_void_p()
    _lib.check(lib.tv_dhopm3_plan_create(comm, part.buf.data_ptr(), mode.tv_storage, mode.tv_compute, d, ext, s,
                                         ctypes.byref(plan)), "plan")
    xs = [tv.kernels._vec(v, mode, "x").clone() for v in x0]
    norms = torch.zeros(sweeps * d, dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    ptrs = (ctypes.c_void_p * d)(*[x.data_ptr() for x in xs])
    try:
        for sw in range(sweeps):
            _lib.check(lib.tv_dhopm3_sweep(plan, ptrs, norms[sw * d:].data_ptr(), status.data_ptr(),
                                           _lib.stream_ptr()), "sweep")
        _lib.host_wait()
    finally:
        lib.tv_dhopm3_plan_destroy(plan)
    vecs = [_lib.to_host(x).numpy() for x in xs]
    nv = _lib.to_host(norms).tolist()
    return vecs, [nv[i * d:(i + 1) * d] for i in range(sweeps)], int(_lib.to_host(status).item())


def same_run(res, c_vecs, c_norms) -> bool:
    return res.norms == c_norms and all(np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))
                                        for a, b in zip(res.vectors, c_vecs))


def run_capi_checks(rank: int, world: int, tv, comm) -> list:
    """comm: this rank's tv_comm (world > 1).  Returns (what..., ok) tuples."""
    ok = []
    lib = _lib.load()
    group = tv.RankGroup(algo="exact")
    for shape, s, name in [((world * 4, 10, 9), 0, "f64"), ((6, world * 5, 7), 1, "bf16f32"),
                           ((8, 9, world * 3), 2, "f16f32"), ((5, 6, world * 2 + 1, 4), 2, "f32f64"),
                           ((world * 8, 12, 12, 6), 3, "f32")]:
        if tv.make_split_plan(shape[s], s, world).p_eff != world:
            continue
        mode = tv.MODES[name]
        dt = tv.distribute_generated(tv.Shape(shape), s, world, mode, fill="hash", seed=5, group=group)
        x0 = tv.initial_vectors(tv.Shape(shape), mode)
        res = tv.dhopm3(dt, [v.copy() for v in x0], sweeps=3)
        vecs, norms, st = c_dhopm3(tv, comm, dt.parts[rank], shape, s, mode, x0, 3)
        ok.append(("capi-dhopm3", shape, s, name, st == 0 and same_run(res, vecs, norms)))
    # dhopm3(native=True) across the group: the C++ plan on a communicator
    # of its own, the Python driver's bits and counters
    for shape, s, name in [((world * 4, 10, 9), 0, "f64"), ((6, world * 5, 7), 1, "bf16f32")]:
        mode = tv.MODES[name]
        dt = tv.distribute_generated(tv.Shape(shape), s, world, mode, fill="hash", seed=6, group=group)
        x0 = tv.initial_vectors(tv.Shape(shape), mode)
        before = [(c.collective_calls, c.touched_elements) for c in group.counters]
        py = tv.dhopm3(dt, [v.copy() for v in x0], sweeps=2)
        mid = [(c.collective_calls, c.touched_elements) for c in group.counters]
        nat = tv.dhopm3(dt, [v.copy() for v in x0], sweeps=2, native=True)
        after = [(c.collective_calls, c.touched_elements) for c in group.counters]
        same_counts = all((m[0] - b0[0], m[1] - b0[1]) == (a[0] - m[0], a[1] - m[1])
                          for b0, m, a in zip(before, mid, after))
        ok.append(("native-dhopm3", shape, name, same_run(py, nat.vectors, nat.norms) and same_counts
                   and nat.iteration_touched == py.iteration_touched))
    # allreduce: small (one gather) and large (chunk exchange) buffers
    for n in (1001, 600_003):
        for name, algo in (("f64", _lib.TV_AR_EXACT), ("f32", _lib.TV_AR_EXACT), ("bf16f32", _lib.TV_AR_MIXED),
                           ("f16f32", _lib.TV_AR_MIXED), ("f64", _lib.TV_AR_NCCL)):
            mode = tv.MODES[name]
            g = torch.Generator().manual_seed(rank * 7 + n)
            host = tv.demote(torch.randn(n, generator=g, dtype=torch.float64).numpy(), mode)
            a = tv.kernels._vec(host, mode, "x").clone()
            b = a.clone()
            need = lib.tv_allreduce_workspace_bytes(comm, n, mode.tv_storage, algo)
            ws = torch.empty(max(need, 1), dtype=torch.uint8, device="cuda")
            _lib.check(lib.tv_allreduce(comm, a.data_ptr(), n, mode.tv_storage, mode.tv_compute, algo,
                                        ws.data_ptr(), need, _lib.stream_ptr()), "allreduce")
            if algo == _lib.TV_AR_NCCL:
                group.t.all_reduce(b, "sum")
                same = torch.allclose(a, b, rtol=1e-12, atol=0)
            else:
                (group.all_reduce_sum_mixed(rank, b, mode) if mode.mixed else group.all_reduce_sum(rank, b))
                same = torch.equal(_lib.to_host(a.view(torch.int16) if a.element_size() == 2 else a),
                                   _lib.to_host(b.view(torch.int16) if b.element_size() == 2 else b))
            ok.append(("capi-allreduce", n, name, algo, bool(same)))
    # allgather of ragged parts
    counts = [5 + 3 * r for r in range(world)]
    local = torch.arange(counts[rank], dtype=torch.float64, device="cuda") + 1000 * rank
    out = torch.empty(sum(counts), dtype=torch.float64, device="cuda")
    cnt = (ctypes.c_int64 * world)(*counts)
    _lib.check(lib.tv_allgather(comm, local.data_ptr(), out.data_ptr(), cnt, 8, _lib.stream_ptr()), "allgather")
    want = torch.cat([torch.arange(c, dtype=torch.float64) + 1000 * r for r, c in enumerate(counts)])
    ok.append(("capi-allgather", bool(torch.equal(_lib.to_host(out), want))))
    return ok
