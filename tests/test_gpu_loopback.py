"""The one-process-per-GPU transports of RankGroup -- "fused" (the split-mode
TVC writing owner ranges into peer slots, owner fold, peer gather, with and
without the side-stream finish), "p2p", "exact" and dHOPM3's
fold-and-normalise -- run as p thread-ranks on ONE GPU through the loopback
transport (paper_2501_03121_b200/loopback.py), with the same kernels, the same
device barrier and the same index math as across GPUs.  The checks are
tests/multirank_checks.py, shared with the NCCL test; here they run in the
one-GPU driver suite.  Plus the failure semantics of the reference's
WorkerGroup (comm.py:206-235): absent ranks named by a device barrier or a
host collective that times out, kind mismatches, and the collective
peer-memory fallback."""

import os
import warnings

import numpy as np
import pytest
import torch

import multirank_checks
from paper_2501_03121_b200._lib import to_host

pytestmark = pytest.mark.gpu


# world 8 runs with one owner-launch lane per rank: 8 thread-ranks with two
# lanes each exceed the GPU's 32 hardware queues (CUDA_DEVICE_MAX_CONNECTIONS),
# two ranks' streams then alias one queue and a spinning barrier blocks the
# other rank's arrival (measured: the host all_gather timed out); one process
# per GPU has no such aliasing
@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_loopback_transports_match_oracle(tv, oracle, world, monkeypatch):
    from paper_2501_03121_b200.loopback import LoopbackWorld

    if world > 4:
        monkeypatch.setenv("TENVEC_B200_OWNER_LANES", "1")

    lw = LoopbackWorld(world, timeout=120)
    out = lw.run(lambda rank, tr: multirank_checks.run_checks(
        rank, world, lambda algo: tv.RankGroup(algo=algo, transport=tr, timeout=120), tv, oracle))
    for rank, res in enumerate(out):
        bad = [c for c in res if not c[-1]]
        assert not bad, (rank, bad)
        assert len(res) > 100


def test_fused_plan_geometry(tv):
    from paper_2501_03121_b200.comm import fused_plan

    # slab owners with a ragged and an empty last owner: u = 5 over 4 ranks
    pl = fused_plan(5, 7, 4, 8)
    assert pl.along_u and pl.bounds == ((0, 2), (2, 4), (4, 5), (5, 5)) and pl.sizes == (14, 14, 7, 0)
    assert pl.n == 35 and pl.slot_bytes % 16 == 0 and pl.slot_elems * 8 == pl.slot_bytes
    # column owners (u == 1) and the fallback (1 < u < p)
    pl = fused_plan(1, 153, 4, 4)
    assert not pl.along_u and pl.sizes == (39, 39, 39, 36)
    assert fused_plan(2, 10, 3, 8) is None and fused_plan(9, 10, 1, 8) is None


def _run_catching(lw, fn):
    def body(rank, tr):
        try:
            return fn(rank, tr)
        except Exception as exc:  # noqa: BLE001 - the test inspects it
            return exc
    return lw.run(body)


def test_device_barrier_timeout_names_the_absent_rank(tv, oracle):
    """Rank 1 skips the second fused reduction: rank 0's device barrier gives
    up after the group timeout (no trap, no hang) and wait() raises
    CollectiveTimeout naming rank 1; the group stays failed."""
    from paper_2501_03121_b200.loopback import LoopbackWorld

    shape = (6, 8, 4)
    lw = LoopbackWorld(2, timeout=30)

    def fn(rank, tr):
        g = tv.RankGroup(algo="fused", transport=tr, timeout=1.5)
        dt = tv.distribute_generated(tv.Shape(shape), 0, 2, tv.F64, group=g)
        x = np.ones(shape[0])
        tv.dtvc(dt, x, 0)
        g.wait()
        if rank == 1:
            return "left"
        tv.dtvc(dt, x, 0)
        try:
            g.wait()
        except tv.CollectiveTimeout as exc:
            again = None
            try:
                g.barrier(0)
            except tv.CollectiveTimeout as exc2:
                again = exc2
            return exc, again
        return "no timeout"

    res = _run_catching(lw, fn)
    assert res[1] == "left"
    exc, again = res[0]
    assert exc.kind == "dtvc_reduce" and exc.absent == [1]
    assert again is exc


def test_host_collective_timeout_and_kind_mismatch(tv):
    from paper_2501_03121_b200.loopback import LoopbackWorld

    lw = LoopbackWorld(2, timeout=1.0)

    def absent(rank, tr):
        g = tv.RankGroup(algo="exact", transport=tr)
        if rank == 1:
            return "left"
        return g.all_gather(0, torch.ones(4, device="cuda"))

    res = _run_catching(lw, absent)
    assert isinstance(res[0], tv.CollectiveTimeout) and res[0].absent == [1] and res[0].kind == "all_gather"

    lw = LoopbackWorld(2, timeout=10.0)

    def mismatch(rank, tr):
        g = tv.RankGroup(algo="exact", transport=tr, check=True)
        buf = torch.ones(8, device="cuda")
        return g.all_reduce_sum(rank, buf) if rank == 0 else g.all_gather(rank, buf)

    res = _run_catching(lw, mismatch)
    for r in (0, 1):
        assert isinstance(res[r], tv.CollectiveError) and not isinstance(res[r], tv.CollectiveTimeout)
        assert "while others run" in str(res[r])


def test_peer_memory_fallback_is_collective(tv, oracle):
    """One rank cannot map peer memory: EVERY rank falls back to the exact
    transport together (no rank left waiting in a device barrier) and the
    results are still the reference's."""
    from paper_2501_03121_b200.loopback import LoopbackWorld

    O = oracle
    shape = (8, 12, 5)
    full = O.fill_values(shape, "hash", seed=2).reshape(shape)
    x = (np.arange(shape[0]) % 7) + 1.0
    parts, ranges = O.split(full, 0, 2)
    _, outs, _ = O.dtvc(parts, ranges, 0, x, 0, "f64")
    lw = LoopbackWorld(2, timeout=30, fail_peer_rank=1)

    def fn(rank, tr):
        g = tv.RankGroup(algo="fused", transport=tr)
        dt = tv.distribute_generated(tv.Shape(shape), 0, 2, tv.F64, fill="hash", seed=2, group=g)
        with warnings.catch_warnings(record=True):
            warnings.simplefilter("always")
            got = tv.dtvc(dt, x, 0).parts[0].to_numpy()
        g.wait()
        return g.algo, got

    for algo, got in lw.run(fn):
        assert algo == "exact"
        assert np.array_equal(got, outs[0].reshape(-1))


def test_dhopm3_timeout_argument_bounds_the_group(tv):
    """dhopm3(timeout=) is the group's collective timeout for the run (the
    reference's WorkerGroup(timeout), hopm.py:263) and is restored after."""
    from paper_2501_03121_b200.loopback import LoopbackWorld

    lw = LoopbackWorld(2, timeout=30)
    seen = []

    def fn(rank, tr):
        g = tv.RankGroup(algo="fused", transport=tr, timeout=77.0)
        A = tv.Tensor.from_array(np.random.default_rng(3).standard_normal((6, 5, 4)))
        orig = g.wait

        def spy(timeout=None):
            seen.append(g.timeout)
            return orig(timeout)

        g.wait = spy
        tv.dhopm3(tv.distribute(A, 0, 2, group=g), sweeps=2, timeout=12.5)
        return g.timeout

    assert lw.run(fn) == [77.0, 77.0]
    assert seen == [12.5, 12.5]


@pytest.mark.parametrize("world", [2, 4])
def test_loopback_dhopm3_order4_twenty_sweeps_equals_in_process(tv, oracle, world):
    """C4's code path at 96^4 across a RankGroup (fold-and-normalise epilogue,
    the split mode's gather, NCCL-free loopback): 20 sweeps bit-identical to
    the in-process run of the same split, within 1e-12 of the oracle."""
    from paper_2501_03121_b200.loopback import LoopbackWorld

    O = oracle
    shape = (96,) * 4
    vals = O.fill_values(shape, "hash", seed=1).reshape(shape)
    x0 = O.initial_vectors(shape, "f64")
    A = tv.Tensor.from_array(vals)
    inproc = tv.dhopm3(tv.distribute(A, 3, world), [v.copy() for v in x0], sweeps=20)

    def fn(rank, tr):
        g = tv.RankGroup(transport=tr, timeout=120)
        dt = tv.distribute_generated(tv.Shape(shape), 3, world, tv.F64, fill="hash", seed=1, group=g)
        return tv.dhopm3(dt, [v.copy() for v in x0], sweeps=20)

    for res in LoopbackWorld(world, timeout=120).run(fn):
        assert res.norms == inproc.norms
        for a, b in zip(res.vectors, inproc.vectors):
            assert np.array_equal(a.view(np.uint8), b.view(np.uint8))
    vecs, norms = O.dhopm3(vals, 3, world, x0, 20, "f64")
    np.testing.assert_allclose(np.asarray(inproc.norms), np.asarray(norms), rtol=1e-12, atol=0)


def test_c3_full_size_dtvc_split_mode_sampled(tv):
    """C3 at full size, 96^5 fp32 split along s = 4: every mode of a sweep
    over 4 thread-ranks with the default transport ("fused"; the 340 MB
    split-mode reduction finishes on the side stream under the other modes),
    then the in-process 8-rank split with the exact reduction and with
    defer -- sampled outputs bitwise equal to the closed form of the hash
    fill (exact: fp32 sums of 96 products <= 97 * 5 stay below 2^24)."""
    import gc

    from paper_2501_03121_b200 import verify
    from paper_2501_03121_b200.loopback import LoopbackWorld

    shape = (96,) * 5
    s = 4
    xs = [((np.arange(96) % 5) + 1.0).astype(np.float32) for _ in range(5)]
    idx = {k: verify.sample_outputs(shape, k, 192, seed=k) for k in range(5)}
    want = {k: verify.tvc_expected(shape, k, xs[k], "hash", 3, idx[k]) for k in range(5)}

    def fn(rank, tr):
        g = tv.RankGroup(transport=tr, timeout=300)
        dt = tv.distribute_generated(tv.Shape(shape), s, 4, tv.F32, fill="hash", seed=3, group=g)
        out = tv.dtvc_sweep(dt, xs)
        g.wait()
        res = {}
        for k in range(5):
            if k == s:
                res[k] = to_host(out[k].parts[0].buf[torch.from_numpy(idx[k]).cuda()]).numpy()
        # the ranks own slabs of the k != s outputs along the split mode
        # (now mode 3); rank 0 checks its own outputs' samples
        return res, {k: to_host(out[k].parts[rank].buf).numpy() if k != s else None for k in range(5)}

    lw = LoopbackWorld(4, timeout=300)
    results = lw.run(fn)
    for rank, (red, _) in enumerate(results):
        assert verify.check_tvc_samples(red[s], want[s], "single"), rank
    # reassemble the k != s outputs (split along mode 3 of the output) and check
    for k in range(4):
        # rank r holds output columns [24 r, 24 r + 24) of the last output mode
        full = np.stack([results[r][1][k].reshape(-1, 24) for r in range(4)], axis=1).reshape(-1)
        assert verify.check_tvc_samples(full[idx[k]], want[k], "single"), k
    del results
    gc.collect()
    torch.cuda.empty_cache()

    dt = tv.distribute_generated(tv.Shape(shape), s, 8, tv.F32, fill="hash", seed=3)
    red = tv.dtvc(dt, xs[s], s)
    got = red.parts[0].buf[torch.from_numpy(idx[s]).cuda()].cpu().numpy()
    assert verify.check_tvc_samples(got, want[s], "single")
    part = tv.dtvc(dt, xs[s], s, defer=True)
    assert part.kind == tv.PARTIAL_SUM and len(part.parts) == 8
    acc = sum(p.buf[torch.from_numpy(idx[s]).cuda()].double().cpu().numpy() for p in part.parts)
    assert np.array_equal(acc, want[s])
