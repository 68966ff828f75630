"""The checks every RankGroup transport must pass, shared by the two ways of
running ranks: one process per GPU over NCCL (tests/test_gpu_multi.py, needs
>= 2 GPUs) and p thread-ranks on one GPU over the loopback transport
(tests/test_gpu_loopback.py, runs in the one-GPU driver suite).  Both run the
same RankGroup code -- fused / p2p / exact transports, the device barrier,
the fold-and-normalise -- so a pass on the loopback is evidence for the code
path behind every N > 1 number.

``run_checks(rank, world, make_group)`` returns a list of
(what..., passed) tuples; ``make_group(algo)`` builds this rank's RankGroup.
Reference semantics checked: dtvc hopm.py:95-150, ring folds comm.py:84-134,
undistribute hopm.py:76-84, dhopm3 hopm.py:229-354.
"""

from __future__ import annotations

import threading

import numpy as np
import torch

from paper_2501_03121_b200._lib import to_host

_CACHE: dict = {}
_LOCK = threading.Lock()


def _memo(key, fn):
    """Oracle results computed once per process (thread-ranks share them)."""
    with _LOCK:
        if key not in _CACHE:
            _CACHE[key] = fn()
        return _CACHE[key]

MODES = ("f64", "f32", "f32f64", "bf16f32", "f16f32")
# float-data tolerance of one contraction per mode (normwise)
FLOAT_TOL = {"f64": 1e-12, "f32": 1e-5, "f32f64": 1e-6, "f16f32": 2e-3, "bf16f32": 1.6e-2}


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def _same(a, b) -> bool:
    return bool(np.array_equal(_bits(a), _bits(np.asarray(b).reshape(-1))))


def _dev(v: torch.Tensor) -> torch.Tensor:
    return v.cuda() if v.dtype != torch.uint16 else v.view(torch.int16).cuda().view(torch.uint16)


def _normwise(got, want, name, O) -> float:
    g = O.promote(np.asarray(got).reshape(-1), name).astype(np.float64)
    w = O.promote(np.asarray(want).reshape(-1), name).astype(np.float64)
    return float(np.linalg.norm(g - w) / max(np.linalg.norm(w), 1e-300))


def run_checks(rank: int, world: int, make_group, tv, O, *, quick: bool = False) -> list:
    ok: list = []
    group = make_group("exact")

    # dtvc on a device-generated 5-mode tensor: every k, split on / off k,
    # single calls and sweeps (side-stream reduction on and off)
    shape = (6, 8, world * 3, 5, 4)
    full = O.fill_values(shape, "hash", seed=4).reshape(shape)
    for name in MODES[:2] if quick else MODES:
        mode = tv.MODES[name]
        host = O.demote(full.reshape(-1), name).reshape(shape)
        for s in sorted({2} | ({4} if tv.make_split_plan(4, 4, world).p_eff == world else set())):
            dt = tv.distribute_generated(tv.Shape(shape), s, world, mode, fill="hash", seed=4, group=group)
            parts, ranges = O.split(host, s, world)
            xs = [O.demote((np.arange(shape[k]) % 5) + 1.0, name).copy() for k in range(5)]
            sweeps = {ov: tv.dtvc_sweep(dt, xs, overlap=ov) for ov in (False, True)}
            for k in range(5):
                res = tv.dtvc(dt, xs[k], k)
                _, outs, _ = _memo(("5d", world, name, s, k), lambda: O.dtvc(parts, ranges, s, xs[k], k, name))
                want = outs[0] if k == s else outs[rank]
                for tag, r in (("dtvc", res), ("sweep", sweeps[False][k]), ("sweep-ovl", sweeps[True][k])):
                    got = (r.parts[0] if k == s else r.parts[rank]).to_numpy()
                    ok.append((name, s, k, tag, _same(got, want)))

    # reductions above the small-gather threshold: all-to-all + fold +
    # all-gather ("exact"), and the same fold over peer memory ("p2p")
    big = (64, 64, 2 * world, 64)
    fullb = O.fill_values(big, "hash", seed=6).reshape(big)
    p2p = make_group("p2p")
    for name in ("f32", "bf16f32", "f64"):
        mode = tv.MODES[name]
        hostb = O.demote(fullb.reshape(-1), name).reshape(big)
        x = O.demote((np.arange(big[2]) % 3) + 1.0, name).copy()
        parts, ranges = O.split(hostb, 2, world)
        _, outs, _ = O.dtvc(parts, ranges, 2, x, 2, name)
        for tag, grp in (("exact", group), ("p2p", p2p)):
            dt = tv.distribute_generated(tv.Shape(big), 2, world, mode, fill="hash", seed=6, group=grp)
            for _ in range(2):  # twice: the peer buffer is reused
                got = tv.dtvc(dt, x, 2).parts[0].to_numpy()
            ok.append((name, "big-reduce", tag, _same(got, outs[0])))
    # ragged reduction (n not a multiple of p or of 16 bytes) over peer memory
    rag = torch.arange(1, 300_003, dtype=torch.float32, device="cuda") * (rank + 1)
    want = torch.arange(1, 300_003, dtype=torch.float32) * sum(r + 1 for r in range(world))
    p2p.all_reduce_sum(rank, rag)
    ok.append(("f32", "ragged-p2p", 0, bool(torch.equal(to_host(rag), want))))

    # the split-mode contraction fused with its reduction over peer memory
    # (algo="fused"): slab-range owners (u >= p, a ragged / empty last
    # owner), column-range owners (u == 1, unaligned columns), the fallback
    # (1 < u < p); single calls, and sweeps with the fold + gather on the
    # side stream (finish_stream) or in line
    fused = make_group("fused")
    fshapes = [((5, 6, world * 3, 7), 2), ((world * 4, 30, 7), 0), ((3 * world + 1, 9, 17), 0),
               ((5, world * 3, 6), 1), ((3, world * 2, 50), 1), ((2, world * 3, 40), 1)]
    for fshape, s in fshapes[:3] if quick else fshapes:
        fullf = O.fill_values(fshape, "hash", seed=8).reshape(fshape)
        if tv.make_split_plan(fshape[s], s, world).p_eff != world:
            continue
        for name in MODES:
            mode = tv.MODES[name]
            hostf = O.demote(fullf.reshape(-1), name).reshape(fshape)
            xs = [O.demote((np.arange(n) % 7) + 1.0, name).copy() for n in fshape]
            parts, ranges = O.split(hostf, s, world)
            _, outs, _ = O.dtvc(parts, ranges, s, xs[s], s, name)
            dt = tv.distribute_generated(tv.Shape(fshape), s, world, mode, fill="hash", seed=8, group=fused)
            for _ in range(2):  # twice: the peer slots are reused
                got = tv.dtvc(dt, xs[s], s).parts[0].to_numpy()
            ok.append((name, "fused", fshape, _same(got, outs[0])))
            for ov in (False, True):
                sweep = tv.dtvc_sweep(dt, xs, overlap=ov)
                for k in range(len(fshape)):
                    _, ko, _ = _memo(("fs", world, fshape, name, s, k),
                                     lambda: O.dtvc(parts, ranges, s, xs[k], k, name))
                    want = ko[0] if k == s else ko[rank]
                    got = (sweep[k].parts[0] if k == s else sweep[k].parts[rank]).to_numpy()
                    ok.append((name, "fused-sweep", fshape, k, ov, _same(got, want)))
    # float data: the fused transport's owner-range launches may round
    # differently from the full-slab TVC of the exact transport; within the
    # per-mode TVC tolerance of each other and of the oracle
    fshape = (4 * world, 33, 70)
    rng = np.random.default_rng(11)
    vals = rng.standard_normal(fshape)
    for name in MODES:
        mode = tv.MODES[name]
        A = tv.Tensor.from_array(vals, mode)
        x = O.demote(rng.standard_normal(fshape[0]), name).copy()
        got_f = tv.dtvc(tv.distribute(A, 0, world, group=fused), x, 0).parts[0].to_numpy()
        got_e = tv.dtvc(tv.distribute(A, 0, world, group=group), x, 0).parts[0].to_numpy()
        host = A.to_numpy().reshape(fshape)
        parts, ranges = O.split(host, 0, world)
        _, outs, _ = O.dtvc(parts, ranges, 0, x, 0, name)
        tol = FLOAT_TOL[name]
        ok.append((name, "fused-float", _normwise(got_f, outs[0], name, O) <= tol
                   and _normwise(got_f, got_e, name, O) <= tol))

    # on-device assembly: disjoint results gathered and repacked, deferred
    # partial sums gathered and folded (undistribute, hopm.py:76-84)
    ashape = (5, world * 3, 4, 6)
    fulla = O.fill_values(ashape, "hash", seed=9).reshape(ashape)
    for name in ("f64", "f32", "bf16f32"):
        mode = tv.MODES[name]
        hosta = O.demote(fulla.reshape(-1), name).reshape(ashape)
        dt = tv.distribute_generated(tv.Shape(ashape), 1, world, mode, fill="hash", seed=9, group=group)
        ok.append((name, "assemble-input", _same(tv.undistribute(dt).to_numpy(), hosta)))
        # the same through the fused group: interleave = repack straight from
        # the peers' parts in peer memory; gather-copy = NCCL all-gather + repack
        dtf = tv.distribute_generated(tv.Shape(ashape), 1, world, mode, fill="hash", seed=9, group=fused)
        for strategy in ("interleave", "gather-copy"):
            for _ in range(2):  # twice: the peer buffer is reused
                got = tv.undistribute(dtf, strategy).to_numpy()
            ok.append((name, "assemble-peer", strategy, _same(got, hosta)))
            x = O.demote((np.arange(ashape[0]) % 4) + 1.0, name).copy()
            got = tv.undistribute(tv.dtvc(dtf, x, 0), strategy).to_numpy()
            ok.append((name, "assemble-peer-out", strategy, _same(got, O.tvc(hosta.reshape(-1), ashape, x, 0, name))))
        pb = getattr(fused, "_peer", None)
        if pb is not None and pb.mc:  # 16-byte runs: one multicast store per unit, forced from 2 ranks on
            from paper_2501_03121_b200 import comm as C

            saved, C._MULTICAST_MIN = C._MULTICAST_MIN, 2
            try:
                for _ in range(2):
                    got = tv.undistribute(dtf, "interleave").to_numpy()
            finally:
                C._MULTICAST_MIN = saved
            ok.append((name, "assemble-multicast", fused.assembly_path == "multicast" and _same(got, hosta)))
        # runs that are not 16-byte multiples take the per-peer push
        oshape = (3, world * 3 - 1, 5)
        hosto = O.demote(O.fill_values(oshape, "hash", seed=4), name).reshape(oshape)
        dto = tv.distribute_generated(tv.Shape(oshape), 1, world, mode, fill="hash", seed=4, group=fused)
        ok.append((name, "assemble-peer-ragged", _same(tv.undistribute(dto, "interleave").to_numpy(), hosto)))
        for k in (0, 3):
            x = O.demote((np.arange(ashape[k]) % 4) + 1.0, name).copy()
            got = tv.undistribute(tv.dtvc(dt, x, k)).to_numpy()
            ok.append((name, "assemble", k, _same(got, O.tvc(hosta.reshape(-1), ashape, x, k, name))))
        x = O.demote((np.arange(ashape[1]) % 4) + 1.0, name).copy()
        got = tv.undistribute(tv.dtvc(dt, x, 1, defer=True)).to_numpy()
        want = O.tvc(hosta.reshape(-1), ashape, x, 1, name)
        # brain storage truncates each rank's partial sum before the fold
        ok.append((name, "assemble-partial", bool(np.allclose(O.promote(got, name), O.promote(want, name),
                                                              rtol=1e-2 if name == "bf16f32" else 1e-6))))
        parts_h, ranges_h = O.split(hosta, 1, world)
        _, pouts, _ = O.dtvc(parts_h, ranges_h, 1, x, 1, name, defer=True)
        ok.append((name, "assemble-partial-exact", _same(got, O.undistribute_partial(pouts, name))))

    # the dHOPM3 reduction with the normalisation in the fold's epilogue:
    # the same bits as all_reduce_sum + normalize
    for name in MODES:
        mode = tv.MODES[name]
        for n in (384, 4096, 1001):
            v = _dev(torch.from_numpy(O.demote(np.random.default_rng(rank + n).standard_normal(n), name).copy()))
            ref = v.clone()
            group.all_reduce_sum_mixed(rank, ref, mode) if mode.mixed else group.all_reduce_sum(rank, ref)
            ref_norm = tv.normalize(ref, mode=mode)
            dst = torch.empty_like(v)
            slot = torch.empty(1, dtype=torch.float64, device="cuda")
            cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
            okf = group.all_reduce_normalize(rank, v, mode, dst, slot, None, cnt)
            same = bool(torch.equal(to_host(as_i(dst)), to_host(as_i(ref))))
            ok.append((name, "fold-normalize", n, okf and same and float(to_host(slot).item()) == ref_norm))

    # dhopm3 across the group: bit-identical to the in-process run of the
    # same split (the reference's threads-as-ranks model) and within
    # tolerance of the oracle
    hshape = (world * 4, 10, 9)
    vals = np.random.default_rng(7).standard_normal(hshape)
    for name, s in (("f64", 0), ("f64", 2), ("f32", 1), ("bf16f32", 0), ("f16f32", 0), ("f32f64", 1)):
        mode = tv.MODES[name]
        A = tv.Tensor.from_array(vals, mode)
        if tv.make_split_plan(hshape[s], s, world).p_eff != world:
            continue
        x0 = O.initial_vectors(hshape, name)
        res = tv.dhopm3(tv.distribute(A, s, world, group=group), [v.copy() for v in x0], sweeps=3)
        inproc = tv.dhopm3(tv.distribute(A, s, world), [v.copy() for v in x0], sweeps=3)
        vecs, norms = _memo(("hopm", world, name, s),
                            lambda: O.dhopm3(A.to_numpy().reshape(hshape), s, world, x0, 3, name))
        tol = {"f64": 1e-11, "f32": 1e-4, "f32f64": 1e-5, "bf16f32": 5e-2, "f16f32": 5e-3}[name]
        close = all(np.allclose(O.promote(a, name), O.promote(b, name), rtol=tol, atol=tol)
                    for a, b in zip(res.vectors, vecs))
        ok.append((name, "hopm-oracle", s, bool(close and np.allclose(res.norms, norms, rtol=tol))))
        ok.append((name, "hopm-inprocess", s, all(_same(a, b) for a, b in zip(res.vectors, inproc.vectors))
                   and res.norms == inproc.norms))
    return ok


def as_i(t: torch.Tensor) -> torch.Tensor:
    return t.view(torch.int16) if t.dtype in (torch.uint16, torch.float16, torch.bfloat16) else \
        t.view(torch.int32) if t.element_size() == 4 else t.view(torch.int64)
