"""One process per GPU over NCCL (RankGroup): dtvc with the split on and off the
contraction mode, and dhopm3, against the oracle.  Needs >= 2 visible GPUs
(skipped otherwise; run with `gpurun --gpus 2|4`)."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def _worker(rank, world, port, q):
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import torch.distributed as dist

    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    ok = []
    try:
        import tenvec_oracle as O
        import paper_2501_03121_b200 as tv

        group = tv.RankGroup(algo="exact")
        # dtvc on a device-generated 5-mode tensor: every k, split on / off k
        shape = (6, 8, world * 3, 5, 4)
        full = O.fill_values(shape, "hash", seed=4).reshape(shape)
        for name in ("f64", "f32", "f32f64", "bf16f32", "f16f32"):
            mode = tv.MODES[name]
            host = O.demote(full.reshape(-1), name).reshape(shape)
            for s in sorted({2} | ({4} if tv.make_split_plan(4, 4, world).p_eff == world else set())):
                dt = tv.distribute_generated(tv.Shape(shape), s, world, mode, fill="hash", seed=4, group=group)
                parts, ranges = O.split(host, s, world)
                xs = [O.demote((np.arange(shape[k]) % 5) + 1.0, name).copy() for k in range(5)]
                sweep = tv.dtvc_sweep(dt, xs)
                for k in range(5):
                    x = xs[k]
                    res = tv.dtvc(dt, x, k)
                    kind, outs, s2 = O.dtvc(parts, ranges, s, x, k, name)
                    want = outs[0] if k == s else outs[rank]
                    for tag, r in (("dtvc", res), ("sweep", sweep[k])):
                        got = (r.parts[0] if k == s else r.parts[rank]).to_numpy()
                        ok.append((name, s, k, tag, bool(np.array_equal(_bits(got), _bits(want.reshape(-1))))))
        # a reduction above the small-gather threshold: all-to-all + fold + all-gather
        big = (64, 64, 2 * world, 64)
        fullb = O.fill_values(big, "hash", seed=6).reshape(big)
        p2p = tv.RankGroup(algo="p2p")  # the same fold over symmetric (peer) memory
        for name in ("f32", "bf16f32", "f64"):
            mode = tv.MODES[name]
            hostb = O.demote(fullb.reshape(-1), name).reshape(big)
            x = O.demote((np.arange(big[2]) % 3) + 1.0, name).copy()
            parts, ranges = O.split(hostb, 2, world)
            _, outs, _ = O.dtvc(parts, ranges, 2, x, 2, name)
            for tag, grp in (("exact", group), ("p2p", p2p)):
                dt = tv.distribute_generated(tv.Shape(big), 2, world, mode, fill="hash", seed=6, group=grp)
                for _ in range(2):  # twice: the symmetric buffer is reused
                    got = tv.dtvc(dt, x, 2).parts[0].to_numpy()
                ok.append((name, "big-reduce", tag, bool(np.array_equal(_bits(got), _bits(outs[0].reshape(-1))))))
        # ragged reduction (n not a multiple of p or of 16 bytes) over peer memory
        rag = torch.arange(1, 300_003, dtype=torch.float32, device="cuda") * (rank + 1)
        want = torch.arange(1, 300_003, dtype=torch.float32) * sum(r + 1 for r in range(world))
        p2p.all_reduce_sum(rank, rag)
        ok.append(("f32", "ragged-p2p", 0, bool(torch.equal(rag.cpu(), want))))
        # the split-mode contraction fused with its reduction over peer memory
        # (algo="fused"): slab-range owners (u >= p), column-range owners
        # (u == 1, unaligned columns), the fallback (1 < u < p), every mode
        fused = tv.RankGroup(algo="fused")
        for fshape, s in (((5, 6, world * 3, 7), 2), ((world * 4, 30, 7), 0), ((3, world * 2, 50), 1),
                          ((2, world * 3, 40), 1)):
            fullf = O.fill_values(fshape, "hash", seed=8).reshape(fshape)
            for name in ("f64", "f32", "f32f64", "bf16f32", "f16f32"):
                mode = tv.MODES[name]
                hostf = O.demote(fullf.reshape(-1), name).reshape(fshape)
                x = O.demote((np.arange(fshape[s]) % 7) + 1.0, name).copy()
                parts, ranges = O.split(hostf, s, world)
                _, outs, _ = O.dtvc(parts, ranges, s, x, s, name)
                dt = tv.distribute_generated(tv.Shape(fshape), s, world, mode, fill="hash", seed=8, group=fused)
                for _ in range(2):  # twice: the symmetric slots are reused
                    got = tv.dtvc(dt, x, s).parts[0].to_numpy()
                ok.append((name, "fused", fshape, bool(np.array_equal(_bits(got), _bits(outs[0].reshape(-1))))))
                sweep = tv.dtvc_sweep(dt, [O.demote(np.ones(n), name).copy() for n in fshape])
                ok.append((name, "fused-sweep", fshape, sweep[s].parts[0].size == outs[0].size))
        # on-device assembly over NCCL: disjoint results gathered and repacked,
        # deferred partial sums gathered and folded (undistribute, hopm.py:76-84)
        ashape = (5, world * 3, 4, 6)
        fulla = O.fill_values(ashape, "hash", seed=9).reshape(ashape)
        for name in ("f64", "f32", "bf16f32"):
            mode = tv.MODES[name]
            hosta = O.demote(fulla.reshape(-1), name).reshape(ashape)
            dt = tv.distribute_generated(tv.Shape(ashape), 1, world, mode, fill="hash", seed=9, group=group)
            whole = tv.undistribute(dt).to_numpy()
            ok.append((name, "assemble-input", 0, bool(np.array_equal(_bits(whole), _bits(hosta.reshape(-1))))))
            for k in (0, 3):
                x = O.demote((np.arange(ashape[k]) % 4) + 1.0, name).copy()
                got = tv.undistribute(tv.dtvc(dt, x, k)).to_numpy()
                want = O.tvc(hosta.reshape(-1), ashape, x, k, name)
                ok.append((name, "assemble", k, bool(np.array_equal(_bits(got), _bits(want)))))
            x = O.demote((np.arange(ashape[1]) % 4) + 1.0, name).copy()
            got = tv.undistribute(tv.dtvc(dt, x, 1, defer=True)).to_numpy()
            want = O.tvc(hosta.reshape(-1), ashape, x, 1, name)
            ok.append((name, "assemble-partial", 1,
                       bool(np.allclose(O.promote(got, name), O.promote(want, name), rtol=1e-2 if name == "bf16f32" else 1e-6))))
        # the dHOPM3 reduction with the normalisation in the fold's epilogue:
        # the same bits as all_reduce_sum + normalize
        for name in ("f64", "f32", "f32f64", "bf16f32", "f16f32"):
            mode = tv.MODES[name]
            for n in (384, 4096, 1001):
                v = torch.from_numpy(O.demote(np.random.default_rng(rank + n).standard_normal(n), name).copy())
                v = v.cuda() if v.dtype != torch.uint16 else v.view(torch.int16).cuda().view(torch.uint16)
                ref = v.clone()
                group.all_reduce_sum_mixed(rank, ref, mode) if mode.mixed else group.all_reduce_sum(rank, ref)
                ref_norm = tv.normalize(ref, mode=mode)
                dst = torch.empty_like(v)
                slot = torch.empty(1, dtype=torch.float64, device="cuda")
                cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
                okf = group.all_reduce_normalize(rank, v, mode, dst, slot, None, cnt)
                same = bool(torch.equal(dst.view(torch.uint8) if dst.dtype != torch.uint16 else dst.view(torch.int16),
                                        ref.view(torch.uint8) if ref.dtype != torch.uint16 else ref.view(torch.int16)))
                ok.append((name, "fold-normalize", n, okf and same and float(slot.item()) == ref_norm))
        # dhopm3 over NCCL equals the in-process oracle run
        hshape = (world * 4, 10, 9)
        vals = np.random.default_rng(7).standard_normal(hshape)
        for name, s in (("f64", 0), ("f64", 2), ("f32", 1), ("bf16f32", 0)):
            mode = tv.MODES[name]
            A = tv.Tensor.from_array(vals, mode)
            if tv.make_split_plan(hshape[s], s, world).p_eff != world:
                continue
            dt = tv.distribute(A, s, world, group=group)
            x0 = O.initial_vectors(hshape, name)
            res = tv.dhopm3(dt, [v.copy() for v in x0], sweeps=3)
            vecs, norms = O.dhopm3(A.to_numpy().reshape(hshape), s, world, x0, 3, name)
            tol = {"f64": 1e-11, "f32": 1e-4, "bf16f32": 5e-2}[name]
            same = all(np.allclose(O.promote(a, name), O.promote(b, name), rtol=tol, atol=tol)
                       for a, b in zip(res.vectors, vecs))
            ok.append((name, "hopm", s, bool(same and np.allclose(res.norms, norms, rtol=tol))))
        q.put((rank, ok))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, [("error", repr(exc)[:500], 0, False)]))
    finally:
        dist.destroy_process_group()


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
        r, res = q.get(timeout=600)
        results[r] = res
    for p in procs:
        p.join(timeout=120)
    for r, res in results.items():
        bad = [c for c in res if not c[-1]]
        assert not bad, (r, bad)
