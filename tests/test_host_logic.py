"""CPU-only checks of the host side: mode table, shapes and split plans,
schedule and traffic model (against the reference's recorded counts), counters,
the WorkerGroup rendezvous, and the C-ABI library's exports and argument
validation (no kernel launches)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, load_golden
import paper_2501_03121_b200 as tv
from paper_2501_03121_b200 import _lib, build


def test_mode_table():
    assert sorted(tv.MODES) == ["bf16f32", "f16f32", "f32", "f32f64", "f64"]
    assert tv.BF16F32.storage_bytes == 2 and tv.BF16F32.compute_bytes == 4 and tv.BF16F32.mixed
    assert tv.F32F64.mixed and not tv.F64.mixed
    assert tv.BF16F32.storage_dtype == np.uint16
    with pytest.raises(tv.ModeError):
        tv.parse_mode("f8")


def test_shapes_and_views():
    s = tv.Shape((2, 3, 4))
    assert s.order == 3 and s.size == 24 and str(s) == "2x3x4"
    assert s.drop(1).extents == (2, 4) and tv.Shape((5,)).drop(0).extents == (1,)
    assert tv.parse_shape("979^3").extents == (979,) * 3
    assert tv.parse_shape("2,3,4") == s and tv.parse_shape("2x3x4") == s
    md = tv.matricize_dims(s, 1)
    assert (md.u, md.nk, md.v) == (2, 3, 4)
    assert tv.linear_index(s, (1, 2, 3)) == 23
    with pytest.raises(IndexError):
        tv.matricize_dims(s, 3)
    with pytest.raises(ValueError):
        tv.Shape(())


def test_division_rule():
    assert tv.optimal_division(4, 3, 8) == (2, 2)
    assert tv.optimal_division(96, 8, 8) == (16, 6)  # the vl=8 trap on C3
    assert tv.optimal_division(96, 8, 1) == (12, 8)
    rng = np.random.default_rng(41)
    for _ in range(500):
        n, p, vl = int(rng.integers(1, 2000)), int(rng.integers(1, 64)), int(2 ** rng.integers(0, 6))
        q, pe = tv.optimal_division(n, p, vl)
        assert 1 <= pe <= p and q * pe >= n > q * (pe - 1)
        if n >= vl:
            assert q == n or q % vl == 0
    plan = tv.make_split_plan(10, 1, 4)
    assert plan.ranges == ((0, 3), (3, 6), (6, 9), (9, 10)) and plan.extent == 10


def test_task_ranges_and_counters():
    for total in (1, 5, 8, 17):
        for tasks in (1, 2, 3, 8, 30):
            hits = np.zeros(total, dtype=int)
            for a, b in tv.task_ranges(total, tasks):
                hits[a:b] += 1
            assert np.all(hits == 1)
    kc = tv.KernelCounters()
    kc.count("tvc", 68, 16, 8)
    other = tv.KernelCounters()
    other.count("tvc", 4, 4, 2)
    kc.add(other)
    assert kc.elements_touched == 92 and kc.bytes_touched == 84 * 8 + 16 and kc.invocations == {"tvc": 2}


def test_schedule_counts():
    for d in range(2, 11):
        assert tv.tvc_per_sweep(d, True) == (d - 1) * (d + 2) // 2
        assert tv.tvc_per_sweep(d, False) == d * (d - 1)
    assert tv.iteration_plan(5, 3, True) == (frozenset({0, 1}), [2, 4])
    assert tv.mode_remap(2, {0, 1}) == 0 and tv.mode_remap(3, {1}) == 2
    with pytest.raises(ValueError):
        tv.mode_remap(1, {1})


def test_simulation_matches_reference_runs():
    """iteration_touched recorded from the reference's dhopm3 equals the traffic
    model restated in schedule.py (the roofline numerator of bench.py)."""
    g = load_golden("hopm")
    for c in range(int(g["n"])):
        meta = [int(e) for e in g[f"c{c}_meta"]]
        d = meta[0]
        shape = tuple(meta[1:1 + d])
        s, p, sweeps = meta[1 + d:4 + d]
        sim = tv.simulate_hopm(shape, s, p, reuse=True)
        touched = g[f"c{c}_touched"].tolist()
        for r in range(len(sim)):
            assert touched[r] == sim[r].iteration_touched * sweeps
        assert int(g[f"c{c}_tvc_count"]) == sim[0].tvc_count * sweeps


def test_baseline_traffic_figures():
    # 384^4 fp64 p=8 s=3 -> 43,770,757,632 B per rank per sweep
    assert tv.schedule.sweep_bytes((384,) * 4, 3, 8, 8)[0] == 43_770_757_632
    assert sum(tv.schedule.sweep_bytes((384,) * 4, 3, 1, 8)) == 350_165_609_472


def test_ring_chunks():
    assert tv.ring_chunks(10, 3) == [(0, 4), (4, 8), (8, 10)]
    assert tv.ring_chunks(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    assert tv.ring_chunks(0, 3) == [(0, 0)] * 3


def test_worker_group_rendezvous_errors():
    g = tv.WorkerGroup(3, timeout=0.5)

    def body(rank):
        if rank != 2:
            g.barrier(rank)
        return rank

    with pytest.raises(tv.CollectiveTimeout) as info:
        g.run(body)
    assert info.value.absent == [2]

    g = tv.WorkerGroup(2, timeout=2.0)

    def mismatch(rank):
        if rank == 0:
            g.barrier(rank)
        else:
            g.all_gather(rank, None)

    with pytest.raises(tv.CollectiveError):
        g.run(mismatch)

    g = tv.WorkerGroup(2, timeout=0.5)

    def failing(rank):
        if rank == 1:
            raise ValueError("boom")
        g.barrier(rank)

    with pytest.raises(ValueError):
        g.run(failing)
    with pytest.raises(ValueError):
        tv.WorkerGroup(0)


def _header_symbols() -> set[str]:
    text = (ROOT / "include" / "tenvec_b200.h").read_text()
    return set(re.findall(r"^\s*(?:const char\*|int64_t|unsigned long long|int)\s+(tv_\w+)\s*\(", text, flags=re.M))


def test_library_builds_loads_and_exports_every_header_symbol():
    build.build()
    lib = _lib.load()
    declared = _header_symbols()
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.tv_version().startswith(b"tenvec_b200")


def test_library_argument_validation_without_gpu():
    lib = _lib.load()
    # nk = 0 and bad modes are rejected before any launch
    assert lib.tv_tvc(None, 0, 0, 4, 0, 4, None, 1.0, 0.0, None, None) == 1
    assert b"nk" in lib.tv_last_error()
    assert lib.tv_tvc_regime(None, 0, 4, 0, 4) == -1
    assert lib.tv_getvc(2, None, 0, 0, 2, 2, 2, None, 1.0, 0.0, None, None) == 1
    assert lib.tv_getvc(0, None, 0, 0, 2, 3, 2, None, 1.0, 0.0, None, None) == 1
    assert lib.tv_convert(None, 0, None, 1, -1, None) == 1
    assert lib.tv_rank_fold(None, 0, 4, 0, 0, 0, 0, 0, None, None) == 4
    ext = (ctypes.c_int64 * 3)(2, 3, 4)
    assert lib.tv_fill(None, 0, 0, 1, ext, 3, 1, 2, 1, None) == 1
    # regime choice is host logic: aligned fake pointers, no dereference
    p = 1 << 20
    assert lib.tv_tvc_regime(p, 1, 1000, 256, 1) == 1      # rows
    assert lib.tv_tvc_regime(p, 1, 1000, 96, 1) == 8       # aligned rows <= 512 B -> staged
    assert lib.tv_tvc_regime(p, 1, 1, 12, 1) == 10         # one 3-vector row -> flat rows
    assert lib.tv_tvc_regime(p, 1, 1000, 160, 1) == 1      # aligned longer rows stay rows
    assert lib.tv_tvc_regime(p, 1, 1, 2048, 4096) == 3     # columns
    assert lib.tv_tvc_regime(p, 1, 1000, 96, 12) == 8      # small aligned 3-vector slabs -> staged
    assert lib.tv_tvc_regime(p, 1, 1000, 4000, 12) == 4    # larger ones -> slabs
    assert lib.tv_tvc_regime(p, 1, 1000, 13, 1) == 8       # unaligned short rows -> staged
    assert lib.tv_tvc_regime(p, 0, 1000, 13, 13) == 8      # unaligned small slabs -> staged
    assert lib.tv_tvc_regime(p, 1, 1000, 200, 48) == 9     # width 12 vectors -> flat
    assert lib.tv_tvc_regime(p, 1, 1000, 200, 20) == 8     # width 5, fits a tile -> staged
    assert lib.tv_tvc_regime(p, 1, 1000, 4000, 20) == 4    # width 5 -> slabs
    assert lib.tv_tvc_regime(p + 4, 1, 1000, 96, 12) == 7  # misaligned -> scalar slabs
    assert lib.tv_tvc_regime(p, 0, 1000, 13, 1) == 8       # odd fp64 rows -> staged
    assert lib.tv_tvc_regime(p, 0, 1000, 131, 1) == 8      # odd fp64 rows <= 2 KB -> staged
    assert lib.tv_tvc_regime(p, 0, 1000, 301, 1) == 5      # odd fp64 long rows -> scalar rows
    assert lib.tv_tvc_regime(p, 0, 9, 979, 979) == 6       # odd fp64 columns -> scalar columns
    assert lib.tv_tvc_regime(p, 0, 130321, 19, 361) == 11  # many 55 KB unaligned slabs -> row-run tiles
    assert lib.tv_tvc_regime(p, 0, 30625, 175, 175) == 11  # 175-column slabs: two row groups
    assert lib.tv_tvc_regime(p, 0, 30625, 175, 97) == 6    # narrower -> scalar columns
    assert lib.tv_tvc_regime(p, 0, 100000, 10, 1000) == 11  # aligned short columns -> row-run tiles
    assert lib.tv_tvc_regime(p, 0, 2048, 2048, 4096) == 3  # aligned long columns stay COLS
    assert lib.tv_tvc_regime(p, 0, 979, 979, 979) == 6     # too few slabs to balance -> scalar columns
    assert lib.tv_tvc_regime(p, 3, 8, 1000000, 12) == 13   # tall unaligned bf16 slabs -> row tiles
    assert lib.tv_tvc_regime(p, 1, 8, 1000000, 12) == 4    # the same in fp32 (aligned) -> slabs
    assert lib.tv_tvc_regime(p, 0, 1, 3000001, 7) == 13    # tall unaligned fp64 -> row tiles
    # the diagnostic override pins a regime only where the view can take it
    prev = lib.tv_set_regime_override(1)
    try:
        assert lib.tv_tvc_regime(p, 1, 1000, 96, 1) == 1       # rows forced
        assert lib.tv_tvc_regime(p, 1, 1000, 13, 1) == 8       # rows invalid (unaligned)
    finally:
        lib.tv_set_regime_override(prev)
    assert lib.tv_tvc_regime(p, 1, 1000, 96, 1) == 8


def test_distributed_cabi_validates_arguments_without_gpu():
    """The distributed C-ABI rejects bad calls before touching a device or
    NCCL (include/tenvec_b200.h): null plans / communicators, bad modes and
    splits, bad repack geometry; destroying NULL is a no-op."""
    lib = _lib.load()
    plan = ctypes.c_void_p()
    ext = (ctypes.c_int64 * 3)(4, 5, 6)
    assert lib.tv_dhopm3_plan_create(None, None, 0, 0, 3, ext, 0, ctypes.byref(plan)) == 1
    assert lib.tv_dhopm3_plan_create(None, 1 << 20, 0, 0, 3, ext, 3, ctypes.byref(plan)) == 1  # s out of range
    assert lib.tv_dhopm3_plan_create(None, 1 << 20, 2, 2, 3, ext, 0, ctypes.byref(plan)) == 2  # f16 compute
    assert lib.tv_dhopm3_sweep(None, None, None, None, None) == 1
    assert lib.tv_dhopm3_plan_destroy(None) == 0 and lib.tv_comm_destroy(None) == 0
    assert lib.tv_allreduce(None, None, 8, 0, 0, 1, None, 0, None) == 4
    assert lib.tv_allreduce_workspace_bytes(None, 8, 0, 1) == -1
    assert lib.tv_allgather(None, None, None, None, 8, None) == 4
    assert lib.tv_comm_rank_size(None, None, None) == 4
    assert lib.tv_comm_init_rank(None, 2, 0, ctypes.byref(plan)) == 4
    srcs = (ctypes.c_void_p * 2)(1 << 20, 1 << 21)
    assert lib.tv_repack(srcs, 2, 1, 10, 1, 0, 8, 1 << 22, None) == 1     # chunk q = 0
    assert lib.tv_repack(srcs, 2, 1, 10, 1, 5, 3, 1 << 22, None) == 1     # 3-byte elements
    assert lib.tv_repack(srcs, 2, 0, 10, 1, 5, 8, None, None) == 0       # empty: nothing to do
    bases = (ctypes.c_void_p * 2)(1 << 20, 1 << 21)
    assert lib.tv_peer_barrier(bases, 2, 2, 1, 0, None, None) == 4         # rank out of range
    assert lib.tv_launch_count() >= 0


def test_no_oracle_import_in_product():
    pkg = ROOT / "paper_2501_03121_b200"
    for f in pkg.rglob("*.py"):
        text = f.read_text()
        assert "tenvec_oracle" not in text and "oracle/" not in text, f


class _FakeTransport:
    size, rank, backend, store = 2, 0, "fake", None


def test_rank_group_validates_knobs_up_front(monkeypatch):
    """A malformed TENVEC_B200_OWNER_LANES / timeout fails at construction,
    before any barrier could be enqueued (comm.py _owner_streams)."""
    from paper_2501_03121_b200 import RankGroup
    from paper_2501_03121_b200.errors import CollectiveError

    monkeypatch.setenv("TENVEC_B200_OWNER_LANES", "two")
    with pytest.raises(CollectiveError):
        RankGroup(transport=_FakeTransport())
    monkeypatch.setenv("TENVEC_B200_OWNER_LANES", "0")
    with pytest.raises(CollectiveError):
        RankGroup(transport=_FakeTransport())
    monkeypatch.setenv("TENVEC_B200_OWNER_LANES", "3")
    g = RankGroup(transport=_FakeTransport(), timeout=5)
    assert g.lanes == 3 and g.size == 2 and g.timeout == 5.0
    with pytest.raises(CollectiveError):
        RankGroup(transport=_FakeTransport(), timeout=0)
    with pytest.raises(CollectiveError):
        RankGroup(transport=_FakeTransport(), algo="ring")


def _reference_tensor_module():
    """The reference's tensor.py (tensor.py:25-144 is the geometry), from the
    installed baseline/_ref or the read-only source tree; None when neither
    is here (the GPU box has neither)."""
    import importlib
    import sys

    for path in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (path / "tenvec" / "tensor.py").exists():
            sys.path.insert(0, str(path))
            try:
                return importlib.import_module("tenvec.tensor")
            except Exception:  # noqa: BLE001
                return None
            finally:
                sys.path.remove(str(path))
    return None


def test_geometry_matches_the_reference_package():
    """geometry.py restates the reference's integer geometry: the same drop,
    block view, linear index, division rule and split ranges on random
    shapes (hypothesis), compared with the reference module itself."""
    from hypothesis import given, settings
    from hypothesis import strategies as st

    RT = _reference_tensor_module()
    if RT is None:
        pytest.skip("the reference package is not in this container")

    @settings(max_examples=300, deadline=None)
    @given(st.lists(st.integers(1, 9), min_size=1, max_size=6), st.data())
    def check(ext, data):
        k = data.draw(st.integers(0, len(ext) - 1))
        ours, ref = tv.Shape(tuple(ext)), RT.Shape(tuple(ext))
        assert ours.size == ref.size and ours.order == ref.order
        assert ours.drop(k).extents == tuple(ref.drop(k).extents)
        md, rmd = tv.matricize_dims(ours, k), RT.matricize_dims(ref, k)
        assert (md.u, md.nk, md.v) == (rmd.u, rmd.nk, rmd.v)
        idx = tuple(data.draw(st.integers(0, n - 1)) for n in ext)
        assert tv.linear_index(ours, idx) == RT.linear_index(ref, idx)
        p = data.draw(st.integers(1, 12))
        vl = data.draw(st.sampled_from([1, 2, 4, 8]))
        assert tv.optimal_division(ext[k], p, vl) == tuple(RT.optimal_division(ext[k], p, vl))
        ours_plan, ref_plan = tv.make_split_plan(ext[k], k, p, vl), RT.make_split_plan(ext[k], k, p, vl)
        assert ours_plan.p_eff == ref_plan.p_eff and ours_plan.chunk == ref_plan.chunk
        assert [tuple(r) for r in ours_plan.ranges] == [tuple(r) for r in ref_plan.ranges]
        text = "x".join(map(str, ext))
        assert tv.parse_shape(text).extents == tuple(RT.parse_shape(text).extents)

    check()


def _fold_range_host(slots, p, n, ring_chunk, offset, mode, mixed, O):
    """numpy restatement of tv_rank_fold_range: element e of the range is
    global index offset + e; the mixed ring starts it at rank
    ((offset + e) // ring_chunk) % p (include/tenvec_b200.h)."""
    out = np.empty(n, dtype=slots[0].dtype)
    for e in range(n):
        r0 = ((offset + e) // ring_chunk) % p if mixed else 0
        cur = slots[r0][e]
        for i in range(1, p):
            b = slots[(r0 + i) % p][e]
            cur = O.demote(O.promote(np.array([cur]), mode) + O.promote(np.array([b]), mode), mode)[0] \
                if mixed or O.MODES[mode][2] or O.MODES[mode][0] != O.MODES[mode][1] else cur + b
        out[e] = cur
    return out


@pytest.mark.parametrize("p", [2, 3, 4, 5])
def test_fused_plan_index_math_on_host(oracle, p):
    """RankGroup's fused split-mode reduction, its index math restated on
    the host (fused_plan's owner ranges and slots, the owner fold over its
    range, the select over the owners): every rank's partial sums -- the
    oracle's -- reduce to exactly the reference's exact / mixed ring result,
    for slab owners (u >= p, ragged and empty last owners) and column owners
    (u == 1)."""
    from paper_2501_03121_b200.comm import fused_plan

    O = oracle
    rng = np.random.default_rng(p)
    for u, v in ((p * 3 + 1, 5), (p, 7), (p + 2, 1), (1, 13 * p + 3), (1, p)):
        plan = fused_plan(u, v, p, 8)
        assert plan is not None
        n = u * v
        for mode in ("f64", "bf16f32", "f16f32"):
            mixed = O.is_mixed(mode)
            partials = [O.demote(rng.uniform(-4, 4, n), mode) for _ in range(p)]
            want = O.fold_mixed([q.copy() for q in partials], mode) if mixed else O.fold_exact(partials)
            folded = []
            for c in range(p):
                lo, hi = plan.bounds[c]
                a, b = lo * plan.unit, hi * plan.unit
                assert b - a == plan.sizes[c]
                slots = [q[a:b] for q in partials]  # rank r's owner-c range, as it lands in slot r
                folded.append(_fold_range_host(slots, p, b - a, plan.ring_chunk, c * plan.chunk, mode, mixed, O))
            got = np.concatenate(folded)  # tv_rank_select: chunk c from owner c
            assert np.array_equal(got.view(np.uint8), np.asarray(want).view(np.uint8)), (u, v, mode)
