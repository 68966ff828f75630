"""Bounds checks without compute-sanitizer (closed on this pool): every
buffer a kernel touches is placed against an UNMAPPED guard page, so one
16-byte vector read or written past the end (``--align end``) or before the
start (``--align start``) of any input, output or workspace faults the
launch (illegal address) instead of silently touching a neighbour.

Run as a subprocess (a fault is sticky for the process):
    python tests/guarded_run.py --align end|start [--quick]
prints one line per case and exits 0 when every case ran and matched; on a
fault the last "case ..." line names the culprit.  Results are compared with
the oracle (integer data, bitwise) or with the same call on ordinary torch
memory (bitwise).  Test infrastructure: driven by tests/test_gpu_guards.py.
"""

from __future__ import annotations

import argparse
import ctypes
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

import tenvec_oracle as O  # noqa: E402

import paper_2501_03121_b200 as tv  # noqa: E402
from paper_2501_03121_b200 import _lib  # noqa: E402

from cuda.bindings import driver as drv  # noqa: E402


def _ok(res):
    err = res[0] if isinstance(res, tuple) else res
    if err != drv.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"driver call failed: {err}")
    return res[1] if isinstance(res, tuple) and len(res) == 2 else res


class Guarded:
    """nbytes of device memory flush against an unmapped page."""

    def __init__(self, nbytes: int, align: str):
        dev = torch.cuda.current_device()
        prop = drv.CUmemAllocationProp()
        prop.type = drv.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        prop.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        prop.location.id = dev
        gran = int(_ok(drv.cuMemGetAllocationGranularity(
            prop, drv.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM)))
        self.nbytes = max(int(nbytes), 1)
        self.size = -(-self.nbytes // gran) * gran
        self.gran = gran
        self.base = int(_ok(drv.cuMemAddressReserve(self.size + 2 * gran, 0, 0, 0)))
        self.handle = _ok(drv.cuMemCreate(self.size, prop, 0))
        _ok(drv.cuMemMap(self.base + gran, self.size, 0, self.handle, 0))
        acc = drv.CUmemAccessDesc()
        acc.location = prop.location
        acc.flags = drv.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        _ok(drv.cuMemSetAccess(self.base + gran, self.size, [acc], 1))
        lo = self.base + gran
        # end: the data ends where the mapping ends (16-byte aligned start, so
        # the aligned kernel forms run; slack < 16 bytes); start: it begins
        # at the mapping's first byte
        self.ptr = lo + self.size - (-(-self.nbytes // 16) * 16) if align == "end" else lo

    def upload(self, arr: np.ndarray) -> "Guarded":
        b = np.ascontiguousarray(arr).view(np.uint8)
        _ok(drv.cuMemcpyHtoD(self.ptr, b.ctypes.data, b.nbytes))
        return self

    def download(self, dtype, count: int) -> np.ndarray:
        out = np.empty(count, dtype=dtype)
        _ok(drv.cuMemcpyDtoH(out.ctypes.data, self.ptr, out.nbytes))
        return out

    def free(self):
        _ok(drv.cuMemUnmap(self.base + self.gran, self.size))
        _ok(drv.cuMemRelease(self.handle))
        _ok(drv.cuMemAddressFree(self.base, self.size + 2 * self.gran))


def _np_storage(name):
    return O.MODES[name][0]


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


class Runner:
    def __init__(self, align: str):
        self.align = align
        self.lib = _lib.load()
        self.cases = 0
        self.bad: list = []
        self.bufs: list[Guarded] = []

    def g(self, arr=None, nbytes=None) -> Guarded:
        b = Guarded(arr.nbytes if arr is not None else nbytes, self.align)
        if arr is not None:
            b.upload(arr)
        self.bufs.append(b)
        return b

    def done(self, what, ok):
        torch.cuda.synchronize()
        for b in self.bufs:
            b.free()
        self.bufs.clear()
        self.cases += 1
        if not ok:
            self.bad.append(what)
        print(("ok  " if ok else "BAD ") + str(what), flush=True)

    # -- tv_tvc_ws on the (u, nk, v) view with a pinned regime ---------------
    def tvc(self, shape, k, name, regime=None, alpha=1.0, ints=(1, 98)):
        print("case tvc", shape, k, name, regime, flush=True)
        mode = tv.MODES[name]
        rng = np.random.default_rng(hash((shape, k, name)) % 2**32)
        vals = O.demote(rng.integers(*ints, shape).astype(np.float64).reshape(-1), name)
        x = O.demote(rng.integers(1, 3, shape[k]).astype(np.float64), name)
        u, nk, v = math.prod(shape[:k]), shape[k], math.prod(shape[k + 1:])
        A, X = self.g(vals), self.g(x)
        Y = self.g(nbytes=u * v * vals.itemsize)
        codes = {n: c for c, n in _lib.REGIMES.items()}
        prev = self.lib.tv_set_regime_override(codes[regime] if regime else -1)
        try:
            need = self.lib.tv_tvc_workspace_bytes(A.ptr, mode.tv_storage, mode.tv_compute, u, nk, v)
            W = self.g(nbytes=need) if need > 0 else None
            _lib.check(self.lib.tv_tvc_ws(A.ptr, mode.tv_storage, mode.tv_compute, u, nk, v, X.ptr, alpha, 0.0,
                                          Y.ptr, W.ptr if W else None, need, _lib.stream_ptr()), "tvc")
            torch.cuda.synchronize()
        finally:
            self.lib.tv_set_regime_override(prev)
        got = Y.download(vals.dtype, u * v)
        want = O.tvc(vals, shape, x, k, name, alpha=alpha)
        self.done(("tvc", shape, k, name, regime), np.array_equal(_bits(got), _bits(want)))

    def sweep(self, shape, name):
        print("case sweep", shape, name, flush=True)
        mode = tv.MODES[name]
        rng = np.random.default_rng(sum(shape))
        vals = O.demote(rng.integers(1, 98, shape).astype(np.float64).reshape(-1), name)
        xs = [O.demote(rng.integers(1, 3, n).astype(np.float64), name) for n in shape]
        A = self.g(vals)
        X = [self.g(x) for x in xs]
        n = vals.size
        Y = [self.g(nbytes=n // e * vals.itemsize) for e in shape]
        d = len(shape)
        ext = (ctypes.c_int64 * d)(*shape)
        need = self.lib.tv_tvc_sweep_workspace_bytes(A.ptr, mode.tv_storage, mode.tv_compute, d, ext)
        W = self.g(nbytes=need) if need > 0 else None
        _lib.check(self.lib.tv_tvc_sweep(A.ptr, mode.tv_storage, mode.tv_compute, d, ext,
                                         (ctypes.c_void_p * d)(*[b.ptr for b in X]),
                                         (ctypes.c_void_p * d)(*[b.ptr for b in Y]),
                                         W.ptr if W else None, need, _lib.stream_ptr()), "sweep")
        torch.cuda.synchronize()
        ok = all(np.array_equal(_bits(Y[k].download(vals.dtype, n // shape[k])),
                                _bits(O.tvc(vals, shape, xs[k], k, name))) for k in range(d))
        self.done(("sweep", shape, name), ok)

    def getvc(self, trans, m, n, lda, name):
        print("case getvc", trans, m, n, lda, name, flush=True)
        mode = tv.MODES[name]
        rng = np.random.default_rng(m * 7 + n)
        full = rng.integers(1, 4, (m, lda)).astype(np.float64)
        vals = O.demote(full.reshape(-1), name)[: (m - 1) * lda + n]  # the strided window's extent
        xlen = n if trans == 0 else m
        x = O.demote(rng.integers(1, 3, xlen).astype(np.float64), name)
        ylen = m if trans == 0 else n
        A, X, Y = self.g(vals), self.g(x), self.g(nbytes=ylen * vals.itemsize)
        need = self.lib.tv_getvc_workspace_bytes(trans, A.ptr, mode.tv_storage, mode.tv_compute, m, n, lda)
        W = self.g(nbytes=need) if need > 0 else None
        _lib.check(self.lib.tv_getvc_ws(trans, A.ptr, mode.tv_storage, mode.tv_compute, m, n, lda, X.ptr, 1.0, 0.0,
                                        Y.ptr, W.ptr if W else None, need, _lib.stream_ptr()), "getvc")
        torch.cuda.synchronize()
        win = O.promote(O.demote(full.reshape(-1), name), name).astype(np.float64).reshape(m, lda)[:, :n]
        xf = O.promote(x, name).astype(np.float64)
        want = O.demote(win @ xf if trans == 0 else xf @ win, name)
        self.done(("getvc", trans, m, n, lda, name), np.array_equal(_bits(Y.download(vals.dtype, ylen)), _bits(want)))

    # -- the collective and vector kernels: guarded vs ordinary memory ------
    def vector_ops(self, n, name, p=3):
        print("case vector_ops", n, name, p, flush=True)
        mode = tv.MODES[name]
        st, ct, sb = mode.tv_storage, mode.tv_compute, mode.storage_bytes
        rng = np.random.default_rng(n + p)
        srcs = [O.demote(rng.standard_normal(n), name) for _ in range(p)]
        dt = srcs[0].dtype
        lib, sp = self.lib, _lib.stream_ptr()
        results = {}
        for where in ("guarded", "plain"):
            keep = []

            def buf(arr=None, nbytes=None):
                if where == "guarded":
                    return self.g(arr, nbytes).ptr
                t = torch.empty(max(arr.nbytes if arr is not None else nbytes, 1), dtype=torch.uint8, device="cuda")
                if arr is not None:
                    t.copy_(torch.from_numpy(np.ascontiguousarray(arr).view(np.uint8)))
                keep.append(t)
                return t.data_ptr()

            def read(ptr, count, dtype=dt):
                out = np.empty(count, dtype=dtype)
                torch.cuda.synchronize()
                _ok(drv.cuMemcpyDtoH(out.ctypes.data, ptr, out.nbytes))
                return out

            r = {}
            sptrs = [buf(s) for s in srcs]
            arr = (ctypes.c_void_p * p)(*sptrs)
            chunk = -(-n // p)
            for mixed in (0, 1):
                dst = buf(nbytes=n * sb)
                _lib.check(lib.tv_rank_fold(arr, p, n, chunk, 0, st, ct, mixed, dst, sp), "fold")
                r[f"fold{mixed}"] = read(dst, n)
            strided = buf(np.concatenate(srcs))
            dst = buf(nbytes=n * sb)
            _lib.check(lib.tv_rank_fold_strided(strided, n, p, n, chunk, 0, st, ct, 1, dst, sp), "fold_strided")
            r["fold_strided"] = read(dst, n)
            off = n // 3
            dst = buf(nbytes=(n - off) * sb)
            _lib.check(lib.tv_rank_fold_range(strided, n, p, n - off, chunk, off, st, ct, 1, dst, sp), "fold_range")
            r["fold_range"] = read(dst, n - off)
            dst = buf(nbytes=n * sb)
            _lib.check(lib.tv_rank_select(arr, p, n, chunk, st, dst, sp), "select")
            r["select"] = read(dst, n)
            norm, status = buf(nbytes=8), buf(np.zeros(1, np.int32))
            cnt = buf(np.zeros(1, np.uint32))
            dst = buf(nbytes=n * sb)
            _lib.check(lib.tv_rank_fold_normalize(strided, n, p, n, chunk, st, ct, 1, dst, norm, status, cnt, sp),
                       "fold_normalize")
            r["fold_normalize"] = read(dst, n)
            r["fold_normalize_norm"] = read(norm, 1, np.float64)
            _lib.check(lib.tv_norm2(sptrs[0], st, ct, n, norm, sp), "norm2")
            r["norm2"] = read(norm, 1, np.float64)
            xv = buf(srcs[1])
            _lib.check(lib.tv_normalize(xv, st, ct, n, norm, status, sp), "normalize")
            r["normalize"] = read(xv, n)
            y = buf(srcs[2])
            _lib.check(lib.tv_axpby(1.5, sptrs[0], -0.5, y, st, ct, n, sp), "axpby")
            r["axpby"] = read(y, n)
            if name != "f64":
                wide = buf(nbytes=n * 8)
                _lib.check(lib.tv_convert(sptrs[0], st, wide, _lib.TV_F64, n, sp), "convert up")
                r["convert_up"] = read(wide, n, np.float64)
                back = buf(nbytes=n * sb)
                _lib.check(lib.tv_convert(wide, _lib.TV_F64, back, st, n, sp), "convert down")
                r["convert_down"] = read(back, n)
            ext = (ctypes.c_int64 * 3)(7, n, 3)
            fill = buf(nbytes=7 * 2 * 3 * sb) if n >= 3 else None
            if fill:
                _lib.check(lib.tv_fill(fill, st, _lib.TV_FILL_HASH, 5, ext, 3, 1, 1, 3, sp), "fill")
                r["fill"] = read(fill, 7 * 2 * 3)
            torch.cuda.synchronize()
            results[where] = r
            if where == "guarded":
                torch.cuda.synchronize()
                for b in self.bufs:
                    b.free()
                self.bufs.clear()
        ok = all(np.array_equal(_bits(results["guarded"][key]), _bits(results["plain"][key]))
                 for key in results["plain"])
        self.cases += 1
        if not ok:
            self.bad.append(("vector_ops", n, name))
        print(("ok  " if ok else "BAD ") + str(("vector_ops", n, name, p)), flush=True)

    def repack(self, u, ns, v, q, p, eb):
        """tv_repack and tv_repack_part (the interleave assembly kernels) on
        guarded parts and destinations vs plain buffers vs numpy."""
        print("case repack", u, ns, v, q, p, eb, flush=True)
        rng = np.random.default_rng(u * 7 + ns + p)
        exts = [max(0, min(q, ns - r * q)) for r in range(p)]
        parts = [rng.integers(0, 256, u * e * v * eb, dtype=np.uint8) for e in exts]
        want = np.concatenate([pt.reshape(u, e * v * eb) for pt, e in zip(parts, exts)], axis=1).reshape(-1)
        lib, sp = self.lib, _lib.stream_ptr()
        results = {}
        for where in ("guarded", "plain"):
            keep = []

            def buf(arr=None, nbytes=None):
                if where == "guarded":
                    return self.g(arr, nbytes).ptr
                t = torch.empty(max(arr.nbytes if arr is not None else nbytes, 1), dtype=torch.uint8, device="cuda")
                if arr is not None:
                    t.copy_(torch.from_numpy(arr))
                keep.append(t)
                return t.data_ptr()

            def read(ptr, count):
                out = np.empty(count, dtype=np.uint8)
                torch.cuda.synchronize()
                _ok(drv.cuMemcpyDtoH(out.ctypes.data, ptr, out.nbytes))
                return out

            sptrs = [buf(pt) for pt in parts]
            arr = (ctypes.c_void_p * p)(*sptrs)
            dst = buf(nbytes=want.nbytes)
            _lib.check(lib.tv_repack(arr, p, u, ns, v, q, eb, dst, sp), "repack")
            got = read(dst, want.nbytes)
            dst2 = buf(nbytes=want.nbytes)
            for r in range(p):
                if exts[r]:
                    _lib.check(lib.tv_repack_part(sptrs[r], r, p, u, ns, v, q, eb, dst2, sp), "repack_part")
            got2 = read(dst2, want.nbytes)
            # the one-launch push into several joint copies (16-byte units only)
            d3, d4 = buf(nbytes=want.nbytes), buf(nbytes=want.nbytes)
            rb, qb = ns * v * eb, q * v * eb
            for r in range(p):
                eb_r = exts[r] * v * eb
                if exts[r] and (sptrs[r] | d3 | d4 | rb | qb | eb_r) % 16 == 0:
                    dsts = (ctypes.c_void_p * 2)(d3, d4)
                    _lib.check(lib.tv_repack_part_peers(sptrs[r], r, p, u, ns, v, q, eb, dsts, 2, sp), "peers")
                else:
                    for dd in (d3, d4):
                        if exts[r]:
                            _lib.check(lib.tv_repack_part(sptrs[r], r, p, u, ns, v, q, eb, dd, sp), "part")
            got3, got4 = read(d3, want.nbytes), read(d4, want.nbytes)
            results[where] = (got, got2, got3, got4)
            if where == "guarded":
                torch.cuda.synchronize()
                for b in self.bufs:
                    b.free()
                self.bufs.clear()
        ok = all(np.array_equal(results[w][i], want) for w in results for i in range(4))
        self.cases += 1
        if not ok:
            self.bad.append(("repack", u, ns, v, q, p, eb))
        print(("ok  " if ok else "BAD ") + str(("repack", u, ns, v, q, p, eb)), flush=True)

    def tvc_normalize(self, shape, name):
        print("case tvc_normalize", shape, name, flush=True)
        mode = tv.MODES[name]
        rng = np.random.default_rng(sum(shape))
        vals = O.demote(rng.standard_normal(math.prod(shape)), name)
        x = O.demote(rng.standard_normal(shape[1]), name)
        u, nk, v = shape
        got = {}
        for where in ("guarded", "plain"):
            if where == "guarded":
                A, X, Y = self.g(vals).ptr, self.g(x).ptr, self.g(nbytes=u * v * vals.itemsize).ptr
                norm, cnt = self.g(nbytes=8).ptr, self.g(np.zeros(1, np.uint32)).ptr
            else:
                ts = [torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)).cuda() for a in (vals, x)]
                yt = torch.empty(u * v * vals.itemsize, dtype=torch.uint8, device="cuda")
                nt = torch.empty(8, dtype=torch.uint8, device="cuda")
                ct = torch.zeros(4, dtype=torch.uint8, device="cuda")
                A, X, Y, norm, cnt = ts[0].data_ptr(), ts[1].data_ptr(), yt.data_ptr(), nt.data_ptr(), ct.data_ptr()
            _lib.check(self.lib.tv_tvc_normalize(A, mode.tv_storage, mode.tv_compute, u, nk, v, X, Y, norm, None, cnt,
                                                 _lib.stream_ptr()), "tvc_normalize")
            torch.cuda.synchronize()
            out = np.empty(u * v, dtype=vals.dtype)
            _ok(drv.cuMemcpyDtoH(out.ctypes.data, Y, out.nbytes))
            got[where] = out
            if where == "guarded":
                for b in self.bufs:
                    b.free()
                self.bufs.clear()
        self.cases += 1
        ok = np.array_equal(_bits(got["guarded"]), _bits(got["plain"]))
        if not ok:
            self.bad.append(("tvc_normalize", shape, name))
        print(("ok  " if ok else "BAD ") + str(("tvc_normalize", shape, name)), flush=True)


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--align", choices=["end", "start"], default="end")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--control", action="store_true", help="run one deliberate overrun; must fault")
    args = ap.parse_args()
    torch.zeros(1, device="cuda")  # the primary context is current
    _lib.preload()
    from test_gpu_tvc import REGIME_CASES, TALL

    r = Runner(args.align)
    if args.control:
        # positive control: a view one slab longer than its guarded buffer
        # must fault (proves the guard pages are live)
        A = r.g(np.ones(64 * 256, np.float64))
        X = r.g(np.ones(256, np.float64))
        Y = r.g(nbytes=65 * 8)
        off = -64 * 256 * 8 if args.align == "start" else 0
        _lib.check(r.lib.tv_tvc(A.ptr + off, 0, 0, 65, 256, 1, X.ptr, 1.0, 0.0, Y.ptr, _lib.stream_ptr()), "ctl")
        torch.cuda.synchronize()
        print("CONTROL DID NOT FAULT", flush=True)
        return 3
    names = ("f64", "f32", "bf16f32") if args.quick else ("f64", "f32", "f32f64", "f16f32", "bf16f32")
    for shape, k, regime in REGIME_CASES:
        for name in names:
            r.tvc(shape, k, name, regime)
    for shape, k, regime in TALL:
        for name in ("f64", "bf16f32"):
            r.tvc(shape, k, name, None, alpha=2.0, ints=(1, 4))
    for shape in [(7, 9, 11, 13), (256, 256, 256), (3, 4096, 5), (979, 33, 2), (2, 3, 1 << 15)]:
        for name in ("f64", "bf16f32"):
            r.sweep(shape, name)
    for trans, m, n, lda in [(1, 200_000, 8, 12), (0, 1, 3_000_000, 3_000_000), (1, 64, 1000, 1003),
                             (0, 333, 77, 80), (1, 5, 7, 7)]:
        for name in ("f64", "f16f32"):
            r.getvc(trans, m, n, lda, name)
    for n in (1, 7, 384, 4096, 100_003):
        for name in ("f64", "f32", "bf16f32", "f16f32"):
            r.vector_ops(n, name)
    for shape in [(3, 50, 7), (1, 4096, 1), (64, 33, 5)]:
        for name in ("f64", "bf16f32"):
            r.tvc_normalize(shape, name)
    # interleave assembly: 16-byte short runs (thread per unit), unaligned and
    # long runs (warp segments), a short last part
    for u, ns, v, q, p, eb in [(1000, 6, 4, 3, 2, 4), (37, 10, 3, 4, 3, 2), (5, 4096, 1, 1024, 4, 8),
                               (200, 96, 1, 48, 2, 4), (3, 7, 5, 3, 3, 8), (64, 96, 1, 24, 4, 4)]:
        r.repack(u, ns, v, q, p, eb)
    print(f"DONE {r.cases} cases, {len(r.bad)} mismatches: {r.bad}", flush=True)
    return 1 if r.bad else 0


if __name__ == "__main__":
    sys.exit(main())
