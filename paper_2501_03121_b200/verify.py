"""Spot checks of device results against closed forms of the synthetic fills.

The benchmark tensors are generated on the device from their GLOBAL linear
index (tv_fill: ones, ramp = (g mod 97) + 1, hash = splitmix64(seed, g) mod
97 + 1).  Any output element of a contraction of such a tensor with an
integer vector is therefore an exact integer sum that numpy can recompute
from the index alone -- no copy of the tensor, no second implementation of the
kernel.  ``bench.py`` uses this to prove that the timed launches computed the
right values (its ``"parity"`` key); the tests use it at sizes where a full
oracle run would not fit host memory.

This module restates the FILL (a hash of an index), not the algorithm under
test; it never calls the CUDA library.
"""

from __future__ import annotations

import math

import numpy as np

__all__ = ["fill_at", "tvc_expected", "tvc_expected_slab", "sample_outputs", "check_tvc_samples",
           "hopm_last_update_expected"]

_MASK = np.uint64(0xFFFFFFFFFFFFFFFF)


def _hash(seed: int, g: np.ndarray) -> np.ndarray:
    # the same finalizer as fill_hash in csrc/util.cu
    with np.errstate(over="ignore"):
        z = (g + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15) + np.uint64(seed) * np.uint64(0xD1B54A32D192ED03)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def fill_at(kind: str, seed: int, g: np.ndarray) -> np.ndarray:
    """float64 values of the fill at global linear indices g."""
    g = np.asarray(g, dtype=np.uint64)
    if kind == "ones":
        return np.ones(g.shape)
    if kind == "ramp":
        return (g % np.uint64(97)).astype(np.float64) + 1.0
    if kind == "hash":
        return (_hash(seed, g) % np.uint64(97)).astype(np.float64) + 1.0
    raise ValueError(f"unknown fill {kind!r}")


def sample_outputs(extents, k: int, count: int, seed: int = 0) -> np.ndarray:
    """Flat output indices (of the contraction over mode k) to check: the
    first and last element plus seeded random ones."""
    n_out = math.prod(extents) // extents[k]
    rng = np.random.default_rng(seed)
    idx = rng.integers(0, n_out, size=max(0, count - 2))
    return np.unique(np.concatenate([[0, n_out - 1], idx])).astype(np.int64)


def tvc_expected(extents, k: int, x: np.ndarray, kind: str, seed: int, out_idx: np.ndarray) -> np.ndarray:
    """Exact float64 values of (A x_k x)[out_idx] for the filled tensor A
    (integer fill, integer x: every partial sum is an exact double when
    max|A| * sum|x| < 2^53)."""
    extents = [int(e) for e in extents]
    nk = extents[k]
    v = math.prod(extents[k + 1:])
    out_idx = np.asarray(out_idx, dtype=np.int64)
    i, r = np.divmod(out_idx, v)  # output (i, r) <- A[i, j, r] over j
    j = np.arange(nk, dtype=np.int64)
    g = (i[:, None] * nk + j[None, :]) * v + r[:, None]
    vals = fill_at(kind, seed, g.astype(np.uint64))
    return vals @ np.asarray(x, dtype=np.float64)


def tvc_expected_slab(extents, s: int, lo: int, hi: int, k: int, x: np.ndarray, kind: str, seed: int,
                      out_idx: np.ndarray) -> np.ndarray:
    """tvc_expected for the rank-local slab [lo, hi) along mode s of the
    filled global tensor (k != s: the rank's own output; out_idx indexes the
    contraction of the slab)."""
    ext = [int(e) for e in extents]
    loc = list(ext)
    loc[s] = hi - lo
    nk = loc[k]
    v = math.prod(loc[k + 1:])
    out_idx = np.asarray(out_idx, dtype=np.int64)
    i, r = np.divmod(out_idx, v)
    j = np.arange(nk, dtype=np.int64)
    flat = (i[:, None] * nk + j[None, :]) * v + r[:, None]  # local linear index
    multi = list(np.unravel_index(flat, loc))
    multi[s] = multi[s] + lo
    g = np.ravel_multi_index(multi, ext).astype(np.uint64)
    return fill_at(kind, seed, g) @ np.asarray(x, dtype=np.float64)


def hopm_last_update_expected(extents, vectors, kind: str, seed: int, idx: np.ndarray) -> np.ndarray:
    """The last update of a dHOPM3 sweep contracts every mode but the last
    with the sweep's final vectors x_0 .. x_{d-2}: y[i] = sum A[..., i]
    prod x_m.  Returns y at the sampled last-mode indices in float64 (one
    (n_0 ... n_{d-2}) slice of the fill per sample); the run's x_{d-1}[i]
    must equal y[i] / lambda, lambda = ||y|| = the sweep's last norm."""
    ext = [int(e) for e in extents]
    d = len(ext)
    n_last = ext[-1]
    lead = math.prod(ext[:-1])
    base = np.arange(lead, dtype=np.uint64) * np.uint64(n_last)
    out = []
    for i in np.asarray(idx, dtype=np.int64):
        a = fill_at(kind, seed, base + np.uint64(i)).reshape(ext[:-1])
        for m in range(d - 2, -1, -1):  # contract the trailing mode first
            a = a @ np.asarray(vectors[m], dtype=np.float64)
        out.append(float(a))
    return np.asarray(out)


def check_tvc_samples(got: np.ndarray, expected: np.ndarray, storage: str) -> bool:
    """Bitwise comparison in the storage format: the expected exact sum
    demoted the way the kernels store it (RNE to f32 / f16; brain = f32 RNE
    then truncation of the low 16 bits)."""
    got = np.asarray(got)
    if storage == "double":
        want = expected.astype(np.float64)
    elif storage == "single":
        want = expected.astype(np.float32)
    elif storage == "half":
        want = expected.astype(np.float16)
    else:
        want = (expected.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    return bool(np.array_equal(got.view(np.uint8), want.view(np.uint8)))
