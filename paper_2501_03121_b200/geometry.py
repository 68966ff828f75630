"""Index geometry of the contraction path: extents, the (u, n_k, v) block
view of a mode, and the 1-D split of a mode over ranks.

These are integers the kernels and the collectives agree on, so they follow
the reference exactly (pkg/src/tenvec/tensor.py:25-144): the same
validation, the same ceil(n/p) chunk promoted to the vector length, the
same effective rank count.  Nothing here touches a device.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import reduce
from typing import NamedTuple

__all__ = ["Shape", "parse_shape", "linear_index", "MatricizedDims", "matricize_dims", "optimal_division",
           "SplitPlan", "make_split_plan"]


def _ceil_div(a: int, b: int) -> int:
    return -(-a // b)


@dataclass(frozen=True)
class Shape:
    """Extents, last mode fastest; at least one mode, each >= 1
    (tensor.py:25-60)."""

    extents: tuple[int, ...]

    def __post_init__(self) -> None:
        ext = tuple(self.extents)
        if not ext:
            raise ValueError("a tensor has at least one mode")
        if not all(int(n) == n and n >= 1 for n in ext):
            raise ValueError(f"extents must be positive integers, got {self.extents}")
        object.__setattr__(self, "extents", tuple(map(int, ext)))

    order = property(lambda self: len(self.extents))
    size = property(lambda self: math.prod(self.extents))

    def drop(self, k: int) -> "Shape":
        """The shape left after contracting mode k (a vector contracts to
        one element, kept as shape (1,))."""
        if self.order > 1:
            return Shape(self.extents[:k] + self.extents[k + 1:])
        if k != 0:
            raise IndexError(f"mode {k} out of range for order-1 shape")
        return Shape((1,))

    def with_extent(self, k: int, n: int) -> "Shape":
        return Shape(tuple(n if i == k else e for i, e in enumerate(self.extents)))

    def __str__(self) -> str:
        return "x".join(map(str, self.extents))


def parse_shape(text: str) -> Shape:
    """"2,3,4", "2x3x4" or the hypersquare form "979^3" (tensor.py:63-70)."""
    body = text.strip()
    base, caret, power = body.partition("^")
    if caret:
        return Shape((int(base),) * int(power))
    return Shape(tuple(int(t) for t in body.split("," if "," in body else "x")))


def linear_index(shape: Shape, idx: tuple[int, ...]) -> int:
    """Row-major offset of a multi-index (last mode fastest)."""
    if len(idx) != shape.order:
        raise IndexError(f"index of length {len(idx)} for order-{shape.order} shape")
    for i, n in zip(idx, shape.extents):
        if i < 0 or i >= n:
            raise IndexError(f"component {i} out of range [0, {n})")
    return reduce(lambda acc, pair: acc * pair[1] + pair[0], zip(idx, shape.extents), 0)


class MatricizedDims(NamedTuple):
    """Mode k of a shape seen as u slabs of n_k x v (tensor.py:85-95)."""

    u: int
    nk: int
    v: int


def matricize_dims(shape: Shape, k: int) -> MatricizedDims:
    if k < 0 or k >= shape.order:
        raise IndexError(f"mode {k} out of range for order-{shape.order} shape")
    before, here, after = shape.extents[:k], shape.extents[k], shape.extents[k + 1:]
    return MatricizedDims(math.prod(before), here, math.prod(after))


def optimal_division(n: int, p: int, vl: int = 1) -> tuple[int, int]:
    """(chunk, p_eff) of splitting n indices over p ranks: ceil(n/p), rounded
    up to a multiple of the vector length vl when n >= vl and capped at n
    (tensor.py:105-118)."""
    if min(n, p, vl) < 1:
        raise ValueError("extent, worker count and vector length must be >= 1")
    chunk = _ceil_div(n, p)
    if n >= vl:
        chunk = min(_ceil_div(chunk, vl) * vl, n)
    return chunk, _ceil_div(n, chunk)


@dataclass(frozen=True)
class SplitPlan:
    """The split of mode s: p requested, p_eff ranks own [r*chunk,
    min((r+1)*chunk, n)) (tensor.py:121-138)."""

    s: int
    p_requested: int
    p_eff: int
    chunk: int
    ranges: tuple[tuple[int, int], ...]

    @property
    def extent(self) -> int:
        return self.ranges[-1][1]

    def rank_extent(self, rank: int) -> int:
        lo, hi = self.ranges[rank]
        return hi - lo


def make_split_plan(n: int, s: int, p: int, vl: int = 1) -> SplitPlan:
    chunk, p_eff = optimal_division(n, p, vl)
    bounds = [min(r * chunk, n) for r in range(p_eff + 1)]
    return SplitPlan(s, p, p_eff, chunk, tuple(zip(bounds[:-1], bounds[1:])))
