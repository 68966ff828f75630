"""The dHOPM3 contraction schedule and its per-rank traffic model.

Restates the executable part of the reference cost model
(pkg/src/tenvec/costmodel.py:138-276): Algorithm 1 of the paper
 as an explicit list of TVC steps per rank, used by
``dhopm3`` to drive the device chain and size the three rotation buffers
(hopm.py:264, 273), and by ``bench.py`` for the algorithmic bytes of a sweep
(the roofline numerator).  The closed forms of costmodel.py:56-132 are pure
integer algebra outside the hot path and are not restated.
"""

from __future__ import annotations

from dataclasses import dataclass

from .tensor import make_split_plan

__all__ = ["iteration_plan", "tvc_per_sweep", "TvcStep", "sweep_steps", "HopmSimRank",
           "simulate_hopm", "sweep_bytes"]


def iteration_plan(d: int, j: int, reuse: bool) -> tuple[frozenset, list[int]]:
    """(modes already folded into the iteration's input, modes to contract in
    order) for external iteration j (costmodel.py:138-153).

    reuse: j = 0 contracts 1..d-1 from A; j = 1 contracts 0, 2..d-1 from A (its
    first product is the carried tensor W); j >= 2 starts from W, whose modes
    0..j-2 are gone, and contracts j-1 then j+1..d-1.  Without reuse every
    iteration contracts all modes but j from A.
    """
    above = list(range(j + 1, d))
    if not reuse:
        return frozenset(), list(range(j)) + above
    if j == 0:
        return frozenset(), above
    if j == 1:
        return frozenset(), [0] + above
    return frozenset(range(j - 1)), [j - 1] + above


def tvc_per_sweep(d: int, reuse: bool) -> int:
    return sum(len(iteration_plan(d, j, reuse)[1]) for j in range(d))


@dataclass(frozen=True)
class TvcStep:
    """One contraction of a rank's sweep (costmodel.py:160-169)."""

    j: int
    k: int
    in_elements: int
    out_elements: int
    vec_full: int
    vec_local: int
    is_final: bool
    partial_out: bool


def sweep_steps(extents: tuple[int, ...], s: int, rank_range: tuple[int, int],
                reuse: bool = True) -> list[TvcStep]:
    """The rank's contraction sequence for one sweep (costmodel.py:172-214).

    Until the split mode s is contracted the running tensor is the rank's slab
    (extent q along s); contracting s turns it into a full-size partial sum.
    """
    d = len(extents)
    lo, hi = rank_range
    q = hi - lo

    def volume(gone: frozenset, partial: bool) -> int:
        vol = 1
        for m, n in enumerate(extents):
            if m in gone:
                continue
            vol *= q if (m == s and not partial) else n
        return vol

    out: list[TvcStep] = []
    for j in range(d):
        gone, modes = iteration_plan(d, j, reuse)
        partial = s in gone
        size = volume(gone, partial)
        last = len(modes) - 1
        for t, k in enumerate(modes):
            hits = k == s and not partial
            gone = gone | {k}
            partial = partial or hits
            nxt = volume(gone, partial)
            out.append(TvcStep(j=j, k=k, in_elements=size, out_elements=nxt,
                               vec_full=extents[k], vec_local=q if hits else extents[k],
                               is_final=t == last, partial_out=partial))
            size = nxt
    return out


@dataclass
class HopmSimRank:
    """Streamed elements per external iteration, the largest intermediate and
    the TVC count of one rank's sweep (costmodel.py:217-228)."""

    iteration_touched: list[int]
    buffer_elements: int
    tvc_count: int

    @property
    def touched(self) -> int:
        return sum(self.iteration_touched)


def simulate_hopm(extents: tuple[int, ...], s: int, p: int, vl: int = 1, reuse: bool = True,
                  convention: str = "natural") -> list[HopmSimRank]:
    """Per-rank sweep traffic (costmodel.py:231-276).  "natural" counts what
    the kernels touch (actual sizes, local vector slice at the split, 3n
    normalisation); "model" follows the closed forms' conventions."""
    if convention not in ("natural", "model"):
        raise ValueError(f"unknown convention {convention!r}")
    d = len(extents)
    plan = make_split_plan(extents[s], s, p, vl)
    sims = []
    for lo, hi in plan.ranges:
        steps = sweep_steps(extents, s, (lo, hi), reuse)
        per = [0] * d
        for st in steps:
            if convention == "natural":
                per[st.j] += st.in_elements + st.vec_local + st.out_elements
            else:
                if st.is_final and st.j != s:
                    write = -(-extents[st.j] // plan.p_eff)
                else:
                    write = st.out_elements
                per[st.j] += st.in_elements + st.vec_full + write
        for j in range(d):
            share = (hi - lo) if (convention == "model" and j == s) else extents[j]
            per[j] += 3 * share
        sims.append(HopmSimRank(per, max((st.out_elements for st in steps), default=0), len(steps)))
    return sims


def sweep_bytes(extents: tuple[int, ...], s: int, p: int, storage_bytes: int,
                vl: int = 1) -> list[int]:
    """Algorithmic bytes per rank per sweep (reuse schedule, natural convention)."""
    return [r.touched * storage_bytes for r in simulate_hopm(extents, s, p, vl, reuse=True)]
