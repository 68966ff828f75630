"""The dHOPM3 contraction schedule and its per-rank traffic model.

Restates the executable part of the reference cost model
(pkg/src/tenvec/costmodel.py:138-276): Algorithm 1 of the paper
 as an explicit list of TVC steps per rank, used by
``dhopm3`` to drive the device chain and size the three rotation buffers
(hopm.py:264, 273), and by ``bench.py`` for the algorithmic bytes of a sweep
(the roofline numerator).  The closed forms of costmodel.py:33-135 and
280-320 (the paper's Eqs. (3)-(6): sequential / distributed streamed elements
per external iteration and per sweep, the parallel inflation eta^-1 and the
reuse economy H^-1) are restated at the end as exact rationals; the classical
schedule's device counters are audited against them (tests/test_gpu_hopm.py).
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

from .tensor import make_split_plan

__all__ = ["iteration_plan", "tvc_per_sweep", "TvcStep", "sweep_steps", "HopmSimRank",
           "simulate_hopm", "sweep_bytes", "m_seq", "M_seq", "m_par", "M_par", "M_par_min",
           "M_par_bracketed", "splitting_shift_residual", "ring_overhead", "eta_inv", "H_inv",
           "CostReport", "cost_report"]


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


# -- closed forms (costmodel.py:33-135, 280-320; PAPER Eqs. (3)-(6)) -------
# Streamed elements per rank for a hypersquare order-d, extent-n tensor split
# along mode s over p ranks.  Conventions (costmodel.py:1-22): tensor and
# intermediates charged once per read and once per write, input vectors in
# full on every rank, the final write at one rank's share, normalisation 3
# passes over that share (j = s) or over the full vector.


def _powers(n: int, lo: int, hi: int) -> int:
    """n^lo + ... + n^hi (0 when hi < lo)."""
    return sum(n ** e for e in range(lo, hi + 1)) if hi >= lo else 0


def _valid(d: int, n: int, p: int = 1, s: int = 0) -> None:
    if d < 2:
        raise ValueError("the power method needs order >= 2")
    if n < 1 or p < 1:
        raise ValueError("extent and rank count must be >= 1")
    if not 0 <= s < d:
        raise ValueError(f"split mode {s} out of range for order {d}")


def _rank_share(block: int, n: int, p: int, division: str) -> Fraction:
    """One rank's part of a block split along an extent-n mode: exactly
    block/p, or ("ceiling") block/n times the ceil(n/p) chunk the first rank
    holds."""
    if division == "exact":
        return Fraction(block, p)
    if division == "ceiling":
        return Fraction(block // n * (-(-n // p)))
    raise ValueError(f"unknown division mode {division!r}")


def m_seq(d: int, n: int) -> int:
    """One sequential external iteration: the tensor, the d-2 intermediates
    read and written, d-1 vectors, the output and its 3-pass normalisation."""
    _valid(d, n)
    return n ** d + 2 * _powers(n, 2, d - 1) + (d + 3) * n


def M_seq(d: int, n: int) -> int:
    return d * m_seq(d, n)


def m_par(d: int, n: int, p: int, s: int, j: int, division: str = "ceiling"
          ) -> tuple[Fraction, Fraction]:
    """External iteration j on one rank: (bracketed count, its p | n
    approximation).  Iterations j != s cross the split and carry full-size
    intermediates from there on (exponents up to d-s for j < s, d-s-1 above)."""
    _valid(d, n, p, s)
    if not 0 <= j < d:
        raise ValueError(f"iteration {j} out of range for order {d}")
    rest = Fraction(p - 1, p)
    local = (_rank_share(n ** d, n, p, division)
             + 2 * sum(_rank_share(n ** e, n, p, division) for e in range(2, d))
             + 4 * _rank_share(n, n, p, division) + (d - 1) * n)
    local_approx = Fraction(m_seq(d, n), p) + rest * (d - 1) * n
    if j == s:
        return local, local_approx
    top = d - s - (0 if j < s else 1)
    crossing = rest * (2 * _powers(n, 2, top) + 3 * n)
    return (local + crossing,
            Fraction(m_seq(d, n), p) + rest * (2 * _powers(n, 2, top) + (d + 2) * n))


def M_par(d: int, n: int, p: int, s: int) -> Fraction:
    """Closed-form sweep total per rank, classical schedule (Eq. (5))."""
    _valid(d, n, p, s)
    rest = Fraction(p - 1, p)
    crossing = s * 2 * _powers(n, 2, d - s) + (d - s - 1) * 2 * _powers(n, 2, d - s - 1)
    return Fraction(M_seq(d, n), p) + rest * (d - 1) * (d + 3) * n + rest * crossing


def M_par_min(d: int, n: int, p: int) -> Fraction:
    """The split-independent part of M_par (reached at s = d - 1)."""
    _valid(d, n, p)
    return Fraction(M_seq(d, n), p) + Fraction(p - 1, p) * (d - 1) * (d + 3) * n


def M_par_bracketed(d: int, n: int, p: int, s: int, division: str = "ceiling") -> Fraction:
    return sum((m_par(d, n, p, s, j, division)[0] for j in range(d)), Fraction(0))


def splitting_shift_residual(d: int, n: int, p: int, s: int) -> Fraction:
    """M_par(s-1) - M_par(s) minus the predicted step
    (p-1)/p ((d-s-1) 2 n^(d-s) + (s-1) 2 n^(d-s+1)); zero by Eq. (6)."""
    _valid(d, n, p, s)
    if s < 1:
        raise ValueError("the recursion relates s to s-1, so s >= 1")
    step = Fraction(p - 1, p) * ((d - s - 1) * 2 * n ** (d - s) + (s - 1) * 2 * n ** (d - s + 1))
    return M_par(d, n, p, s - 1) - M_par(d, n, p, s) - step


def ring_overhead(n: int, p: int) -> Fraction:
    """Per-rank elements one ring allreduce of length n touches."""
    if n < 0 or p < 1:
        raise ValueError("need n >= 0 and p >= 1")
    return Fraction(4 * n * (p - 1), p)


def eta_inv(d: int, n: int, p: int, s: int) -> Fraction:
    """Total traffic of p ranks over one rank's: p M_par / M_seq."""
    return p * M_par(d, n, p, s) / M_seq(d, n)


def H_inv(d: int, n: int, p: int, s: int) -> Fraction:
    """Economy of the reuse schedule: closed-form classical M_par over the
    simulated reuse traffic of the widest rank."""
    return M_par(d, n, p, s) / simulate_hopm((n,) * d, s, p, reuse=True)[0].touched


@dataclass
class CostReport:
    d: int
    n: int
    p: int
    s: int
    m_seq: int
    M_par: Fraction
    M_par_min: Fraction
    eta_inv: Fraction
    H_inv: Fraction
    ring_overhead: Fraction


def cost_report(d: int, n: int, p: int, s: int) -> CostReport:
    _valid(d, n, p, s)
    return CostReport(d, n, p, s, m_seq(d, n), M_par(d, n, p, s), M_par_min(d, n, p),
                      eta_inv(d, n, p, s), H_inv(d, n, p, s), ring_overhead(n, p))
