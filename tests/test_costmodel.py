"""The closed-form streamed-memory model (schedule.py, restating
costmodel.py:33-320 / the paper's Eqs. (3)-(6)) against the reference's own
values (tests/golden/costmodel.npz, written by make_golden.py from the
reference package), plus its algebraic identities.  CPU only."""

from fractions import Fraction

import pytest

from conftest import load_golden
from paper_2501_03121_b200 import schedule as S


def test_closed_forms_equal_reference_values():
    g = load_golden("costmodel")
    for (d, n, p, s), mseq, fr in zip(g["meta"].tolist(), g["m_seq"].tolist(), g["fracs"].tolist()):
        r = S.cost_report(d, n, p, s)
        want = [Fraction(a, b) for a, b in fr]
        shift = S.splitting_shift_residual(d, n, p, s) if s >= 1 else Fraction(0)
        got = [r.M_par, r.M_par_min, r.eta_inv, r.H_inv, r.ring_overhead,
               S.M_par_bracketed(d, n, p, s), shift]
        assert r.m_seq == mseq, (d, n, p, s)
        assert got == want, (d, n, p, s)
    for d, n, p, s, j, exact, bn, bd, an, ad in g["m_par"].tolist():
        br, ap = S.m_par(d, n, p, s, j, "exact" if exact else "ceiling")
        assert (br, ap) == (Fraction(bn, bd), Fraction(an, ad)), (d, n, p, s, j, exact)


def test_identities():
    for d in range(2, 9):
        for n in range(1, 7):
            for p in range(1, n + 1):
                for s in range(d):
                    if s >= 1:
                        assert S.splitting_shift_residual(d, n, p, s) == 0
                    if n % p == 0:  # bracketed and approximate coincide
                        assert S.M_par_bracketed(d, n, p, s) == S.M_par(d, n, p, s)
                    assert S.M_par(d, n, p, s) >= S.M_par_min(d, n, p)
                assert S.M_par(d, n, p, d - 1) == S.M_par_min(d, n, p)
    assert S.M_par(4, 8, 1, 2) == S.M_seq(4, 8)
    assert S.ring_overhead(10, 4) == 30


def test_argument_errors():
    with pytest.raises(ValueError):
        S.m_seq(1, 4)
    with pytest.raises(ValueError):
        S.M_par(3, 4, 2, 3)
    with pytest.raises(ValueError):
        S.m_par(3, 4, 2, 0, 3)
    with pytest.raises(ValueError):
        S.splitting_shift_residual(3, 4, 2, 0)
    with pytest.raises(ValueError):
        S.ring_overhead(-1, 2)
    with pytest.raises(ValueError):
        S.m_par(3, 4, 2, 0, 1, division="floor")
