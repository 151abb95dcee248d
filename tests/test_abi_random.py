"""Randomised CPU checks of the host-side rule builder (fqnm_plan_validate, no GPU):
for random exact kappa the derived admissible range is exactly the largest symmetric
range on which the oracle's maps satisfy D8 (or the fast path's cap), and a declared
range is accepted exactly when the oracle's maps satisfy D8 on it."""
from fractions import Fraction

import numpy as np
import pytest
from hypothesis import example, given, settings, strategies as st

import oracle

pytestmark = pytest.mark.filterwarnings("ignore")


@pytest.fixture(scope="module")
def F():
    from paper_2604_06947_b200 import _build
    _build.build()
    import paper_2604_06947_b200 as F
    return F


def _d8_ok(r, lo, hi):
    q = np.arange(lo, hi + 1)
    dp, dm = np.diff(r.phi_plus(q)), np.diff(r.phi_minus(q))
    return bool(((dp >= 0) & (dm <= 0) & (dp - dm <= 1)).all())


@settings(max_examples=25, deadline=None, derandomize=True)
@given(P=st.integers(1, 50), Q=st.integers(2_000, 5_000_000))
@example(P=1, Q=4186126)          # capped by the fast path: kappa A^2 < 2^20 < kappa (A+1)^2
@example(P=1, Q=1724240)          # cfg4's kappa
@example(P=1, Q=750000)           # cfg2's kappa
def test_eo_derived_range_is_the_d8_range(F, P, Q):
    kap = Fraction(P, Q)
    info = F.fqnm_plan_validate(1 << 20, 1.0, float(2 * kap), F.BURGERS_EO, kappa=(P, Q))
    g = int(np.gcd(P, Q))
    assert (info["kappa_num"], info["kappa_den"]) == (P // g, Q // g)
    A = info["q_hi"]
    assert info["q_lo"] == -A and A >= 1
    r = oracle.Rule(oracle.BURGERS_EO, 1, 2 * kap)         # kappa = delta dt/dx / 2 = P/Q
    assert _d8_ok(r, -A, A)
    # the fast closed form's domain: |q| < 2^22 and kappa q^2 <= 2^20 (maps.cuh eo_gm)
    capped = A + 1 > (1 << 22) - 1 or kap * (A + 1) ** 2 > (1 << 20)
    if not capped:
        assert info["d8_lim"] == 0
        assert not _d8_ok(r, -A - 1, A + 1)
    elif info["d8_lim"]:
        # capped: d8_lim is the D8 range, and range-checked steps fall back to int64 there
        D = info["d8_lim"]
        assert D > A and _d8_ok(r, -D, D) and not _d8_ok(r, -D - 1, D + 1)
    else:                          # the D8 range ends exactly at the fast domain's edge
        assert not _d8_ok(r, -A - 1, A + 1)


@settings(max_examples=25, deadline=None, derandomize=True)
@given(lam=st.fractions(Fraction(1, 20), Fraction(3, 2), max_denominator=40),
       alpha=st.fractions(Fraction(1, 2), Fraction(3), max_denominator=10),
       A=st.integers(10, 3000))
def test_lf_declared_range_accepted_iff_d8(F, lam, alpha, A):
    delta = Fraction(1, 1000)
    r = oracle.Rule(oracle.BURGERS_LF, delta, lam, alpha)
    ok = _d8_ok(r, -A, A)
    try:
        info = F.fqnm_plan_validate(1 << 16, float(delta), float(lam), F.BURGERS_LF,
                                    flux_param=float(alpha), q_range=(-A, A))
        accepted = True
        assert info["q_lo"] == -A and info["q_hi"] == A
    except F.FqnmError as e:
        if e.status != 2:                                  # only FQNM_ERR_CFL is expected
            pytest.skip(f"rationalisation refused: {e}")
        accepted = False
    assert accepted == ok
