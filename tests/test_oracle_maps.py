"""Pins for the oracle's rounding and transfer maps (Eq. flux_table).

Each test checks the oracle against something other than itself: library
rounding routines, the SPEC/paper worked examples, closed forms derived by
hand, and the literal Fraction-valued definition of Eq. flux_table.
"""
import decimal
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import rules
from oracle.rules import BURGERS_EO, BURGERS_LF, FLOOR, HALF_EVEN, LINEAR, RHA
import workloads as W


def _rha_decimal(x: Fraction) -> int:
    # decimal's ROUND_HALF_UP rounds ties away from zero: an independent RHA
    with decimal.localcontext() as ctx:
        ctx.prec = 80
        d = decimal.Decimal(x.numerator) / decimal.Decimal(x.denominator)
        return int(d.quantize(decimal.Decimal(1), rounding=decimal.ROUND_HALF_UP))


@pytest.mark.parametrize("x,expect", [(Fraction(5, 2), 3), (Fraction(-5, 2), -3),
                                      (Fraction(12, 5), 2), (Fraction(0), 0),
                                      (Fraction(-12, 5), -2), (Fraction(7, 2), 4)])
def test_rha_worked_examples(x, expect):
    # S:55-57 (2.5 -> 3, -2.5 -> -3, 2.4 -> 2): tie rule of reading A1
    assert rules.round_rational(x, RHA) == expect
    assert oracle.round_rational(x.numerator, x.denominator, RHA) == expect


def test_rounding_rules_match_library_routines():
    rng = np.random.default_rng(1)
    xs = [Fraction(int(n), int(d)) for n, d in zip(rng.integers(-10**6, 10**6, 3000),
                                                    rng.integers(1, 50, 3000))]
    xs += [Fraction(2 * k + 1, 2) for k in range(-20, 20)]          # all ties
    xs += [Fraction(-(10**30) - 10**12, 2 * 10**12), Fraction(10**30 + 10**12, 2 * 10**12),
           Fraction(10**30 + 7, 3 * 10**12)]                              # 128-bit numerators, ties
    for x in xs:
        assert rules.round_rational(x, RHA) == _rha_decimal(x)
        assert rules.round_rational(x, HALF_EVEN) == round(x)          # Python: half-even
        assert rules.round_rational(x, FLOOR) == math.floor(x)
        for r in (RHA, HALF_EVEN, FLOOR):
            assert oracle.round_rational(x.numerator, x.denominator, r) == \
                rules.round_rational(x, r)


def test_spec_worked_examples():
    # advection, delta = 0.1, dt/dx = 0.5: phi+(3) = round(1.5) = 2, phi- = 0
    r = oracle.Rule(LINEAR, "0.1", "0.5")
    assert r.phi_plus(3)[0] == 2
    assert np.all(r.phi_minus(np.arange(-50, 50)) == 0)
    # F(3, 7) = 2 + 0
    assert r.interface_flux(3, 7)[0] == 2
    # nu = 1 gives phi+(q) = q
    r1 = oracle.Rule(LINEAR, "0.1", "1")
    q = np.arange(-1000, 1000)
    assert np.array_equal(r1.phi_plus(q), q)
    # LF split of Burgers at alpha = 1: f+(1) = 0.75, f-(1) = -0.25
    fp, fm = rules.split(BURGERS_LF, 1)
    assert fp(Fraction(1)) == Fraction(3, 4) and fm(Fraction(1)) == Fraction(-1, 4)


def test_half_kappa_closed_form():
    # kappa = 1/2 (cfg1, cfg3): RHA(q/2) = q - trunc(q/2) for every signed q
    r = oracle.Rule(LINEAR, "1e-6", "0.5")
    q = np.arange(-1_000_000, 500_001, dtype=np.int64)    # cfg3's whole range
    trunc_half = np.where(q >= 0, q // 2, -((-q) // 2))
    assert np.array_equal(r.phi_plus(q), q - trunc_half)
    odd = q[q % 2 != 0]
    # every odd q is an exact tie; RHA moves it away from zero
    assert np.array_equal(r.phi_plus(odd), (odd + np.sign(odd)) // 2)


@pytest.mark.parametrize("name,qmax", [("cfg2", 150000), ("cfg4", 1_200_000)])
def test_eo_closed_form_exhaustive(name, qmax):
    w = W.cfg(name)
    lam = W.dt_dx(w, qmax)
    kap = rules.kappa(BURGERS_EO, w.delta, lam)
    assert kap == Fraction(2, 5) / (2 * qmax) == Fraction(1, 5 * qmax)
    P, Q = kap.numerator, kap.denominator
    r = oracle.Rule(BURGERS_EO, w.delta, lam)
    q = np.arange(-qmax, qmax + 1, dtype=np.int64)
    g = (2 * P * q * q + Q) // (2 * Q)                      # floor(kappa q^2 + 1/2)
    assert np.array_equal(r.phi_plus(q), np.where(q > 0, g, 0))
    assert np.array_equal(r.phi_minus(q), np.where(q < 0, g, 0))


@pytest.mark.parametrize("kind,delta,lam,param,lo,hi", [
    (LINEAR, "1e-4", "1/2", 1, -3000, 12000),
    (LINEAR, "0.1", "0.3", -1, -500, 500),
    (LINEAR, "1e-3", "7/9", 2, -800, 800),
    (BURGERS_EO, "1e-5", "4/15", 1, -50000, 150000),
    (BURGERS_LF, "1e-3", "1/3", "1.2", -1200, 1200),
    (BURGERS_LF, "0.01", "0.4", 2, -200, 200),
])
@pytest.mark.parametrize("rounding", [RHA, FLOOR, HALF_EVEN])
def test_c_maps_equal_fraction_definition(kind, delta, lam, param, lo, hi, rounding):
    """The C oracle's phi equals the literal Eq. flux_table (Fraction arithmetic)."""
    r = oracle.Rule(kind, delta, Fraction(lam), Fraction(param), rounding)
    rng = np.random.default_rng(7)
    qs = np.unique(np.concatenate([np.arange(lo, min(hi, lo + 400)),
                                   rng.integers(lo, hi + 1, 1500), [0, 1, -1, lo, hi]]))
    pp, pm = r.phi_plus(qs), r.phi_minus(qs)
    for q, a, b in zip(qs.tolist(), pp.tolist(), pm.tolist()):
        assert a == rules.phi(kind, delta, Fraction(lam), q, +1, Fraction(param), rounding)
        assert b == rules.phi(kind, delta, Fraction(lam), q, -1, Fraction(param), rounding)


def test_eo_ties_are_rounded_away():
    # kappa = 1/18 (delta = 1, dt/dx = 1/9): kappa q^2 = m + 1/2 exactly when q^2 = 9 mod 18
    r = oracle.Rule(BURGERS_EO, "1", Fraction(1, 9))
    P, Q = 1, 18
    q = np.arange(1, 20001, dtype=np.int64)
    ties = q[(2 * P * q * q) % (2 * Q) == Q]
    assert len(ties) > 100
    for t in ties.tolist():
        assert r.phi_plus(t)[0] == (P * t * t) // Q + 1
        assert r.phi_minus(-t)[0] == (P * t * t) // Q + 1
    # cfg2's map (kappa = 1/750000) has no exact ties at all: 2 q^2 = 750000 mod 1.5e6
    # would need q^2 to carry an odd power of two (readings coincide there)
    q = np.arange(1, 150001, dtype=np.int64)
    assert not np.any((2 * q * q) % 1_500_000 == 750_000)


@pytest.mark.parametrize("kind,delta,lam,param,lim", [
    (LINEAR, "1e-4", "1/2", 1, 20000), (BURGERS_EO, "1e-5", "4/15", 1, 20000),
    (BURGERS_LF, "1e-3", "1/3", "1.2", 1200), (LINEAR, "0.1", "0.3", -1, 20000)])
def test_maps_are_monotone(kind, delta, lam, param, lim):
    # Lemma, step 1: phi+ nondecreasing, phi- nonincreasing
    # (LF: on |u| <= alpha, where the split is monotone)
    r = oracle.Rule(kind, delta, Fraction(lam), Fraction(param))
    q = np.arange(-lim, lim + 1)
    assert np.all(np.diff(r.phi_plus(q)) >= 0)
    assert np.all(np.diff(r.phi_minus(q)) <= 0)


def test_map_coefficients_per_config():
    assert rules.kappa(LINEAR, Fraction("1e-4"), W.dt_dx(W.cfg("cfg1"))) == Fraction(1, 2)
    assert rules.kappa(LINEAR, Fraction("1e-6"), W.dt_dx(W.cfg("cfg3"))) == Fraction(1, 2)
    w2 = W.cfg("cfg2")
    assert W.dt_dx(w2, 150000) == Fraction(4, 15)
    assert rules.kappa(BURGERS_EO, w2.delta, W.dt_dx(w2, 150000)) == Fraction(1, 750000)
    c = rules.map_coefficients(BURGERS_EO, w2.delta, Fraction(4, 15), +1)
    assert c == (1, 0, 750000, rules.SUPP_POS)
    c = rules.map_coefficients(BURGERS_EO, w2.delta, Fraction(4, 15), -1)
    assert c == (1, 0, 750000, rules.SUPP_NEG)
    c = rules.map_coefficients(LINEAR, "0.1", Fraction(1, 2), -1, param=-1)
    assert c == (0, -1, 2, rules.SUPP_ALL)
