"""Pins for the oracle's conservative update (Eqs. update_rule / 7-8)
against the paper's theorems and special cases that reduce to library routines."""
from fractions import Fraction
import itertools

import numpy as np
import pytest

import oracle
from oracle import PERIODIC, TRANSMISSIVE, rules
from oracle.rules import BURGERS_EO, BURGERS_LF, FLOOR, HALF_EVEN, LINEAR, RHA
from oracle.reference import classical_step
import workloads as W

RULES = [  # (kind, delta, dt/dx, param, state range admissible under D8)
    (LINEAR, "1e-4", Fraction(1, 2), 1, (-3000, 3000)),
    (LINEAR, "1e-3", Fraction(7, 9), 1, (-3000, 3000)),
    (LINEAR, "1e-3", Fraction(1, 3), -1, (-3000, 3000)),
    (BURGERS_EO, "1e-5", Fraction(4, 15), 1, (-50000, 150000)),
    (BURGERS_LF, "1e-3", Fraction(1, 2), 1, (-1000, 1000)),
]


def tv(q):
    return int(np.abs(np.diff(np.concatenate([q, q[:1]]))).sum())


def test_unit_courant_is_exact_shift():
    # nu = 1: phi+(q) = q, the update is q'_i = q_{i-1}: np.roll by one cell
    rng = np.random.default_rng(2)
    r = oracle.Rule(LINEAR, "0.01", 1)
    q = rng.integers(-10**6, 10**6, 777)
    assert np.array_equal(r.step(q), np.roll(q, 1))
    assert np.array_equal(r.run(q, 5), np.roll(q, 5))
    assert np.array_equal(r.run(q, 777), q)        # N periodic steps return the state
    rl = oracle.Rule(LINEAR, "0.01", 1, -1)          # a = -1 moves left
    assert np.array_equal(rl.step(q), np.roll(q, -1))
    assert np.array_equal(r.step(np.array([0, 2, 0, 0])), [0, 0, 2, 0])


@pytest.mark.parametrize("kind,delta,lam,param,rng_", RULES)
@pytest.mark.parametrize("boundary", [PERIODIC, TRANSMISSIVE])
def test_constant_state_is_fixed_point(kind, delta, lam, param, rng_, boundary):
    r = oracle.Rule(kind, delta, lam, Fraction(param))
    for c in (rng_[0], -7, 0, 13, rng_[1]):
        q = np.full(33, c)
        assert np.array_equal(r.step(q, boundary), q)


@pytest.mark.parametrize("kind,delta,lam,param,rng_", RULES)
def test_conservation_max_principle_tvd(kind, delta, lam, param, rng_):
    """Lemma discrete Stokes and Lemma CFL (i)-(ii), zero tolerance."""
    r = oracle.Rule(kind, delta, lam, Fraction(param))
    rng = np.random.default_rng(3)
    for trial in range(40):
        n = int(rng.integers(2, 200))
        q = rng.integers(rng_[0], rng_[1] + 1, n)
        if trial % 2:
            q = W.smooth_random(rng, n, (rng_[1] - rng_[0]) // 3, 0)
            q = np.clip(q, rng_[0], rng_[1])
        s0 = int(q.sum())
        for _ in range(25):
            qn = r.step(q)
            assert int(qn.sum()) == s0
            assert qn.min() >= q.min() and qn.max() <= q.max()
            assert tv(qn) <= tv(q)
            q = qn


@pytest.mark.parametrize("kind,delta,lam,param,rng_", RULES)
def test_l1_contraction(kind, delta, lam, param, rng_):
    """Lemma CFL (iii), Eq. l1_contraction."""
    r = oracle.Rule(kind, delta, lam, Fraction(param))
    rng = np.random.default_rng(4)
    for _ in range(60):
        n = int(rng.integers(2, 120))
        a = rng.integers(rng_[0], rng_[1] + 1, n)
        b = np.clip(a + rng.integers(-50, 51, n), rng_[0], rng_[1])
        for _ in range(10):
            an, bn = r.step(a), r.step(b)
            assert np.abs(an - bn).sum() <= np.abs(a - b).sum()
            a, b = an, bn


def test_lf_separately_rounded_maps_can_break_monotonicity():
    """Reading A16 / S:237: with each map rounded separately (Eq. flux_table), the LF
    split at dt/dx = 1/3, alpha = 1.2 violates the integer condition D8 although
    nu = 0.4 <= 1, and the scheme really loses TVD there.  The plan must refuse
    such rules (FQNM_ERR_CFL); this documents why D8, not nu <= 1, is checked."""
    r = oracle.Rule(BURGERS_LF, "1e-3", Fraction(1, 3), Fraction("1.2"))
    q = np.arange(-1200, 1201)
    dp, dm = np.diff(r.phi_plus(q)), np.diff(r.phi_minus(q))
    assert np.any(dp - dm > 1)
    rng = np.random.default_rng(3)
    broke = False
    for _ in range(200):
        a = W.smooth_random(rng, 64, 120, 0)
        for _ in range(30):
            b = r.step(a)
            if tv(b) > tv(a):
                broke = True
                break
            a = b
        if broke:
            break
    assert broke


def test_transmissive_mass_change_is_boundary_flux():
    # with ghost copies the telescoping sum leaves F_{-1/2} - F_{N-1/2} (reading A12)
    rng = np.random.default_rng(5)
    for kind, delta, lam, param, rng_ in RULES:
        r = oracle.Rule(kind, delta, lam, Fraction(param))
        q = rng.integers(rng_[0], rng_[1] + 1, 57)
        qn = r.step(q, TRANSMISSIVE)
        Fl = r.interface_flux(q[0], q[0])[0]
        Fr = r.interface_flux(q[-1], q[-1])[0]
        assert int(qn.sum()) - int(q.sum()) == Fl - Fr


@pytest.mark.parametrize("kind,delta,lam,param,rng_", RULES)
def test_fourterm_equals_flux_difference(kind, delta, lam, param, rng_):
    # Eq. update_rule is identical to the flux-difference form
    r = oracle.Rule(kind, delta, lam, Fraction(param))
    rng = np.random.default_rng(6)
    for _ in range(20):
        q = rng.integers(rng_[0], rng_[1] + 1, int(rng.integers(2, 300)))
        assert np.array_equal(r.step(q), r.step_fourterm(q))


def test_flux_difference_by_hand():
    # explicit F_{i+1/2} = phi+(q_i) + phi-(q_{i+1}); q' = q - (F_{i+1/2} - F_{i-1/2})
    r = oracle.Rule(BURGERS_LF, "1e-3", Fraction(1, 3), Fraction("1.2"))
    rng = np.random.default_rng(8)
    q = rng.integers(-1000, 1000, 50)
    F = r.phi_plus(q) + r.phi_minus(np.roll(q, -1))          # F[i] = F_{i+1/2}
    assert np.array_equal(r.step(q), q - (F - np.roll(F, 1)))


def test_translation_equivariance_and_composition():
    rng = np.random.default_rng(9)
    for kind, delta, lam, param, rng_ in RULES:
        r = oracle.Rule(kind, delta, lam, Fraction(param))
        q = rng.integers(rng_[0], rng_[1] + 1, 101)
        for s in (1, 17, 50):
            assert np.array_equal(r.run(np.roll(q, s), 7), np.roll(r.run(q, 7), s))
        assert np.array_equal(r.run(q, 12), r.run(r.run(q, 5), 7))   # step(a+b) = step(b) o step(a)


def test_eo_mirror_equivariance():
    # Burgers is invariant under (x, u) -> (-x, -u); the EO maps satisfy phi+(-q) = phi-(q)
    w = W.cfg("cfg2")
    r = oracle.Rule(BURGERS_EO, w.delta, Fraction(4, 15))
    rng = np.random.default_rng(10)
    q = rng.integers(-50000, 50001, 300)
    assert np.array_equal(r.run(-q[::-1], 9), -r.run(q, 9)[::-1])


def _monotone_under_perturbation(r, states, boundary=PERIODIC):
    """For every state and every cell j, q -> q + e_j must not decrease any q'."""
    ok = True
    for q in states:
        base = r.step(q, boundary)
        for j in range(len(q)):
            p = q.copy(); p[j] += 1
            if np.any(r.step(p, boundary) < base):
                ok = False
                break
        if not ok:
            break
    return ok


def _d8(r, lo, hi):
    q = np.arange(lo, hi + 1)
    dp = np.diff(r.phi_plus(q)); dm = np.diff(r.phi_minus(q))
    return bool(np.all(dp >= 0) and np.all(dm <= 0) and np.all(dp - dm <= 1))


@pytest.mark.parametrize("kind,lam,param,rounding,expect", [
    (LINEAR, Fraction(1, 2), 1, RHA, True),
    (LINEAR, Fraction(1), 1, RHA, True),
    (LINEAR, Fraction(5, 4), 1, RHA, False),          # nu > 1
    (BURGERS_EO, Fraction(1, 10), 1, RHA, True),       # kappa = 1/20
    (BURGERS_EO, Fraction(1, 6), 1, RHA, True),        # kappa = 1/12
    (BURGERS_EO, Fraction(1, 4), 1, RHA, True),        # kappa = 1/8 (holds on [-4,5])
    (BURGERS_EO, Fraction(2, 3), 1, RHA, False),       # kappa = 1/3: phi(3)-phi(2) = 2
    (BURGERS_EO, Fraction(1), 1, RHA, False),          # kappa = 1/2
    (LINEAR, Fraction(1, 2), 1, FLOOR, True),
    (LINEAR, Fraction(1, 2), 1, HALF_EVEN, True),
    (BURGERS_LF, Fraction(1, 3), 1, RHA, None),
])
def test_bruteforce_monotonicity_iff_d8(kind, lam, param, rounding, expect):
    """Every state in [-4,4]^4 (periodic): the update map is order preserving
    exactly when the integer condition D8 holds on the range, and then the
    maximum principle and TVD hold for every state (Lemma P:197-238)."""
    R = 4
    r = oracle.Rule(kind, "1", lam, Fraction(param), rounding)
    d8 = _d8(r, -R, R + 1)
    if expect is not None:
        assert d8 == expect
    states = [np.array(s) for s in itertools.product(range(-R, R + 1), repeat=4)]
    mono = _monotone_under_perturbation(r, states)
    assert mono == d8
    if d8:
        for q in states:
            qn = r.step(q)
            assert qn.sum() == q.sum()
            assert qn.min() >= q.min() and qn.max() <= q.max()
            assert tv(qn) <= tv(q)


@pytest.mark.parametrize("kind,delta,lam,param,rng_", RULES)
def test_prop1_update_level_correspondence(kind, delta, lam, param, rng_):
    """Prop. 1: |delta (q'_i - q_i) + lam (F(u_i,u_{i+1}) - F(u_{i-1},u_i))| <= 2 delta,
    evaluated exactly in rational arithmetic."""
    delta = Fraction(delta)
    fp, fm = rules.split(kind, Fraction(param))
    r = oracle.Rule(kind, delta, lam, Fraction(param))
    rng = np.random.default_rng(11)
    for _ in range(5):
        q = rng.integers(rng_[0], rng_[1] + 1, 40)
        qn = r.step(q)
        u = [delta * int(v) for v in q]
        n = len(u)
        for i in range(n):
            F = lambda a, b: fp(a) + fm(b)
            classical = lam * (F(u[i], u[(i + 1) % n]) - F(u[i - 1], u[i]))
            resid = delta * (int(qn[i]) - int(q[i])) + classical
            assert abs(resid) <= 2 * delta


def test_classical_scheme_and_fqnm_agree_to_o_delta():
    # Prop. 1 / Thm consistency at the trajectory level: |delta q^n - v^n| <= (1/2 + 2n) delta
    rng = np.random.default_rng(12)
    delta = 1e-7
    r = oracle.Rule(BURGERS_EO, "1e-7", Fraction(1, 2))
    x = W.cell_centres(256)
    u0 = 0.3 + 0.5 * np.sin(2 * np.pi * x) + 0.1 * rng.standard_normal(256)
    q = W.quantise(u0, delta)
    v = u0.copy()
    for n in range(1, 41):
        q = r.step(q)
        v = classical_step(v, BURGERS_EO, 0.5)
        assert np.abs(delta * q - v).sum() / 256 <= (0.5 + 2 * n) * delta + 1e-12


def test_survey_crosscheck_cfg1():
    """Cross-check (not a pin): SURVEY §8(c)-C5 lists an independent scratch run of
    cfg1 after 2000 steps: sum 907,484, min 1, max 8511, TV 17,020."""
    w = W.cfg("cfg1")
    q0 = W.q0_cfg1()
    assert int(q0.sum()) == 907484 and int(q0.max()) == 9999
    q = oracle.Rule(LINEAR, w.delta, W.dt_dx(w)).run(q0, 2000)
    assert (int(q.sum()), int(q.min()), int(q.max()), tv(q)) == (907484, 1, 8511, 17020)


def test_observe_is_the_plain_product():
    rng = np.random.default_rng(13)
    q = rng.integers(-2**40, 2**40, 1000)
    for d in (1e-4, 1e-7, 0.1, 3.0):
        assert np.array_equal(oracle.observe(q, d), d * q.astype(np.float64))
