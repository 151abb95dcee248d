"""Pins for the oracle's componentwise-quantised Roe transfer (BJ.cfg5; Roe flux
structure P:564-575, quantised two-point flux Eq.) and for the
exact Sod solution used to judge it.

The paper gives no convergence theorem for systems, so the absolute
accuracy of the quantised Euler scheme is only checked heuristically (parity
unpinned for that claim).  Its arithmetic is pinned by: consistency at equal
states, exact mirror symmetry, reduction to upwinding for supersonic states,
agreement with an independently derived eigen-decomposition form of the Roe
flux, and the exact conservation properties of the update.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import rules
from oracle.reference import riemann_star, sod_exact, sod_wave_data
import workloads as W

G = 1.4
G1 = G - 1.0


def _rha_double(x: float) -> int:
    return rules.round_rational(Fraction(x), rules.RHA)


def _phys(q, delta):
    rho, m, E = (delta * float(v) for v in q)
    u = m / rho
    mu = m * u
    p = G1 * (E - 0.5 * mu)
    return rho, m, E, u, p, np.array([m, mu + p, u * (E + p)])


def _random_state(rng, delta, mach_lo=-0.5, mach_hi=0.5):
    rho = rng.uniform(0.1, 2.0)
    p = rng.uniform(0.1, 2.0)
    c = math.sqrt(G * p / rho)
    u = rng.uniform(mach_lo, mach_hi) * c
    E = p / G1 + 0.5 * rho * u * u
    return np.array([round(rho / delta), round(rho * u / delta), round(E / delta)], dtype=np.int64)


def test_consistency_at_equal_states():
    rng = np.random.default_rng(20)
    delta, lam = 1e-7, 0.3
    s = lam / delta
    for _ in range(300):
        q = _random_state(rng, delta, -3, 3)
        T = oracle.roe_transfer(q, q, delta, lam)
        f = _phys(q, delta)[5]
        assert [_rha_double(fc * s) for fc in f] == T.tolist()


def _roe_speeds(qa, qb, delta):
    rl, ml, El, ul, pl, _ = _phys(qa, delta)
    rr, mr, Er, ur, pr, _ = _phys(qb, delta)
    wl, wr = math.sqrt(rl), math.sqrt(rr)
    ut = (wl * ul + wr * ur) / (wl + wr)
    Ht = (wl * (El + pl) / rl + wr * (Er + pr) / rr) / (wl + wr)
    at = math.sqrt(G1 * (Ht - 0.5 * ut * ut))
    return np.array([ut - at, ut, ut + at]), 0.05 * (abs(ut) + at)


def test_supersonic_states_reduce_to_upwind():
    # all Roe speeds of one sign, no entropy fix active: F_Roe = f(U_upwind) exactly
    rng = np.random.default_rng(21)
    delta, lam = 1e-7, 0.2
    s = lam / delta
    checked = 0
    for sign in (+1, -1):
        for _ in range(400):
            qa = _random_state(rng, delta, 1.6, 3.0)
            qb = _random_state(rng, delta, 1.6, 3.0)
            if sign < 0:
                qa[1] *= -1; qb[1] *= -1
            lams, eps = _roe_speeds(qa, qb, delta)
            if np.any(sign * lams < 1.01 * eps):
                continue
            checked += 1
            T = oracle.roe_transfer(qa, qb, delta, lam)
            up = qa if sign > 0 else qb
            f = _phys(up, delta)[5]
            expect = [_rha_double(fc * s) for fc in f]
            assert np.all(np.abs(T - np.array(expect)) <= 1)
    assert checked > 300


def test_roe_flux_matches_eigendecomposition_form():
    """F = f(U_L) + sum_{lambda_k < 0} lambda_k alpha_k r_k with alpha = R^{-1} dU solved
    numerically from independently assembled Roe-average eigenvectors (no entropy fix
    active): equal to the oracle's 1/2(fL+fR) - 1/2 sum |lambda_k| alpha_k r_k."""
    rng = np.random.default_rng(22)
    delta, lam = 1e-7, 0.25
    s = lam / delta
    checked = 0
    for _ in range(2000):
        qa = _random_state(rng, delta, -1.5, 1.5)
        qb = _random_state(rng, delta, -1.5, 1.5)
        rl, ml, El, ul, pl, fl = _phys(qa, delta)
        rr, mr, Er, ur, pr, fr = _phys(qb, delta)
        Hl, Hr = (El + pl) / rl, (Er + pr) / rr
        wl, wr = math.sqrt(rl), math.sqrt(rr)
        ut = (wl * ul + wr * ur) / (wl + wr)
        Ht = (wl * Hl + wr * Hr) / (wl + wr)
        at = math.sqrt(G1 * (Ht - 0.5 * ut * ut))
        lams = np.array([ut - at, ut, ut + at])
        eps = 0.05 * (abs(ut) + at)
        if np.any(np.abs(lams) < eps * 1.01):
            continue
        R = np.array([[1.0, 1.0, 1.0], [ut - at, ut, ut + at],
                      [Ht - ut * at, 0.5 * ut * ut, Ht + ut * at]])
        dU = np.array([rr - rl, mr - ml, Er - El])
        alpha = np.linalg.solve(R, dU)
        F = fl + sum(lams[k] * alpha[k] * R[:, k] for k in range(3) if lams[k] < 0)
        T = oracle.roe_transfer(qa, qb, delta, lam)
        expect = np.array([_rha_double(v * s) for v in F])
        assert np.all(np.abs(T - expect) <= 1), (qa, qb, T, expect)
        checked += 1
    assert checked > 1000


def _mirror(q):
    m = q[:, ::-1].copy()
    m[1] *= -1
    return m


def test_mirror_symmetry_is_bit_exact():
    rng = np.random.default_rng(23)
    delta = 1e-7
    n = 96
    x = W.cell_centres(n)
    rho = 1.0 + 0.5 * np.sin(2 * np.pi * x) + 0.3 * (x > 0.6)
    u = 0.3 * np.cos(4 * np.pi * x)
    p = 1.0 + 0.4 * (x < 0.3)
    E = p / G1 + 0.5 * rho * u * u
    q = np.stack([np.rint(rho / delta), np.rint(rho * u / delta), np.rint(E / delta)]).astype(np.int64)
    lam = 0.25
    a = oracle.euler_run(q, 40, delta, lam)
    b = oracle.euler_run(_mirror(q), 40, delta, lam)
    assert np.array_equal(_mirror(a), b)


def test_sod_conservation_before_waves_reach_walls():
    n = 200
    nsteps, lam = W.sod_steps_and_dt_dx(n)
    q = W.sod_q0(n)
    delta = 1e-7
    assert q[:, 0].tolist() == [10**7, 0, 25 * 10**6]
    assert q[:, -1].tolist() == [125 * 10**4, 0, 25 * 10**5]
    wall = oracle.roe_transfer(q[:, 0], q[:, 0], delta, lam)[1] - \
        oracle.roe_transfer(q[:, -1], q[:, -1], delta, lam)[1]
    sums = q.sum(axis=1)
    for k in range(1, 41):
        q = oracle.euler_step(q, delta, lam)
        assert q[0].sum() == sums[0] and q[2].sum() == sums[2]
        assert q[1].sum() == sums[1] + k * wall


def test_sod_heuristic_convergence():
    """No theorem for systems: L1(rho) against the exact Sod solution must
    decrease with N and be small; mass is exact.  (Heuristic accuracy check.)"""
    errs = []
    for n in (100, 200, 400):
        nsteps, lam = W.sod_steps_and_dt_dx(n)
        q = oracle.euler_run(W.sod_q0(n, Fraction("1e-9")), nsteps, 1e-9, lam)
        rho = oracle.observe(q[0], 1e-9)
        rho_ex, _, _ = sod_exact(W.cell_centres(n), 0.2)
        errs.append(np.abs(rho - rho_ex).mean())
        assert q.min() >= -10**10
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < 0.02


def test_exact_sod_solution_pins():
    # textbook star state of the Sod problem (recomputed: S:419)
    ps, us, rsl, rsr, S = sod_wave_data()
    assert abs(ps - 0.30313) < 1e-5 and abs(us - 0.92745) < 1e-5
    assert abs(rsl - 0.42632) < 1e-5 and abs(rsr - 0.26557) < 1e-5
    rl, ul, pl = 1.0, 0.0, 1.0
    rr, ur, pr = 0.125, 0.0, 0.1
    # Rankine-Hugoniot across the right shock (mass, momentum, energy fluxes)
    def flux(r, u, p):
        E = p / G1 + 0.5 * r * u * u
        return np.array([r * u, r * u * u + p, u * (E + p)]), np.array([r, r * u, E])
    f1, U1 = flux(rr, ur, pr)
    f2, U2 = flux(rsr, us, ps)
    assert np.allclose(f2 - f1, S * (U2 - U1), rtol=1e-10, atol=1e-12)
    # isentropic left rarefaction; shock position 0.5 + 0.2 S = 0.8504 (inside P:603's zoom)
    assert abs(ps / rsl ** G - pl / rl ** G) < 1e-12
    assert 0.84 < 0.5 + 0.2 * S < 0.86
    rho, u, p = sod_exact(np.array([0.1, 0.6, 0.8, 0.9]), 0.2)
    assert rho[0] == 1.0 and rho[3] == 0.125 and abs(rho[2] - rsr) < 1e-12


def test_sod_config_steps():
    # reading A11: nsteps = ceil(T c_L N / 0.4), lambda = fl(fl(T N)/nsteps)
    nsteps, lam = W.sod_steps_and_dt_dx(1 << 26)
    assert nsteps == 39702140
    assert lam == (0.2 * (1 << 26)) / nsteps
    assert W.sod_steps_and_dt_dx(1 << 16)[0] == 38772


# ---------------------------------------------------------------------------
# density-only quantisation (the paper's Sod prototype; NEXT-f2)

def _sod_mixed(n, delta=1e-7):
    q = W.sod_q0(n, Fraction(str(delta)))
    rho_q = q[0]
    m = np.zeros(n)
    E = np.where(np.arange(n) < n // 2, 1.0 / 0.4, 0.1 / 0.4)
    return oracle.pack_mixed(rho_q, m, E)


def test_density_only_constant_state_is_fixed():
    n = 64
    q = oracle.pack_mixed(np.full(n, 10**7), np.full(n, 0.3), np.full(n, 3.1))
    out = oracle.euler_density_step(q, 1e-7, 0.25)
    assert np.array_equal(out, q)


def test_density_only_mirror_symmetry_is_bit_exact():
    n = 128
    x = W.cell_centres(n)
    rho = 1.0 + 0.5 * np.sin(2 * np.pi * x) + 0.3 * (x > 0.6)
    u = 0.3 * np.cos(4 * np.pi * x)
    p = 1.0 + 0.4 * (x < 0.3)
    E = p / G1 + 0.5 * rho * u * u
    q = oracle.pack_mixed(np.rint(rho / 1e-7).astype(np.int64), rho * u, E)
    a = oracle.euler_density_run(q, 40, 1e-7, 0.25)

    def mirror(qq):
        r, m_, e_ = oracle.unpack_mixed(qq)
        return oracle.pack_mixed(r[::-1], -m_[::-1], e_[::-1])
    b = oracle.euler_density_run(mirror(q), 40, 1e-7, 0.25)
    assert np.array_equal(mirror(a), b)


def test_density_only_mass_is_exact_and_matches_full_quantisation_flux():
    n = 200
    nsteps, lam = W.sod_steps_and_dt_dx(n)
    q = _sod_mixed(n)
    s0 = q[0].sum()
    for _ in range(40):
        q = oracle.euler_density_step(q, 1e-7, lam)
        assert q[0].sum() == s0                    # integer density: exact (waves off the walls)
    r, m, E = oracle.unpack_mixed(q)
    assert abs(E.sum() - _sod_mixed(n)[2].view(np.float64).sum()) < 1e-9 * n


def test_density_only_sod_heuristic_convergence():
    """Heuristic accuracy (no theorem for systems): L1(rho) vs exact Sod
    decreases with N for the density-only prototype."""
    errs = []
    for n in (100, 200, 400):
        nsteps, lam = W.sod_steps_and_dt_dx(n)
        q = oracle.euler_density_run(_sod_mixed(n, 1e-9), nsteps, 1e-9, lam)
        rho = oracle.observe(q[0], 1e-9)
        rho_ex, _, _ = sod_exact(W.cell_centres(n), 0.2)
        errs.append(np.abs(rho - rho_ex).mean())
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < 0.02
