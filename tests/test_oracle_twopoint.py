"""Oracle pins for the quantised two-point transfer rules and the checker of
Thm transfer-operator equivalence (Remark P:284-288) — CPU only.

Phi(qL, qR) = round(F(delta qL, delta qR) dt/dx / delta), rounded once,
for the Godunov, Engquist-Osher and Lax-Friedrichs fluxes of Burgers.  The C oracle
evaluates them from integer coefficients; the pins below hold them against:
  * the literal Fraction definition, with the Godunov flux taken from the exact
    Riemann solution sampled at x/t = 0 (a definition independent of the max formula);
  * consistency Phi(q, q) = round(f(delta q) dt/dx / delta);
  * monotonicity of the Godunov flux, F_God <= F_EO, F_God = F_EO off transonic pairs;
  * the theorem itself: equal Phi on every visited state -> identical trajectories,
    and a brute-force recount of the checker's statistics on a tiny case;
  * conservation and the L1 ladder against the closed-form entropy solution.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import rules as R
from oracle.reference import burgers_tophat_exact
import workloads as W

KINDS = [R.BURGERS_GODUNOV, R.BURGERS_EO2, R.BURGERS_LF2]


def _rule(kind, delta="1/10", lam=Fraction(1, 2), alpha=Fraction(2)):
    return oracle.TransferRule(kind, delta, lam, alpha)


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("rounding", [R.RHA, R.FLOOR, R.HALF_EVEN])
def test_c_transfer_equals_literal_definition(kind, rounding):
    delta, lam, alpha = Fraction(1, 10), Fraction(1, 2), Fraction(2)
    t = oracle.TransferRule(kind, delta, lam, alpha, rounding)
    a, b = np.meshgrid(np.arange(-30, 31), np.arange(-30, 31), indexing="ij")
    got = t.phi(a.ravel(), b.ravel())
    ref = [R.two_point_phi(kind, delta, lam, int(x), int(y), alpha, rounding)
           for x, y in zip(a.ravel(), b.ravel())]
    assert got.tolist() == ref


@pytest.mark.parametrize("kind", KINDS)
def test_c_transfer_at_cfg2_scale(kind):
    # cfg2-like parameters, values up to the int32 state range of cfg2
    delta, lam = Fraction("1e-5"), Fraction(4, 15)
    t = oracle.TransferRule(kind, delta, lam, Fraction(3, 2))
    rng = np.random.default_rng(3)
    a = rng.integers(-150000, 150001, 400)
    b = rng.integers(-150000, 150001, 400)
    got = t.phi(a, b)
    ref = [R.two_point_phi(kind, delta, lam, int(x), int(y), Fraction(3, 2)) for x, y in zip(a, b)]
    assert got.tolist() == ref


def test_godunov_flux_textbook_cases():
    f = R.burgers_f
    F = lambda a, b: R.two_point_flux(R.BURGERS_GODUNOV, Fraction(a), Fraction(b))
    assert F(2, 1) == f(2)                 # right-moving shock: upwind from the left
    assert F(-1, -2) == f(-2)              # left-moving shock
    assert F(1, -3) == f(-3)               # transonic shock, speed -1 < 0
    assert F(3, -1) == f(3)                # transonic shock, speed 1 > 0
    assert F(-1, 2) == 0                   # transonic rarefaction: sonic point u = 0
    assert F(1, 2) == f(1) and F(-3, -1) == f(-1)
    for a in range(-6, 7):
        for b in range(-6, 7):
            A, B = Fraction(a, 3), Fraction(b, 3)
            # closed form for convex f with its minimum at 0 (independent of the Riemann code)
            assert F(A, B) == max(f(max(A, 0)), f(min(B, 0)))


@pytest.mark.parametrize("kind", KINDS)
def test_consistency(kind):
    delta, lam = Fraction(1, 10), Fraction(1, 2)
    t = _rule(kind, delta, lam)
    q = np.arange(-200, 201)
    ref = [R.round_rational(R.burgers_f(delta * int(x)) * lam / delta) for x in q]
    assert t.phi(q, q).tolist() == ref


def test_godunov_monotone_and_below_eo():
    g, e2 = _rule(R.BURGERS_GODUNOV), _rule(R.BURGERS_EO2)
    a, b = np.meshgrid(np.arange(-40, 41), np.arange(-40, 41), indexing="ij")
    G = g.phi(a.ravel(), b.ravel()).reshape(a.shape)
    E = e2.phi(a.ravel(), b.ravel()).reshape(a.shape)
    assert (np.diff(G, axis=0) >= 0).all()          # nondecreasing in qL
    assert (np.diff(G, axis=1) <= 0).all()          # nonincreasing in qR
    assert (G <= E).all()
    transonic = (a > 0) & (b < 0)
    assert (G[~transonic] == E[~transonic]).all()   # the two maps differ only there
    assert (G[transonic] != E[transonic]).any()


def test_eo2_vs_split_rule_rounding():
    # EO rounded once vs the paper's split rule (each half rounded): equal off
    # transonic pairs (one half vanishes), different on some transonic pairs
    e2 = _rule(R.BURGERS_EO2)
    sp = oracle.Rule(R.BURGERS_EO, "1/10", Fraction(1, 2))
    a, b = np.meshgrid(np.arange(-40, 41), np.arange(-40, 41), indexing="ij")
    E2 = e2.phi(a.ravel(), b.ravel())
    S = sp.interface_flux(a.ravel(), b.ravel())
    tr = ((a > 0) & (b < 0)).ravel()
    assert (E2[~tr] == S[~tr]).all() and (E2[tr] != S[tr]).any()


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("boundary", [oracle.PERIODIC, oracle.TRANSMISSIVE])
def test_conservation(kind, boundary):
    t = _rule(kind, "1e-3", Fraction(1, 2), Fraction(3, 2))
    rng = np.random.default_rng(kind)
    q = rng.integers(-1000, 1001, 301)
    for _ in range(40):
        qn = t.step(q, boundary)
        if boundary == oracle.PERIODIC:
            assert qn.sum() == q.sum()
        else:
            Tl = t.phi(q[0], q[0])[0]
            Tr = t.phi(q[-1], q[-1])[0]
            assert qn.sum() - q.sum() == Tl - Tr
        q = qn


def test_theorem_equal_maps_on_visited_states_give_equal_trajectories():
    """Thm P:274-280 on data whose visited pairs never are transonic (u > 0
    everywhere stays positive under Burgers): Godunov, EO rounded once and the
    split EO rule induce the same transfer on every visited state, so the
    checker reports no mismatch and the trajectories are identical."""
    delta, lam = "1e-4", Fraction(1, 3)
    n = 500
    x = W.cell_centres(n)
    q0 = W.quantise(0.6 + 0.3 * np.sin(2 * np.pi * x), 1e-4)
    g = oracle.TransferRule(R.BURGERS_GODUNOV, delta, lam)
    for other in (oracle.TransferRule(R.BURGERS_EO2, delta, lam),
                  oracle.TransferRule(R.BURGERS_EO, delta, lam)):
        qa, st = g.equivalence(other, q0, 300)
        assert st["mismatches"] == 0 and st["first_mismatch_step"] == -1
        assert st["interface_evals"] == 300 * n
        assert np.array_equal(qa, other.run(q0, 300))


def test_theorem_transonic_states_break_equivalence():
    # sign-changing data visits transonic compressive pairs: the maps differ there
    delta, lam = "1e-4", Fraction(1, 3)
    n = 400
    x = W.cell_centres(n)
    q0 = W.quantise(np.sin(2 * np.pi * x) * 0.8, 1e-4)
    g = oracle.TransferRule(R.BURGERS_GODUNOV, delta, lam)
    e2 = oracle.TransferRule(R.BURGERS_EO2, delta, lam)
    qa, st = g.equivalence(e2, q0, 400)
    assert st["mismatches"] > 0 and st["mismatched_pairs"] > 0
    assert not np.array_equal(qa, e2.run(q0, 400))


def test_checker_statistics_brute_force():
    delta, lam = "1/10", Fraction(1, 2)
    g = oracle.TransferRule(R.BURGERS_GODUNOV, delta, lam)
    lf = oracle.TransferRule(R.BURGERS_LF2, delta, lam, Fraction(2))
    q0 = np.array([7, -5, 3, 0, -2, 9, -9, 1], dtype=np.int64)
    for boundary in (oracle.PERIODIC, oracle.TRANSMISSIVE):
        _, st = g.equivalence(lf, q0, 6, boundary)
        # recount with plain Python loops and the literal Fraction definitions
        q = [int(v) for v in q0]
        N = len(q)
        evals = mism = 0
        first = -1
        seen, bad = set(), set()
        for s in range(6):
            ifs = range(N) if boundary == oracle.PERIODIC else range(-1, N)
            T = {}
            for i in ifs:
                iL, iR = i, i + 1
                if boundary == oracle.PERIODIC:
                    iR %= N
                else:
                    iL, iR = max(iL, 0), min(iR, N - 1)
                a, b = q[iL], q[iR]
                ta = R.two_point_phi(R.BURGERS_GODUNOV, delta, lam, a, b)
                tb = R.two_point_phi(R.BURGERS_LF2, delta, lam, a, b, Fraction(2))
                evals += 1
                seen.add((a, b))
                if ta != tb:
                    mism += 1
                    bad.add((a, b))
                    if first < 0:
                        first = s
                T[i] = ta
            if boundary == oracle.PERIODIC:
                T[-1] = T[N - 1]
            q = [q[i] - (T[i] - T[i - 1]) for i in range(N)]
        assert st == {"interface_evals": evals, "mismatches": mism, "first_mismatch_step": first,
                      "visited_pairs": len(seen), "mismatched_pairs": len(bad)}


def test_godunov_quantised_ladder():
    """Godunov-quantised FQNM vs the closed-form entropy solution of a Burgers
    top-hat (shock + rarefaction): exact conservation, L1 error decreasing with N."""
    delta, lam, T = 1e-9, Fraction(1, 2), 0.25
    g = oracle.TransferRule(R.BURGERS_GODUNOV, "1e-9", lam)
    errs = []
    for n_cells in (256, 1024, 4096):
        nsteps = int(T * n_cells / float(lam))
        x = W.cell_centres(n_cells)
        u0 = np.where((x >= 0.25) & (x < 0.75), 1.0, -0.5)
        q0 = W.quantise(u0, delta)
        q = g.run(q0, nsteps)
        assert q.sum() == q0.sum()
        errs.append(np.abs(delta * q - burgers_tophat_exact(x, T, -0.5, 1.0)).mean())
    assert errs[0] > errs[1] > errs[2] and errs[2] < 0.01
