"""Oracle vs the paper's convergence theory (Thm consistency P:243-250,
Thm convergence) on closed-form Burgers Riemann solutions.

Rigorous bound used: with v^n the real-arithmetic split
scheme from u0 (computed in float64), Prop. 1 (<= 2 delta per cell and step)
and the l1 contraction of the monotone real scheme (Lemma P:213-218, periodic)
give

    ||delta q^n - u_ex||_L1 <= ||v^n - u_ex||_L1 + delta/2 + 2 n delta.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle.reference import burgers_tophat_exact, classical_step
from oracle.rules import BURGERS_EO
import workloads as W


@pytest.mark.parametrize("u_lo,u_hi", [(0.0, 1.0), (-0.5, 1.0)])
def test_burgers_riemann_ladder(u_lo, u_hi):
    delta = 1e-9
    lam = Fraction(1, 2)              # alpha = max|u| = 1, nu = 1/2
    T = 0.25
    r = oracle.Rule(BURGERS_EO, "1e-9", lam)
    errs_q, errs_v = [], []
    for n_cells in (256, 1024, 4096):
        nsteps = int(T * n_cells / float(lam))
        x = W.cell_centres(n_cells)
        u0 = np.where((x >= 0.25) & (x < 0.75), u_hi, u_lo)
        q = r.run(W.quantise(u0, delta), nsteps)
        v = u0.copy()
        for _ in range(nsteps):
            v = classical_step(v, BURGERS_EO, float(lam))
        ue = burgers_tophat_exact(x, T, u_lo, u_hi)
        eq = np.abs(delta * q - ue).mean()
        ev = np.abs(v - ue).mean()
        assert eq <= ev + delta / 2 + 2 * nsteps * delta + 1e-12
        assert int(q.sum()) == int(W.quantise(u0, delta).sum())       # exact conservation
        errs_q.append(eq)
        errs_v.append(ev)
    assert errs_v[0] > errs_v[1] > errs_v[2]
    assert errs_q[0] > errs_q[1] > errs_q[2]
    assert errs_q[2] < 0.01


def test_burgers_coarse_delta_stays_within_bound():
    # with a coarse quantum the O(delta) term is visible but still bounded
    delta = 1e-3
    lam = Fraction(1, 2)
    r = oracle.Rule(BURGERS_EO, "1e-3", lam)
    n_cells, T = 512, 0.25
    nsteps = int(T * n_cells / float(lam))
    x = W.cell_centres(n_cells)
    u0 = np.where((x >= 0.25) & (x < 0.75), 1.0, -0.5)
    q = r.run(W.quantise(u0, delta), nsteps)
    v = u0.copy()
    for _ in range(nsteps):
        v = classical_step(v, BURGERS_EO, float(lam))
    ue = burgers_tophat_exact(x, T, -0.5, 1.0)
    assert np.abs(delta * q - ue).mean() <= np.abs(v - ue).mean() + delta / 2 + 2 * nsteps * delta


def test_exact_tophat_solution_is_weak_solution():
    # pin the closed form itself: mass conservation and the Rankine-Hugoniot shock speed
    x = W.cell_centres(1 << 16)
    for t in (0.05, 0.2, 0.3):
        u = burgers_tophat_exact(x, t, -0.5, 1.0)
        assert abs(u.mean() - (0.5 * 1.0 + 0.5 * -0.5)) < 1e-4
        # shock located at 0.75 + t (u_lo + u_hi)/2
        s = 0.75 + 0.25 * t
        i = int(s * len(x))
        assert u[i - 2] == 1.0 and u[i + 2] == -0.5
