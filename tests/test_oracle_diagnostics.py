"""Pins of oracle/diagnostics.py (SI "Entropy and Statistical Structure",
PAPER.md P:672-783) against things other than itself: Prop. S1(i)'s closed form,
scipy's Shannon entropy, pure-Python brute-force counting, the identities that
Def. S2 states for M^n (column-stochastic on occupied levels, row sums = c^{n+1}
/ c^n mixing, p^{n+1} = M^n p^n) on deliberately non-symmetric data (a
transposed M fails them), and Thm. S2 on constructed doubly stochastic mixing."""
import math
from collections import Counter
from fractions import Fraction

import numpy as np
import pytest
import scipy.stats

from oracle import diagnostics as D


def test_uniform_levels_closed_form():
    """Prop. S1(i): uniform on m occupied levels => S = log m, N_eff = m."""
    rng = np.random.default_rng(1)
    for m in (1, 2, 3, 7, 64, 1000):
        reps = int(rng.integers(1, 9))
        levels = rng.choice(np.arange(-5000, 5000), size=m, replace=False)
        q = rng.permutation(np.repeat(levels, reps))
        assert D.entropy(q) == pytest.approx(math.log(m), abs=1e-12)
        assert D.n_eff(q) == pytest.approx(m, rel=1e-12)


def test_constant_state_zero_entropy():
    for v in (-3, 0, 12345):
        q = np.full(517, v)
        assert D.entropy(q) == 0.0 and D.n_eff(q) == 1.0


def test_matches_scipy_entropy():
    rng = np.random.default_rng(2)
    for n in (10, 1000, 50000):
        q = rng.geometric(0.05, size=n) - 20
        _, c = np.unique(q, return_counts=True)
        assert D.entropy(q) == pytest.approx(scipy.stats.entropy(c), rel=1e-13)


def test_brute_force_counts():
    rng = np.random.default_rng(3)
    for _ in range(20):
        n = int(rng.integers(1, 40))
        q0 = rng.integers(-3, 4, size=n)
        q1 = q0 + rng.integers(-1, 2, size=n)
        brute = Counter()
        for i in range(n):
            brute[(int(q1[i]), int(q0[i]))] += 1        # N_{k'k}: k = q^n_i, k' = q^{n+1}_i
        assert D.transition_counts(q0, q1) == dict(brute)
        c = Counter(int(x) for x in q0)
        S = 0.0
        for k in c:
            pk = c[k] / n
            S -= pk * math.log(pk)
        assert D.entropy(q0) == pytest.approx(S, abs=1e-14)


def _random_step(rng, n):
    q0 = rng.integers(0, 9, size=n) ** 2 // 7            # skewed, non-symmetric levels
    q1 = q0 + rng.choice([-2, 0, 0, 1, 3], size=n)
    return q0, q1


def test_def_s2_identities():
    """Def. S2: sum_{k'} M_{k'k} = 1 where c_k > 0; sum_k N_{k'k} = c^{n+1}_{k'};
    p^{n+1} = M^n p^n (Eq. pn1_equals_Mpn)."""
    rng = np.random.default_rng(4)
    for n in (5, 100, 3000):
        q0, q1 = _random_step(rng, n)
        levels, M = D.transition_matrix(q0, q1)
        k0, c0 = D.level_counts(q0)
        k1, c1 = D.level_counts(q1)
        p0 = np.zeros(levels.size)
        p1 = np.zeros(levels.size)
        p0[np.searchsorted(levels, k0)] = c0 / n
        p1[np.searchsorted(levels, k1)] = c1 / n
        col = M.sum(axis=0)
        assert np.allclose(col[p0 > 0], 1.0, atol=1e-14)
        assert np.all(col[p0 == 0] == 0.0)
        assert np.allclose(M @ p0, p1, atol=1e-14)
        N = Counter()
        for (kp, k), v in D.transition_counts(q0, q1).items():
            N[kp] += v
        assert [N[int(k)] for k in k1] == c1.tolist()


def test_identity_and_level_permutation():
    """q^{n+1} = q^n => M = I, rho = 0, dS = 0; a permutation of the occupied
    levels onto themselves keeps rho = 0 and S (Thm. S2 equality case)."""
    rng = np.random.default_rng(5)
    q0 = rng.integers(-10, 11, size=2000)
    levels, M = D.transition_matrix(q0, q0)
    assert np.array_equal(M, np.eye(levels.size))
    assert D.row_sum_defect(q0, q0) == 0.0
    occ = np.unique(q0)
    sigma = dict(zip(occ.tolist(), rng.permutation(occ).tolist()))
    q1 = np.array([sigma[int(x)] for x in q0])
    assert D.row_sum_defect(q0, q1) == pytest.approx(0.0, abs=1e-15)
    assert D.entropy(q1) == pytest.approx(D.entropy(q0), abs=1e-13)


def test_defect_over_union_of_supports():
    """A17: a level that empties (in supp p^n only) has row sum 0 -> rho = 1."""
    q0 = np.array([0, 0, 1, 1])
    q1 = np.array([1, 1, 1, 1])
    assert D.row_sum_defect(q0, q1) == 1.0      # row 1: M_{1,0} + M_{1,1} = 2, row 0: 0
    q1 = np.array([1, 1, 0, 0])                   # swap: doubly stochastic
    assert D.row_sum_defect(q0, q1) == 0.0


def _doubly_stochastic_step(rng, m, D_, nperm):
    """Cells on m levels with c_k = D_ t_k moved by M = sum_j (a_j / D_) P_j."""
    a = rng.multinomial(D_ - nperm, np.ones(nperm) / nperm) + 1
    perms = [rng.permutation(m) for _ in range(nperm)]
    t = rng.integers(1, 5, size=m)
    levels = np.sort(rng.choice(np.arange(-300, 300), size=m, replace=False))
    q0, q1 = [], []
    for k in range(m):
        for j in range(nperm):
            cnt = int(a[j] * t[k])
            q0 += [levels[k]] * cnt
            q1 += [levels[perms[j][k]]] * cnt
    order = rng.permutation(len(q0))
    M = sum(Fraction(int(a[j]), D_) * np.eye(m, dtype=object)[perms[j]].T for j in range(nperm))
    return np.array(q0)[order], np.array(q1)[order], levels, M


def test_theorem_s2_doubly_stochastic_mixing():
    """Thm. S2: M^n doubly stochastic => S^{n+1} >= S^n, strict unless p^{n+1}
    is a permutation of p^n; the oracle recovers the constructed M exactly."""
    rng = np.random.default_rng(6)
    strict = 0
    for trial in range(40):
        m = int(rng.integers(2, 9))
        D_ = int(rng.integers(2, 7))
        q0, q1, levels, Mx = _doubly_stochastic_step(rng, m, D_, min(D_, int(rng.integers(1, 4))))
        lv, M = D.transition_matrix(q0, q1)
        assert np.array_equal(lv, levels)
        assert np.allclose(M, np.array(Mx, dtype=float), atol=1e-15)
        assert D.row_sum_defect(q0, q1) <= 1e-15
        S0, S1 = D.entropy(q0), D.entropy(q1)
        p0 = np.sort(D.level_distribution(q0)[1])
        p1 = np.sort(D.level_distribution(q1)[1])
        if p0.size == p1.size and np.allclose(p0, p1, atol=1e-15):
            assert S1 == pytest.approx(S0, abs=1e-13)
        else:
            assert S1 > S0 + 1e-12
            strict += 1
    assert strict >= 10


def test_theorem_s2_worked_example():
    """c = (4, 2) mixed by M = [[1/2, 1/2], [1/2, 1/2]] -> c' = (3, 3):
    S goes from H(2/3) to log 2 (hand computation)."""
    q0 = np.array([0, 0, 0, 0, 1, 1])
    q1 = np.array([0, 0, 1, 1, 0, 1])
    assert D.transition_counts(q0, q1) == {(0, 0): 2, (1, 0): 2, (0, 1): 1, (1, 1): 1}
    assert D.row_sum_defect(q0, q1) == 0.0
    assert D.entropy(q0) == pytest.approx(-(2 / 3) * math.log(2 / 3) - (1 / 3) * math.log(1 / 3))
    assert D.entropy(q1) == pytest.approx(math.log(2))
    assert D.entropy_rate(q0, q1, 0.5) == pytest.approx(2 * (D.entropy(q1) - D.entropy(q0)))


def test_fqnm_dynamics_bistochastic_steps_do_not_lower_entropy():
    """On actual quantised Burgers steps (oracle), every step whose M^n is
    exactly doubly stochastic has S^{n+1} >= S^n (Thm. S2); M^n stays
    column-stochastic throughout."""
    import oracle
    import workloads as W
    w = W.cfg("cfg2")
    n = 512
    rng = np.random.default_rng(7)
    q = W.smooth_random(rng, n, 3000, 500)
    lam = W.dt_dx(w, int(np.abs(q).max()))
    rule = oracle.Rule(oracle.BURGERS_EO, "1e-5", lam)
    for _ in range(60):
        q1 = rule.step(q)
        levels, M = D.transition_matrix(q, q1)
        assert np.allclose(M.sum(axis=0)[M.sum(axis=0) > 0], 1.0)
        if D.row_sum_defect(q, q1) == 0.0:
            assert D.entropy(q1) >= D.entropy(q) - 1e-13
        q = q1
