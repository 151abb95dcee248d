"""GPU parity of the level-space diagnostics (SI P:672-783):
fqnm_levels / fqnm_transitions (CUDA, through the C ABI) against
oracle/diagnostics.py on the same seeded states.  Integer outputs (counts,
occupied levels, non-zero transitions, outside cells) are bit-exact; S, N_eff
and rho are float64 reductions in a different order: |err| <= 1e-12 relative
for S (each c log c term carries <= 2 ulp, the sum <= L terms) and 1e-12
absolute for rho (row sums of <= L fractions <= 1).  All states come from the
oracle (workloads + oracle stepping), never from the CUDA path."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads as W
from oracle import diagnostics as D

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2604_06947_b200 as F
    F._load()
    return F


def _check_levels(got, q, lo, hi):
    q = np.asarray(q).ravel()
    inside = q[(q >= lo) & (q <= hi)]
    assert got["outside"] == q.size - inside.size
    if inside.size == 0:
        assert got["occupied"] == 0 and got["S"] == 0.0
        return
    S = D.entropy(inside)
    assert got["occupied"] == D.level_counts(inside)[0].size
    assert got["S"] == pytest.approx(S, rel=1e-12, abs=1e-13)
    assert got["N_eff"] == pytest.approx(np.exp(S), rel=1e-12)


def _check_transitions(got, q0, q1):
    _check_levels(got["before"], q0, -(1 << 62), 1 << 62)
    _check_levels(got["after"], q1, -(1 << 62), 1 << 62)
    assert got["overflow"] == 0
    assert got["nonzeros"] == len(D.transition_counts(q0, q1))
    assert got["rho"] == pytest.approx(D.row_sum_defect(q0, q1), abs=1e-12)
    assert got["dS"] == pytest.approx(D.entropy(q1) - D.entropy(q0), abs=1e-12)


def _burgers_pair(n, seed, steps=1):
    rng = np.random.default_rng(seed)
    q = W.smooth_random(rng, n, 3000, 500)
    lam = W.dt_dx(W.cfg("cfg2"), int(np.abs(q).max()))
    rule = oracle.Rule(oracle.BURGERS_EO, "1e-5", lam)
    q0 = rule.run(q, 40)                    # past the first steepening
    return q0, rule.run(q0, steps), lam


@pytest.mark.parametrize("n", [2, 33, 1000, 100003])
def test_levels_counts_exact(F, n):
    rng = np.random.default_rng(n)
    q = rng.integers(-700, 900, size=n)
    lo, hi = int(q.min()), int(q.max())
    plan = F.fqnm_plan(n, 1e-4, 0.5, F.LINEAR, F.PERIODIC)
    counts = torch.zeros(hi - lo + 1, dtype=torch.int32, device=DEV)
    got = F.fqnm_levels(plan, torch.tensor(q, dtype=torch.int32, device=DEV), lo, hi, counts)
    _check_levels(got, q, lo, hi)
    ref = np.zeros(hi - lo + 1, dtype=np.int64)
    k, c = D.level_counts(q)
    ref[k - lo] = c
    assert np.array_equal(counts.cpu().numpy().astype(np.int64), ref)


def test_levels_window_and_outside(F):
    rng = np.random.default_rng(9)
    n = 50001
    q = rng.integers(-100, 100, size=n)
    plan = F.fqnm_plan(n, 1e-4, 0.5, F.LINEAR, F.PERIODIC)
    qd = torch.tensor(q, dtype=torch.int32, device=DEV)
    for lo, hi in [(-100, 99), (-20, 30), (0, 0), (500, 600)]:
        _check_levels(F.fqnm_levels(plan, qd, lo, hi), q, lo, hi)


@pytest.mark.parametrize("n,steps", [(512, 1), (4099, 1), (4099, 25), (262147, 1)])
def test_transitions_burgers_step(F, n, steps):
    q0, q1, lam = _burgers_pair(n, n, steps)
    plan = F.fqnm_plan(n, 1e-5, float(lam), F.BURGERS_EO, F.PERIODIC)
    lo = int(min(q0.min(), q1.min()))
    hi = int(max(q0.max(), q1.max()))
    got = F.fqnm_transitions(plan, torch.tensor(q0, dtype=torch.int32, device=DEV),
                             torch.tensor(q1, dtype=torch.int32, device=DEV), lo, hi)
    _check_transitions(got, q0, q1)


def test_transitions_entropy_trace_cfg2(F):
    """The paper's Burgers measurement: S^n and rho^n along a run,
    one (q^n, q^{n+1}) pair per step, all computed on the GPU."""
    w = W.cfg("cfg2")
    q = W.q0_cfg2()
    qmax = int(np.abs(q).max())
    lam = W.dt_dx(w, qmax)
    rule = oracle.Rule(oracle.BURGERS_EO, w.delta, lam)
    plan = F.fqnm_plan(w.n, float(w.delta), W.dt_dx_double(w, qmax), F.BURGERS_EO, F.PERIODIC)
    q = rule.run(q, 3000)
    for _ in range(4):
        q1 = rule.run(q, 250)
        lo, hi = int(min(q.min(), q1.min())), int(max(q.max(), q1.max()))
        got = F.fqnm_transitions(plan, torch.tensor(q, dtype=torch.int32, device=DEV),
                                 torch.tensor(q1, dtype=torch.int32, device=DEV), lo, hi)
        _check_transitions(got, q, q1)
        q = q1


def test_transitions_doubly_stochastic(F):
    """Constructed doubly stochastic mixing: rho == 0 on the GPU too, dS > 0."""
    rng = np.random.default_rng(12)
    m, reps = 37, 64
    levels = np.arange(-18, 19)
    q0 = np.repeat(levels, reps * (1 + np.arange(m) % 3))
    perm = rng.permutation(m)
    # half of each level's cells stay, half move to perm(level): M = (I + P) / 2
    q1 = q0.copy()
    for j, k in enumerate(levels):
        idx = np.flatnonzero(q0 == k)
        q1[idx[: idx.size // 2]] = levels[perm[j]]
    order = rng.permutation(q0.size)
    q0, q1 = q0[order], q1[order]
    plan = F.fqnm_plan(q0.size, 1e-4, 0.5, F.LINEAR, F.PERIODIC)
    got = F.fqnm_transitions(plan, torch.tensor(q0, dtype=torch.int32, device=DEV),
                             torch.tensor(q1, dtype=torch.int32, device=DEV), -18, 18)
    _check_transitions(got, q0, q1)
    assert got["rho"] <= 1e-15 and got["dS"] > 0


def test_levels_euler_density_channel(F):
    """Euler plans: the level channel is the integer density component."""
    n = 4096
    nsteps, lam5 = W.sod_steps_and_dt_dx(n)
    q0 = W.sod_q0(n)
    q1 = oracle.euler_run(q0, 30, 1e-7, lam5)
    plan = F.fqnm_plan(n, 1e-7, lam5, F.EULER_ROE, F.TRANSMISSIVE)
    r0, r1 = q0.reshape(3, n)[0], q1.reshape(3, n)[0]
    lo, hi = int(min(r0.min(), r1.min())), int(max(r0.max(), r1.max()))
    got = F.fqnm_transitions(plan, torch.tensor(q0, dtype=torch.int64, device=DEV),
                             torch.tensor(q1, dtype=torch.int64, device=DEV), lo, hi)
    _check_transitions(got, r0, r1)


def test_diagnostics_errors(F):
    plan = F.fqnm_plan(64, 1e-4, 0.5, F.LINEAR, F.PERIODIC)
    q = torch.zeros(64, dtype=torch.int32, device=DEV)
    with pytest.raises(F.FqnmError):
        F.fqnm_levels(plan, q, 5, 4)
    with pytest.raises(F.FqnmError):
        F.fqnm_levels(plan, q, 0, 1 << 31)
