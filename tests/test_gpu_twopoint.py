"""GPU parity of the quantised two-point transfer rules and of the transfer-operator
equivalence checker (Thm P:262-280) against the oracle (oracle.TransferRule).

* the kernels' own interface-transfer code (fqnm_transfer2_device) over a grid of
  interface states, bit-exact, for the three two-point kinds and the split kinds;
* stepping parity for every kernel family (naive, blocked V = 8/16, warp ensemble,
  CTA ensemble, resident), both boundaries, ragged sizes;
* fqnm_equivalence statistics (mismatch count, first step, distinct visited and
  mismatching pairs) equal to the oracle's plain recount, and the theorem's
  conclusion on the GPU (no mismatch -> identical trajectories).
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda"

# (kind, delta, dt/dx, alpha, amplitude of the test data)
TP = [
    (oracle.BURGERS_GODUNOV, "1e-5", Fraction(4, 15), 1, 100000),
    (oracle.BURGERS_EO2, "1e-5", Fraction(4, 15), 1, 100000),
    (oracle.BURGERS_LF2, "1e-3", Fraction(1, 2), 1, 900),
]


@pytest.fixture(scope="module")
def F():
    import paper_2604_06947_b200 as F
    return F


def _plan(F, kind, delta, lam, alpha, n, boundary=W.PERIODIC, **kw):
    return F.fqnm_plan_ex(n, float(Fraction(delta)), float(lam), kind, boundary,
                          flux_param=float(alpha), **kw)


@pytest.mark.parametrize("case", range(len(TP)))
def test_transfer2_device_grid(F, case):
    kind, delta, lam, alpha, amp = TP[case]
    plan = _plan(F, kind, delta, lam, alpha, 1024)
    rng = np.random.default_rng(case)
    a = np.concatenate([np.repeat(np.arange(-60, 61), 121), rng.integers(-amp, amp + 1, 200000)])
    b = np.concatenate([np.tile(np.arange(-60, 61), 121), rng.integers(-amp, amp + 1, 200000)])
    T = F.fqnm_transfer2_device(plan, torch.tensor(a, dtype=torch.int32, device=DEV),
                                torch.tensor(b, dtype=torch.int32, device=DEV))
    ref = oracle.TransferRule(kind, delta, lam, alpha).phi(a, b)
    assert np.array_equal(T.cpu().numpy().astype(np.int64), ref)
    for x, y in ((5, -7), (-3, 3), (0, 0), (amp, -amp)):
        assert F.fqnm_transfer2(plan, x, y) == int(oracle.TransferRule(kind, delta, lam, alpha).phi(x, y)[0])
    with pytest.raises(F.FqnmError):
        F.fqnm_transfer(plan, 3)                  # no split maps for a two-point rule


@pytest.mark.parametrize("kind,delta,lam,alpha", [
    (oracle.BURGERS_EO, "1e-5", Fraction(4, 15), 1),      # R_EO_P1
    (oracle.BURGERS_EO, "1e-5", Fraction(3, 10), 1),      # R_EO_FAST (P = 3)
    (oracle.LINEAR, "1e-4", Fraction(1, 2), 1),           # R_LIN_HALF
    (oracle.BURGERS_LF, "1e-3", Fraction(1, 2), 1),       # generic
])
def test_transfer2_device_split_rules(F, kind, delta, lam, alpha):
    plan = _plan(F, kind, delta, lam, alpha, 1024)
    rng = np.random.default_rng(7)
    a = rng.integers(-900, 901, 50000)
    b = rng.integers(-900, 901, 50000)
    T = F.fqnm_transfer2_device(plan, torch.tensor(a, dtype=torch.int32, device=DEV),
                                torch.tensor(b, dtype=torch.int32, device=DEV))
    ref = oracle.TransferRule(kind, delta, lam, alpha).phi(a, b)
    assert np.array_equal(T.cpu().numpy().astype(np.int64), ref)


@pytest.mark.parametrize("case", range(len(TP)))
@pytest.mark.parametrize("boundary", [W.PERIODIC, W.TRANSMISSIVE])
@pytest.mark.parametrize("n", [3, 64, 1000, 1024, 20000, 65536 + 129])
def test_two_point_stepping_all_families(F, case, boundary, n):
    kind, delta, lam, alpha, amp = TP[case]
    rng = np.random.default_rng(31 * n + case)
    q0 = np.clip(W.smooth_random(rng, n, amp, amp // 5), -amp, amp)
    rule = oracle.TransferRule(kind, delta, lam, alpha)
    for nsteps in (1, 7, 40):
        ref = rule.run(q0, nsteps, boundary)
        fams = [(0, 0), (1, 0)]
        if n >= 64:
            fams += [(2, 8), (2, 16), (6, 0)]
        if n <= 16384:
            fams.append((4, 0))
        if n % 32 == 0 and n // 32 in (1, 2, 4, 8, 16, 32):
            fams.append((3, 0))
        for fam, V in fams:
            plan = _plan(F, kind, delta, lam, alpha, n, boundary)
            if fam:
                F.fqnm_debug_override(plan, fam)
            if V:
                F.fqnm_debug_override(plan, 0, 0, V)
            q = torch.tensor(q0, dtype=torch.int32, device=DEV)
            F.fqnm_step(plan, q, nsteps)
            assert np.array_equal(q.cpu().numpy().astype(np.int64), ref), (fam, V, nsteps)


@pytest.mark.parametrize("pair", [
    (oracle.BURGERS_GODUNOV, oracle.BURGERS_EO2),
    (oracle.BURGERS_GODUNOV, oracle.BURGERS_EO),
    (oracle.BURGERS_EO2, oracle.BURGERS_EO),
    (oracle.BURGERS_EO, oracle.BURGERS_GODUNOV),
])
@pytest.mark.parametrize("boundary", [W.PERIODIC, W.TRANSMISSIVE])
def test_equivalence_checker_matches_oracle(F, pair, boundary):
    ka, kb = pair
    delta, lam = "1e-4", Fraction(1, 3)
    n, nsteps = 777, 700                 # t = 0.3: past shock formation (t* = 0.2)
    x = W.cell_centres(n)
    q0 = W.quantise(0.8 * np.sin(2 * np.pi * x) + 0.1, 1e-4)
    ra, rb = oracle.TransferRule(ka, delta, lam), oracle.TransferRule(kb, delta, lam)
    q_ref, st_ref = ra.equivalence(rb, q0, nsteps, boundary)
    pa = _plan(F, ka, delta, lam, 1, n, boundary)
    pb = _plan(F, kb, delta, lam, 1, n, boundary)
    q = torch.tensor(q0, dtype=torch.int32, device=DEV)
    st = F.fqnm_equivalence(pa, pb, q, nsteps, pair_capacity=1 << 20)
    assert np.array_equal(q.cpu().numpy().astype(np.int64), q_ref)
    assert st["overflow"] == 0
    got = {k: st[k] for k in st_ref}
    assert got == st_ref
    assert st_ref["mismatches"] > 0


def test_equivalence_theorem_on_gpu(F):
    """Positive data never visits a transonic pair: Godunov, EO rounded once and the
    split EO rule agree on every visited state, so their GPU trajectories coincide."""
    delta, lam = "1e-5", Fraction(4, 15)
    n, nsteps = 65536, 3000
    q0 = W.quantise(1.0 + 0.4 * np.sin(2 * np.pi * W.cell_centres(n)), 1e-5)
    plans = {k: _plan(F, k, delta, lam, 1, n) for k in
             (oracle.BURGERS_GODUNOV, oracle.BURGERS_EO2, oracle.BURGERS_EO)}
    q = torch.tensor(q0, dtype=torch.int32, device=DEV)
    st = F.fqnm_equivalence(plans[oracle.BURGERS_GODUNOV], plans[oracle.BURGERS_EO2], q, nsteps)
    assert st["mismatches"] == 0 and st["first_mismatch_step"] == -1
    assert st["visited_pairs"] == -1                     # pair tracking off
    outs = []
    for k, p in plans.items():
        qq = torch.tensor(q0, dtype=torch.int32, device=DEV)
        F.fqnm_step(p, qq, nsteps)
        outs.append(qq.cpu().numpy())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    assert np.array_equal(outs[0], q.cpu().numpy())


def test_equivalence_argument_checks(F):
    pa = _plan(F, oracle.BURGERS_GODUNOV, "1e-4", Fraction(1, 3), 1, 100)
    pb = _plan(F, oracle.BURGERS_EO, "1e-4", Fraction(1, 3), 1, 101)
    q = torch.zeros(100, dtype=torch.int32, device=DEV)
    with pytest.raises(F.FqnmError):
        F.fqnm_equivalence(pa, pb, q, 3)
    pc = _plan(F, oracle.BURGERS_EO, "1e-4", Fraction(1, 3), 1, 100, W.TRANSMISSIVE)
    with pytest.raises(F.FqnmError):
        F.fqnm_equivalence(pa, pc, q, 3)


@pytest.mark.parametrize("lam", [Fraction(4, 15), Fraction(3, 10)])          # P = 1 and general P
@pytest.mark.parametrize("sign", [1, -1, 0])
@pytest.mark.parametrize("fam,n", [(2, 300_007), (6, 65_536 + 77)])
def test_godunov_sign_uniform_windows_take_the_eo_step(F, lam, sign, fam, n):
    """Godunov fast rule (R_TP_FAST) in K2 (V = 32) and K6: windows whose cells are all >= 0
    or all <= 0 (zeros included) step with the EO sign-uniform form, the rest with the
    two-point evaluation; bit-exact against the oracle's Godunov rule on positive, negative
    and patchwise mixed data, both boundaries."""
    rng = np.random.default_rng(1000 * fam + n + sign)
    q0 = np.abs(W.smooth_random(rng, n, 100000, 30000)) + 1
    q0[rng.integers(0, n, 200)] = 0
    if sign < 0:
        q0 = -q0
    elif sign == 0:
        q0[n // 4: n // 2] *= -1                       # patches of each sign, two sign changes
        q0[7 * n // 8:] *= -1
    rule = oracle.TransferRule(oracle.BURGERS_GODUNOV, "1e-5", lam)
    for boundary in (W.PERIODIC, W.TRANSMISSIVE):
        plan = _plan(F, oracle.BURGERS_GODUNOV, "1e-5", lam, 1, n, boundary)
        assert plan.info()["rule"] == 7                 # R_TP_FAST
        F.fqnm_debug_override(plan, fam)
        q = torch.tensor(q0, dtype=torch.int32, device=DEV)
        F.fqnm_step(plan, q, 61)
        assert np.array_equal(q.cpu().numpy().astype(np.int64), rule.run(q0, 61, boundary)), boundary
