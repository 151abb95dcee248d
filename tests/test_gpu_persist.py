"""K2P, the persistent temporally blocked stepper (all blocks of k steps in one launch,
(block, window) items claimed in order, acquire/release flags between the block b-1
windows covering an input window and the item): bit-exact against the oracle for the
fast rules, both boundaries, ragged sizes, several k and step counts (odd and even
block counts, short last blocks), repeated calls (monotone flag tags), and the auto
cfg3-sized problem equal to the launch-per-block K2.  (K2P is opt-in, kernel 12: it
measured slower than K2.)"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda"

RULES = [  # kind, delta, dt/dx, param, amplitude, offset  (-> rule id)
    (W.LINEAR, "1e-4", Fraction(1, 2), 1, 5000, 0),                 # LIN_HALF
    (W.BURGERS_EO, "1e-5", Fraction(4, 15), 1, 100000, 20000),      # EO_P1
    (W.BURGERS_EO, "1e-5", Fraction(3, 10), 1, 100000, 20000),      # EO_FAST (P = 3)
    (W.LINEAR, "1e-3", Fraction(1, 3), -1, 3000, 100),              # LIN_FAST, a < 0
]


@pytest.fixture(scope="module")
def F():
    import paper_2604_06947_b200 as F
    return F


@pytest.mark.parametrize("case", range(len(RULES)))
@pytest.mark.parametrize("boundary", [W.PERIODIC, W.TRANSMISSIVE])
@pytest.mark.parametrize("n,k,steps", [(50003, 24, 100), (50003, 7, 33), (4099, 16, 1), (1024, 8, 20),
                                       (200000, 32, 97), (1000, 4, 41),
                                       # last window shorter than k next to the periodic wrap
                                       # (V = 48 one-sided LIN: S = 1512; V = 32 two-sided: S = 976)
                                       (20 * 1512 + 2, 24, 100), (30 * 976 + 3, 24, 50)])
def test_persistent_matches_oracle(F, case, boundary, n, k, steps):
    kind, delta, lam, param, amp, off = RULES[case]
    rng = np.random.default_rng(n + k + case)
    q0 = np.clip(W.smooth_random(rng, n, amp, off), -amp, amp + off)
    rule = oracle.Rule(kind, delta, lam, Fraction(param))
    plan = F.fqnm_plan_ex(n, float(Fraction(delta)), float(lam), kind, boundary,
                          flux_param=float(param))
    try:
        F.fqnm_debug_override(plan, 12, k, 0)
    except F.FqnmError:
        pytest.skip("k too large for V = 32 with this dependence")
    q = torch.tensor(q0, dtype=torch.int32, device=DEV)
    ref = q0
    for _ in range(2):                         # two calls: flag tags carry over
        F.fqnm_step(plan, q, steps)
        ref = rule.run(ref, steps, boundary)
        assert np.array_equal(q.cpu().numpy().astype(np.int64), ref)


def test_persistent_on_cfg3_size_equals_k2(F):
    """On a cfg3-sized linear problem K2P (forced; not the default) equals the
    launch-per-block K2 bit for bit, in one launch for all 16 blocks."""
    n = 1 << 24
    q0 = torch.tensor(W.q0_cfg3(n), dtype=torch.int32, device=DEV)
    pp = F.fqnm_plan(n, 1e-6, 0.5, F.LINEAR, F.PERIODIC)
    F.fqnm_debug_override(pp, 12)
    k2 = F.fqnm_plan(n, 1e-6, 0.5, F.LINEAR, F.PERIODIC)
    a, b = q0.clone(), q0.clone()
    F.fqnm_profile_enable(pp, True)
    F.fqnm_step(pp, a, 1000)
    _, launches = F.fqnm_profile_read(pp)
    assert launches == 1
    F.fqnm_step(k2, b, 1000)
    assert torch.equal(a, b)
