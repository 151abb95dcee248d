"""2D/3D range guard: the unsplit directional composition (Thm P:364-401) is
not monotone once quantised, so a state inside the plan's admissible range can step
outside it.  A checkerboard of H (odd) and H - 1 under LINEAR with kappa = 1/2 in every
direction gives the H - 1 cells H - 1 - d (H - 1)/2 + d (H + 1)/2 = H + d - 1 > H after
one step (phi+(q) = ceil(q/2) for q > 0; 2D uses kappa = 9/20, where the same pattern at
the range edge also overshoots).  With H = q_hi the state leaves [q_lo, q_hi]:
fqnm_step must report FQNM_ERR_RANGE instead of stepping on with maps outside their
proven domain; the same pattern one level lower stays in range and matches the oracle."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def F():
    import paper_2604_06947_b200 as F
    return F


def _checker(shape, H):
    idx = np.indices(shape).sum(axis=0)
    return np.where(idx % 2 == 0, H, H - 1).astype(np.int64)


# 2D: kappa = 9/20 per direction (the LIN_HALF range edge of 2D cannot be left upward
# by one step, the R_LIN_FAST edge at 9/20 can); 3D: kappa = 1/2 (LIN_HALF)
LAM = {2: Fraction(9, 20), 3: Fraction(1, 2)}


def _plan(F, shape):
    lam = float(LAM[len(shape)])
    if len(shape) == 2:
        ny, nx = shape
        return F.fqnm_plan_2d(nx, ny, 1e-3, lam, lam, F.LINEAR, F.PERIODIC)
    nz, ny, nx = shape
    return F.fqnm_plan_3d(nx, ny, nz, 1e-3, lam, lam, lam, F.LINEAR, F.PERIODIC)


def _oracle(shape):
    h = LAM[len(shape)]
    if len(shape) == 2:
        return oracle.Rule2D(W.LINEAR, "1e-3", h, h)
    return oracle.Rule3D(W.LINEAR, "1e-3", h, h, h)


@pytest.mark.parametrize("shape,kernel", [((64, 256), 0), ((64, 256), 7), ((33, 130), 0),
                                          ((8, 16, 128), 0), ((8, 16, 128), 10)])
@pytest.mark.parametrize("nsteps", [1, 3, 20])
def test_md_state_leaving_range_is_reported(F, shape, kernel, nsteps):
    plan = _plan(F, shape)
    if kernel:
        F.fqnm_debug_override(plan, kernel, 0, 0)
    hi = plan.info()["q_hi"]
    assert hi <= (2**31 - 1) // (1 + 4 * len(shape))      # multi-D clamp: no int32 wrap
    qh = _checker(shape, hi)
    assert _oracle(shape).step(qh).max() > hi            # the pattern leaves the range
    q = torch.tensor(qh, dtype=torch.int32, device=DEV)
    with pytest.raises(F.FqnmError) as e:
        F.fqnm_step(plan, q, nsteps)
    assert e.value.status == 3
    # the plan stays usable: in-range data steps exactly afterwards
    q0 = _checker(shape, 1001)
    q = torch.tensor(q0, dtype=torch.int32, device=DEV)
    F.fqnm_step(plan, q, nsteps)
    assert np.array_equal(q.cpu().numpy().astype(np.int64), _oracle(shape).run(q0, nsteps))


@pytest.mark.parametrize("shape", [(64, 256), (8, 16, 128)])
def test_md_overshoot_inside_range_is_exact(F, shape):
    """The same non-monotone overshoot well inside the range is not an error: exact."""
    plan = _plan(F, shape)
    q0 = _checker(shape, 99999)
    q = torch.tensor(q0, dtype=torch.int32, device=DEV)
    F.fqnm_step(plan, q, 17)
    ref = _oracle(shape).run(q0, 17)
    assert ref.max() > q0.max()                         # the maximum principle fails here
    assert np.array_equal(q.cpu().numpy().astype(np.int64), ref)
