"""GPU parity of the 3D directional composition (K8 and K10, fqnm_plan_3d; Thm P:364-401,
d = 3) against the 3D oracle (oracle.Rule3D), bit-exact: several rules (same and
different per-direction maps, LIN_HALF / EO P = 1 / generic paths), both boundaries,
ragged shapes smaller and larger than one 32 x 8 tile, several step counts; plus
the plan's observe/levels on a 3D state and its argument checks."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda"

RULES3D = [  # kind, delta, (dt/dx, dt/dy, dt/dz), (ax, ay, az), amplitude, offset
    (W.LINEAR, "1e-3", (Fraction(1, 2), Fraction(1, 2), Fraction(1, 2)), (1, 1, 1), 3000, 0),
    (W.LINEAR, "1e-3", (Fraction(1, 4), Fraction(1, 5), Fraction(1, 7)), (-1, 1, -1), 3000, 100),
    (W.BURGERS_EO, "1e-5", (Fraction(1, 15), Fraction(1, 15), Fraction(1, 15)), (1, 1, 1), 100000, 20000),
    (W.BURGERS_EO, "1e-5", (Fraction(1, 15), Fraction(1, 10), Fraction(1, 12)), (1, 1, 1), 100000, 20000),
    (W.BURGERS_LF, "1e-3", (Fraction(1, 6), Fraction(1, 6), Fraction(1, 6)), (1, 1, 1), 900, 0),
]


@pytest.fixture(scope="module")
def F():
    import paper_2604_06947_b200 as F
    return F


def _field(rng, nz, ny, nx, amp, off):
    x = W.cell_centres(nx)[None, None, :]
    y = W.cell_centres(ny)[None, :, None]
    z = W.cell_centres(nz)[:, None, None]
    u = off + amp * 0.5 * (np.sin(2 * np.pi * x + rng.uniform(0, 6)) *
                           np.cos(2 * np.pi * 2 * y + rng.uniform(0, 6)) *
                           np.cos(2 * np.pi * z + rng.uniform(0, 6)))
    return (np.rint(u) + rng.integers(-amp // 50, amp // 50 + 1, (nz, ny, nx))).astype(np.int64)


def _plan(F, case, shape, boundary):
    kind, d, lams, params, amp, off = RULES3D[case]
    nz, ny, nx = shape
    return F.fqnm_plan_3d(nx, ny, nz, float(Fraction(d)), *(float(l) for l in lams), kind,
                          boundary, tuple(float(p) for p in params))


@pytest.mark.parametrize("case", range(len(RULES3D)))
@pytest.mark.parametrize("boundary", [W.PERIODIC, W.TRANSMISSIVE])
@pytest.mark.parametrize("shape", [(2, 3, 5), (7, 9, 33), (19, 17, 70), (40, 24, 64), (5, 11, 260),
                                   (3, 9, 256), (4, 8, 130)])
def test_3d_matches_oracle(F, case, boundary, shape):
    kind, d, lams, params, amp, off = RULES3D[case]
    rng = np.random.default_rng(sum(shape) * 11 + case)
    q0 = _field(rng, *shape, amp, off)
    r = oracle.Rule3D(kind, d, *lams, params=params)
    for nsteps in (1, 4, 11):
        ref = r.run(q0, nsteps, boundary)
        for kern in (0, 8, 10):                    # default, K8 CTA tiles, K10 warp streaming
            plan = _plan(F, case, shape, boundary)
            assert plan.info()["kernel"] == 8
            if kern:
                F.fqnm_debug_override(plan, kern)
            q = torch.tensor(q0, dtype=torch.int32, device=DEV)
            F.fqnm_step(plan, q, nsteps)
            assert np.array_equal(q.cpu().numpy().astype(np.int64), ref), (nsteps, kern)


def test_3d_large_sampled(F):
    """64 x 96 x 128 EO (P = 1), 20 steps, every cell against the oracle; observe and
    level statistics of the 3D state."""
    case = 2
    kind, d, lams, params, amp, off = RULES3D[case]
    shape = (64, 96, 128)
    q0 = _field(np.random.default_rng(5), *shape, amp, off)
    plan = _plan(F, case, shape, W.PERIODIC)
    q = torch.tensor(q0, dtype=torch.int32, device=DEV)
    F.fqnm_step(plan, q, 20)
    ref = oracle.Rule3D(kind, d, *lams, params=params).run(q0, 20)
    assert np.array_equal(q.cpu().numpy().astype(np.int64), ref)
    assert int(q.to(torch.int64).sum()) == int(q0.sum())
    u = F.fqnm_observe(plan, q).cpu().numpy()
    assert np.array_equal(u.ravel(), oracle.observe(ref, 1e-5))
    lv = F.fqnm_levels(plan, q, int(ref.min()), int(ref.max()))
    assert lv["occupied"] == len(np.unique(ref)) and lv["outside"] == 0


def test_3d_argument_checks(F):
    with pytest.raises(F.FqnmError):
        F.fqnm_plan_3d(1, 4, 4, 1e-3, 0.5, 0.5, 0.5)                    # nx < 2
    with pytest.raises(F.FqnmError):
        F.fqnm_plan_3d(4, 4, 4, 1e-3, 0.5, 0.5, 0.5, F.BURGERS_GODUNOV)  # two-point kind
    with pytest.raises(F.FqnmError):
        F.fqnm_plan_3d(4, 4, 4, 1e-3, 1.5, 0.5, 0.5)                    # D8 fails in x
    plan = F.fqnm_plan_3d(4, 4, 4, 1e-3, 0.5, 0.5, 0.5)
    with pytest.raises(F.FqnmError):
        F.fqnm_debug_override(plan, 2)


@pytest.mark.parametrize("case", [1, 3])
@pytest.mark.parametrize("boundary", [W.PERIODIC, W.TRANSMISSIVE])
def test_3d_many_z_chunks(F, case, boundary):
    """A deep z extent (several equal z chunks per tile column, step3d_zchunk) with a
    partial last tile column in x and a partial last tile row in y, against the oracle."""
    kind, d, lams, params, amp, off = RULES3D[case]
    shape = (150, 17, 130)
    q0 = _field(np.random.default_rng(77 + case), *shape, amp, off)
    ref = oracle.Rule3D(kind, d, *lams, params=params).run(q0, 3, boundary)
    plan = _plan(F, case, shape, boundary)
    q = torch.tensor(q0, dtype=torch.int32, device=DEV)
    F.fqnm_step(plan, q, 3)
    assert np.array_equal(q.cpu().numpy().astype(np.int64), ref)
