"""Out-of-bounds write detection without compute-sanitizer (closed on this GPU pool):
every stepping-kernel family runs on a state that is a view into a larger device
buffer whose guard bands hold a canary pattern.  After the call the guard bands must be
intact and the state must equal the oracle's, bit for bit (K2 incl.
the p2p virtual ranks, K6, K2P, K8, K9, plus K1, K3, K4, K5, K7, K10).  Ragged sizes put
the last window / tile / chunk against the band."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
DEV = "cuda"
BAND = 4096
CANARY = -0x5A5A5A5B


@pytest.fixture(scope="module")
def F():
    import paper_2604_06947_b200 as F
    return F


def banded(q0, dtype=torch.int32):
    """(buffer, view): the view holds q0 (flattened), BAND canary elements each side."""
    q0 = np.ascontiguousarray(q0).reshape(-1)
    buf = torch.full((q0.size + 2 * BAND,), CANARY, dtype=dtype, device=DEV)
    view = buf[BAND:BAND + q0.size]
    view.copy_(torch.tensor(q0, dtype=dtype, device=DEV))
    return buf, view


def bands_ok(buf):
    head, tail = buf[:BAND], buf[-BAND:]
    return bool((head == CANARY).all()) and bool((tail == CANARY).all())


EO = (W.BURGERS_EO, "1e-5", Fraction(4, 15))


def _eo_data(n, seed, signed):
    return W.smooth_random(np.random.default_rng(seed), n, 100000, 0 if signed else 20000)


@pytest.mark.parametrize("kernel,V", [(1, 0), (2, 8), (2, 16), (2, 32), (12, 0)])
@pytest.mark.parametrize("n", [1024 * 3 + 1, 50_000 + 3, 262_147])
@pytest.mark.parametrize("boundary", [W.PERIODIC, W.TRANSMISSIVE])
def test_canary_1d_blocked(F, kernel, V, n, boundary):
    if kernel == 12 and boundary == W.TRANSMISSIVE:
        pytest.skip("K2P: periodic single domains")
    q0 = _eo_data(n, n + kernel + V, signed=True)
    plan = F.fqnm_plan_ex(n, 1e-5, float(EO[2]), W.BURGERS_EO, boundary)
    F.fqnm_debug_override(plan, kernel, 0, V)
    buf, q = banded(q0)
    F.fqnm_step(plan, q, 45)
    assert bands_ok(buf)
    assert np.array_equal(q.cpu().numpy().astype(np.int64), oracle.Rule(*EO).run(q0, 45, boundary))


@pytest.mark.parametrize("n", [16384 + 3, 65536 + 513, 200_003])
def test_canary_resident(F, n):
    q0 = _eo_data(n, n, signed=True)
    plan = F.fqnm_plan_ex(n, 1e-5, float(EO[2]), W.BURGERS_EO)
    assert plan.info()["kernel"] == 6
    buf, q = banded(q0)
    F.fqnm_step(plan, q, 130)
    assert bands_ok(buf)
    assert np.array_equal(q.cpu().numpy().astype(np.int64), oracle.Rule(*EO).run(q0, 130))


@pytest.mark.parametrize("n,B", [(1024, 7), (256, 33), (3000, 5), (16384, 2)])
def test_canary_ensembles(F, n, B):
    rng = np.random.default_rng(n + B)
    q0 = np.stack([W.smooth_random(rng, n, 5000, 0) for _ in range(B)])
    plan = F.fqnm_plan_ex(n, 1e-4, 0.5, W.LINEAR, batch=B)
    assert plan.info()["kernel"] in (3, 4)
    buf, q = banded(q0)
    F.fqnm_step(plan, q, 77)
    assert bands_ok(buf)
    ref = oracle.Rule(W.LINEAR, "1e-4", Fraction(1, 2)).run(q0, 77)
    assert np.array_equal(q.view(B, n).cpu().numpy().astype(np.int64), ref)


def test_canary_p2p_virtual_ranks(F):
    """The fused peer push writes into the neighbours' plan buffers: their owned cells
    must match the oracle and nothing outside [H | n | H] of each buffer may change."""
    from paper_2604_06947_b200 import halo
    n = 30_011
    q0 = _eo_data(n, 5, signed=True)
    ref = oracle.Rule(*EO).run(q0, 60)
    for P, H in [(2, 16), (3, 24), (4, 8)]:
        parts = [halo.partition(n, P, r) for r in range(P)]
        plans = [F.fqnm_plan_ex(nl, 1e-5, float(EO[2]), W.BURGERS_EO, F.HALO, halo=H,
                                n_global=n, offset=o, p2p=True) for o, nl in parts]
        ring = halo.P2PRing.virtual(plans)
        ring.load([torch.tensor(q0[o:o + nl], dtype=torch.int32, device=DEV) for o, nl in parts])
        ring.step(60)
        got = np.concatenate([ring.owned(i).cpu().numpy() for i in range(P)]).astype(np.int64)
        assert np.array_equal(got, ref), (P, H)


@pytest.mark.parametrize("kernel", [7, 9])
@pytest.mark.parametrize("shape", [(37, 301), (64, 256), (5, 1000)])
def test_canary_2d(F, kernel, shape):
    ny, nx = shape
    rng = np.random.default_rng(nx + ny + kernel)
    q0 = W.smooth_random(rng, nx * ny, 100000, 20000).reshape(ny, nx)
    lam = Fraction(2, 15)
    plan = F.fqnm_plan_2d(nx, ny, 1e-5, float(lam), float(lam), W.BURGERS_EO)
    F.fqnm_debug_override(plan, kernel, 0, 0)
    buf, q = banded(q0)
    F.fqnm_step(plan, q, 9)
    assert bands_ok(buf)
    ref = oracle.Rule2D(W.BURGERS_EO, "1e-5", lam, lam).run(q0, 9)
    assert np.array_equal(q.view(ny, nx).cpu().numpy().astype(np.int64), ref)


@pytest.mark.parametrize("kernel", [8, 10])
@pytest.mark.parametrize("shape", [(6, 20, 130), (9, 33, 128), (3, 8, 1000)])
def test_canary_3d(F, kernel, shape):
    nz, ny, nx = shape
    rng = np.random.default_rng(nx + ny + nz + kernel)
    q0 = W.smooth_random(rng, nx * ny * nz, 50000, 10000).reshape(nz, ny, nx)
    lam = Fraction(1, 15)
    plan = F.fqnm_plan_3d(nx, ny, nz, 1e-5, float(lam), float(lam), float(lam), W.BURGERS_EO)
    F.fqnm_debug_override(plan, kernel, 0, 0)
    buf, q = banded(q0)
    F.fqnm_step(plan, q, 4)
    assert bands_ok(buf)
    ref = oracle.Rule3D(W.BURGERS_EO, "1e-5", lam, lam, lam).run(q0, 4)
    assert np.array_equal(q.view(nz, ny, nx).cpu().numpy().astype(np.int64), ref)


@pytest.mark.parametrize("V", [1, 2, 4])
def test_canary_euler(F, V):
    n = 1000 + 7
    nsteps, lam = W.sod_steps_and_dt_dx(n)
    q0 = W.sod_q0(n)
    plan = F.fqnm_plan(n, 1e-7, lam, F.EULER_ROE, F.TRANSMISSIVE)
    F.fqnm_debug_override(plan, 0, 0, V)
    buf, q = banded(q0, torch.int64)
    F.fqnm_step(plan, q, 40)
    assert bands_ok(buf)
    assert np.array_equal(q.view(3, n).cpu().numpy(), oracle.euler_run(q0, 40, 1e-7, lam))
