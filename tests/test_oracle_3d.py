"""Pins for the 3D directional-composition oracle (Thm formal Cartesian dimensional
extension, Eq. nd_transfer_rule with d = 3)."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import PERIODIC, TRANSMISSIVE, rules
from oracle.rules import BURGERS_EO, LINEAR
import workloads as W

RULES3D = [  # kind, delta, (dt/dx, dt/dy, dt/dz), (ax, ay, az), amplitude, offset
    (LINEAR, "1e-3", (Fraction(1, 4), Fraction(1, 5), Fraction(1, 6)), (1, 1, 1), 3000, 0),
    (LINEAR, "1e-3", (Fraction(1, 4), Fraction(1, 5), Fraction(1, 7)), (-1, 1, -1), 3000, 100),
    (BURGERS_EO, "1e-5", (Fraction(1, 15), Fraction(1, 10), Fraction(1, 12)), (1, 1, 1), 100000, 20000),
]


def _field(rng, nz, ny, nx, amp, off):
    x = W.cell_centres(nx)[None, None, :]
    y = W.cell_centres(ny)[None, :, None]
    z = W.cell_centres(nz)[:, None, None]
    u = off + amp * 0.5 * (np.sin(2 * np.pi * x + rng.uniform(0, 6)) *
                           np.cos(2 * np.pi * 2 * y + rng.uniform(0, 6)) *
                           np.cos(2 * np.pi * z + rng.uniform(0, 6)))
    return (np.rint(u) + rng.integers(-amp // 50, amp // 50 + 1, (nz, ny, nx))).astype(np.int64)


def _rule(case):
    kind, d, lams, params, amp, off = RULES3D[case]
    return oracle.Rule3D(kind, d, *lams, params=params), amp, off


@pytest.mark.parametrize("case", range(len(RULES3D)))
def test_3d_conservation_periodic(case):
    r, amp, off = _rule(case)
    q = _field(np.random.default_rng(170 + case), 7, 9, 11, amp, off)
    s0 = int(q.sum())
    for _ in range(15):
        q = r.step(q)
        assert int(q.sum()) == s0                    # Thm (i): exact integer mass


@pytest.mark.parametrize("case", range(len(RULES3D)))
def test_3d_reduces_to_2d_and_1d(case):
    """Data constant along z: the z fluxes cancel and every plane is the 2D oracle;
    data constant along y and z: every x line is the 1D oracle."""
    kind, d, lams, params, amp, off = RULES3D[case]
    r, amp, off = _rule(case)
    rng = np.random.default_rng(180 + case)
    plane = _field(rng, 1, 13, 17, amp, off)[0]
    q = np.tile(plane, (5, 1, 1))
    r2 = oracle.Rule2D(kind, d, lams[0], lams[1], params[0], params[1])
    for boundary in (PERIODIC, TRANSMISSIVE):
        out = r.run(q, 12, boundary)
        ref = r2.run(plane, 12, boundary)
        assert all(np.array_equal(out[k], ref) for k in range(5))
    line = W.smooth_random(rng, 29, amp, off)
    q = np.tile(line, (4, 6, 1))
    out = r.run(q, 12, TRANSMISSIVE)
    ref = r.rs[0].run(line, 12, TRANSMISSIVE)
    assert all(np.array_equal(out[k, j], ref) for k in range(4) for j in range(6))
    # and along z alone
    col = W.smooth_random(rng, 23, amp, off)
    q = np.tile(col[:, None, None], (1, 3, 5))
    out = r.run(q, 12)
    ref = r.rs[2].run(col, 12)
    assert all(np.array_equal(out[:, j, i], ref) for j in range(3) for i in range(5))


def test_3d_translation_and_axis_permutation():
    kind, d, lams, params, amp, off = RULES3D[2]
    r = oracle.Rule3D(kind, d, *lams)
    rp = oracle.Rule3D(kind, d, lams[2], lams[0], lams[1])      # (x, y, z) <- (z, x, y)
    q = _field(np.random.default_rng(190), 6, 8, 10, amp, off)
    ref = r.run(q, 7)
    for s in ((1, 0, 0), (0, 3, 0), (0, 0, 5), (2, 5, 7)):
        assert np.array_equal(r.run(np.roll(q, s, (0, 1, 2)), 7), np.roll(ref, s, (0, 1, 2)))
    # new axes: x' = z, y' = x, z' = y  ->  array [y][x][z]
    qp = np.transpose(q, (1, 2, 0))
    assert np.array_equal(rp.run(qp, 7), np.transpose(ref, (1, 2, 0)))


@pytest.mark.parametrize("case", range(len(RULES3D)))
def test_3d_update_level_consistency(case):
    """Thm (iii): the reconstructed 3D update equals the dimension-by-dimension split
    classical form up to O(delta): <= 6 delta per cell and step (six rounded maps),
    checked exactly in rational arithmetic."""
    kind, d, lams, params, amp, off = RULES3D[case]
    delta = Fraction(d)
    sp = [rules.split(kind, Fraction(a)) for a in params]
    r = oracle.Rule3D(kind, d, *lams, params=params)
    q = _field(np.random.default_rng(200 + case), 4, 5, 6, amp, off)
    qn = r.step(q)
    nz, ny, nx = q.shape
    u = lambda k, j, i: delta * int(q[k % nz, j % ny, i % nx])
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                cls = Fraction(0)
                for m, (dk, dj, di) in enumerate(((0, 0, 1), (0, 1, 0), (1, 0, 0))):
                    fp, fm = sp[m]
                    F = lambda a, b: fp(a) + fm(b)
                    c = u(k, j, i)
                    cls += lams[m] * (F(c, u(k + dk, j + dj, i + di)) - F(u(k - dk, j - dj, i - di), c))
                assert abs(delta * (int(qn[k, j, i]) - int(q[k, j, i])) + cls) <= 6 * delta


def test_3d_constant_state_and_single_cell_spread():
    r = oracle.Rule3D(LINEAR, "0.1", Fraction(1, 4), Fraction(1, 4), Fraction(1, 4))
    assert np.array_equal(r.step(np.full((4, 5, 6), 77)), np.full((4, 5, 6), 77))
    q = np.zeros((5, 5, 5), dtype=np.int64)
    q[2, 2, 2] = 6
    out = r.step(q)
    # RHA(6/4) = 2 quanta leave in +x, +y and +z; the cell keeps 6 - 3 * 2 = 0
    assert out[2, 2, 2] == 0 and out[2, 2, 3] == 2 and out[2, 3, 2] == 2 and out[3, 2, 2] == 2
    assert out.sum() == 6
    # with kappa = 1/2 per direction (Courant sum 3/2 > 1) the unsplit composition
    # overshoots: 3 * RHA(3) = 9 > 6 quanta leave, the cell goes negative (the
    # theorem claims conservation and O(delta) consistency, not monotonicity)
    r2 = oracle.Rule3D(LINEAR, "0.1", Fraction(1, 2), Fraction(1, 2), Fraction(1, 2))
    out = r2.step(q)
    assert out[2, 2, 2] == -3 and out.sum() == 6
