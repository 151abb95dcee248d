"""Pins for the 2D directional-composition oracle (Thm formal Cartesian
dimensional extension)."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import PERIODIC, TRANSMISSIVE, rules
from oracle.rules import BURGERS_EO, LINEAR
import workloads as W

RULES2D = [  # kind, delta, dt/dx, dt/dy, ax, ay, amplitude, offset
    (LINEAR, "1e-3", Fraction(1, 4), Fraction(1, 5), 1, 1, 3000, 0),
    (LINEAR, "1e-3", Fraction(1, 3), Fraction(1, 4), -1, 1, 3000, 100),
    (BURGERS_EO, "1e-5", Fraction(2, 15), Fraction(1, 10), 1, 1, 100000, 20000),
]


def _field(rng, ny, nx, amp, off):
    x = W.cell_centres(nx)[None, :]
    y = W.cell_centres(ny)[:, None]
    u = off + amp * 0.5 * (np.sin(2 * np.pi * x + rng.uniform(0, 6)) *
                           np.cos(2 * np.pi * 2 * y + rng.uniform(0, 6)))
    return (np.rint(u) + rng.integers(-amp // 50, amp // 50 + 1, (ny, nx))).astype(np.int64)


@pytest.mark.parametrize("case", range(len(RULES2D)))
def test_2d_conservation_periodic(case):
    kind, d, lx, ly, ax, ay, amp, off = RULES2D[case]
    r = oracle.Rule2D(kind, d, lx, ly, ax, ay)
    rng = np.random.default_rng(70 + case)
    q = _field(rng, 37, 53, amp, off)
    s0 = int(q.sum())
    for _ in range(20):
        q = r.step(q)
        assert int(q.sum()) == s0                    # Thm (i): exact integer mass


@pytest.mark.parametrize("case", range(len(RULES2D)))
def test_2d_reduces_to_1d(case):
    """Data constant along y: the y fluxes cancel and every row is the 1D oracle
    with the x rule (and columns with the y rule for data constant along x)."""
    kind, d, lx, ly, ax, ay, amp, off = RULES2D[case]
    r = oracle.Rule2D(kind, d, lx, ly, ax, ay)
    rng = np.random.default_rng(80 + case)
    row = W.smooth_random(rng, 61, amp, off)
    q = np.tile(row, (17, 1))
    out = r.run(q, 25)
    ref = r.rx.run(row, 25)
    assert all(np.array_equal(out[j], ref) for j in range(17))
    col = W.smooth_random(rng, 43, amp, off)
    q = np.tile(col[:, None], (1, 9))
    out = r.run(q, 25, TRANSMISSIVE)
    ref = r.ry.run(col, 25, TRANSMISSIVE)
    assert all(np.array_equal(out[:, i], ref) for i in range(9))


def test_2d_translation_and_transpose_symmetry():
    kind, d, lx, ly, ax, ay, amp, off = RULES2D[2]
    r = oracle.Rule2D(kind, d, lx, ly)
    rt = oracle.Rule2D(kind, d, ly, lx)                 # directions swapped
    rng = np.random.default_rng(90)
    q = _field(rng, 24, 40, amp, off)
    for s in ((3, 0), (0, 7), (5, 11)):
        assert np.array_equal(r.run(np.roll(q, s, (0, 1)), 9), np.roll(r.run(q, 9), s, (0, 1)))
    assert np.array_equal(rt.run(q.T, 9), r.run(q, 9).T)


@pytest.mark.parametrize("case", range(len(RULES2D)))
def test_2d_update_level_consistency(case):
    """Thm (iii): the reconstructed 2D update equals the dimension-by-dimension split
    classical form up to O(delta): per cell and step the residual is <= 4 delta
    (four rounded maps), checked exactly in rational arithmetic."""
    kind, d, lx, ly, ax, ay, amp, off = RULES2D[case]
    delta = Fraction(d)
    fpx, fmx = rules.split(kind, Fraction(ax))
    fpy, fmy = rules.split(kind, Fraction(ay))
    r = oracle.Rule2D(kind, d, lx, ly, ax, ay)
    rng = np.random.default_rng(100 + case)
    q = _field(rng, 8, 9, amp, off)
    qn = r.step(q)
    ny, nx = q.shape
    u = [[delta * int(v) for v in row] for row in q]
    for j in range(ny):
        for i in range(nx):
            Fx = lambda a, b: fpx(a) + fmx(b)
            Fy = lambda a, b: fpy(a) + fmy(b)
            cls = (lx * (Fx(u[j][i], u[j][(i + 1) % nx]) - Fx(u[j][i - 1], u[j][i])) +
                   ly * (Fy(u[j][i], u[(j + 1) % ny][i]) - Fy(u[j - 1][i], u[j][i])))
            assert abs(delta * (int(qn[j, i]) - int(q[j, i])) + cls) <= 4 * delta


def test_2d_constant_state_fixed_and_single_cell_spread():
    r = oracle.Rule2D(LINEAR, "0.1", Fraction(1, 2), Fraction(1, 2))
    q = np.full((6, 7), 123)
    assert np.array_equal(r.step(q), q)
    q = np.zeros((5, 5), dtype=np.int64)
    q[2, 2] = 4
    out = r.step(q)
    # unsplit composition: RHA(4/2) = 2 quanta leave in +x and 2 in +y; the cell
    # keeps 4 - 2 - 2 = 0 (not the diagonal shift of dimensional splitting)
    assert out[2, 2] == 0 and out[2, 3] == 2 and out[3, 2] == 2 and out.sum() == 4
