"""The float64 form of the EO magnitude map used by the stepping kernels (maps.cuh eo_g_dp,
DESIGN.md section 6): g = rint(fl(q^2 d)) with d = fl((1/Q)(1 + 2^-46)) must equal the rule's
RHA(q^2/Q) = floor((2 q^2 + Q) / (2 Q)) whenever q^2 < 2^44.  This test replays the kernel's
three operations in exact rational arithmetic (the FMA forms q^2 d exactly and rounds once to
binary64; the magic add rounds to nearest-even integer) on ties, near-ties and random states,
against the oracle's integer definition -- the argument itself, independent of any GPU."""
from fractions import Fraction

import numpy as np
import pytest

import oracle.rules as R


def _dinv(P, Q):
    # as the planner: (P/Q)(1 + 2^-46) in extended precision, rounded to binary64; float(Fraction)
    # rounds correctly, which is within the 2^-52 the argument allows
    return float(Fraction(P, Q) * (1 + Fraction(1, 2 ** 46)))


def _g_f64(q, d):
    t1 = float(Fraction(q * q) * Fraction(d))          # FMA: exact product, one rounding
    return int(np.rint(t1))                             # + 1.5 2^52: round to nearest even


def _g_ref(q, P, Q):
    return (2 * P * q * q + Q) // (2 * Q)               # RHA of a non-negative rational


@pytest.mark.parametrize("Q", [2, 3, 10, 750000, 1724240, 4186126, (1 << 31) - 1, 1 << 30])
def test_f64_map_equals_rha(Q):
    d = _dinv(1, Q)
    rng = np.random.default_rng(Q % 1000)
    qmax = min((1 << 22) - 1, int((Q * (1 << 20)) ** 0.5))     # fast-path domain: kappa q^2 <= 2^20
    qs = set(int(x) for x in rng.integers(0, qmax + 1, 4000))
    qs |= {0, 1, 2, qmax, qmax - 1}
    # ties and nearest misses: q with 2 q^2 = (2k + 1) Q +- small
    for k in list(range(0, 50)) + [int(x) for x in rng.integers(0, 1 << 20, 300)]:
        root = int(((2 * k + 1) * Q / 2) ** 0.5)
        for q in range(max(0, root - 2), min(qmax, root + 2) + 1):
            qs.add(q)
    bad = [(q, _g_f64(q, d), _g_ref(q, 1, Q)) for q in qs if _g_f64(q, d) != _g_ref(q, 1, Q)]
    assert not bad, bad[:5]
    # and the reference itself is the oracle's rule (Eq. flux_table with RHA)
    for q in list(qs)[:200]:
        lam_over_delta_half = Fraction(1, Q)           # kappa = dt/dx * delta / 2 = 1/Q
        assert _g_ref(q, 1, Q) == R.round_rational(lam_over_delta_half * q * q, R.RHA)


def test_f64_map_exact_ties_round_away():
    # Q = 2: q^2/2 is a tie for every odd q; RHA rounds up
    d = _dinv(1, 2)
    for q in range(1, 2001, 2):
        assert _g_f64(q, d) == (q * q + 1) // 2


def _round_div_f64(num, den):
    """maps.cuh round_div_dp replayed exactly: d = (1/den)(1 + 2^-46) rounded to binary64 with
    its last two significand bits cleared (so that 1.5 2^52 d is exact), X = 1.5 2^52 + num,
    t = fma(X, d, -1.5 2^52 d) (one rounding), result = rint(t)."""
    import struct
    d = float(Fraction(1, den) * (1 + Fraction(1, 2 ** 46)))
    bits = struct.unpack("<Q", struct.pack("<d", d))[0] & ~3
    d = struct.unpack("<d", struct.pack("<Q", bits))[0]
    c = -(d * 2.0 ** 52 + d * 2.0 ** 51)
    assert Fraction(c) == -Fraction(d) * 3 * 2 ** 51            # the constant is exact
    X = float(Fraction(3 * 2 ** 51) + num)
    assert Fraction(X) == Fraction(3 * 2 ** 51) + num           # and so is the conversion
    return int(np.rint(float(Fraction(X) * Fraction(d) + Fraction(c))))


@pytest.mark.parametrize("den", [1, 2, 3, 9, 18, 750000, 1724240, (1 << 31) - 1, 10 ** 9 + 7, (1 << 40) + 15])
def test_f64_rounded_division_equals_rha(den):
    """RHA(num / den) for |num| < 2^44, both signs, exact ties and their neighbours."""
    rng = np.random.default_rng(den % 997)

    def ref(num):
        r = (2 * abs(num) + den) // (2 * den)
        return -r if num < 0 else r

    nums = [int(x) for x in rng.integers(-(1 << 44) + 1, 1 << 44, 3000)]
    for k in range(-60, 60):
        for dn in (-1, 0, 1):
            nums.append((2 * k + 1) * den // 2 + dn)
    nums += [0, 1, -1, (1 << 44) - 1, -(1 << 44) + 1]
    bad = [(x, _round_div_f64(x, den), ref(x)) for x in nums if abs(x) < (1 << 44) and _round_div_f64(x, den) != ref(x)]
    assert not bad, bad[:5]
