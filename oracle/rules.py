"""Exact (Fraction) definitions of the FQNM transfer maps — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this.

This is Eq. flux_table of the paper written out literally in exact rational
arithmetic (reading D2: the maps are evaluated exactly, never as a float
chain):

    phi^{+/-}(q) = round( f^{+/-}(delta q) * (dt/dx) * delta^{-1} )

with round = round-half-away-from-zero (reading A1/D1; FLOOR and HALF_EVEN
are available for the brute-force studies), and the flux splittings

    LINEAR      f(u) = a u,   upwind split f+ = max(a,0) u, f- = min(a,0) u
    BURGERS_EO  f(u) = u^2/2, f+ = max(u,0)^2/2, f- = min(u,0)^2/2          (BJ.cfg2/cfg4, A4)
    BURGERS_LF  f+- = (u^2/2 +- alpha u)/2                                 ("Lax-Friedrichs")
"""
from __future__ import annotations

from fractions import Fraction
from math import gcd
from typing import Callable, Tuple

LINEAR, BURGERS_EO, BURGERS_LF = 0, 1, 2
RHA, FLOOR, HALF_EVEN = 0, 1, 2
SUPP_ALL, SUPP_POS, SUPP_NEG = 0, 1, 2


def round_rational(x: Fraction, rounding: int = RHA) -> int:
    """round(x) for an exact rational x (reading A1)."""
    x = Fraction(x)
    if rounding == FLOOR:
        return x.numerator // x.denominator
    a = abs(x)
    fl = a.numerator // a.denominator
    frac = a - fl
    if rounding == RHA:
        r = fl + 1 if frac >= Fraction(1, 2) else fl
    else:
        if frac > Fraction(1, 2):
            r = fl + 1
        elif frac < Fraction(1, 2):
            r = fl
        else:
            r = fl if fl % 2 == 0 else fl + 1
    return -r if x < 0 else r


def split(kind: int, param: Fraction = Fraction(1)) -> Tuple[Callable, Callable]:
    """The monotone flux splitting f = f+ + f- (Eq. flux_splitting)."""
    param = Fraction(param)
    if kind == LINEAR:
        a = param
        return (lambda u: max(a, 0) * u), (lambda u: min(a, 0) * u)
    if kind == BURGERS_EO:
        return (lambda u: max(u, 0) ** 2 / 2), (lambda u: min(u, 0) ** 2 / 2)
    if kind == BURGERS_LF:
        alpha = param
        return (lambda u: (u * u / 2 + alpha * u) / 2), (lambda u: (u * u / 2 - alpha * u) / 2)
    raise ValueError(f"unknown scalar flux kind {kind}")


def phi(kind: int, delta, dt_dx, q: int, sign: int, param=Fraction(1), rounding: int = RHA) -> int:
    """phi^{sign}(q) = round(f^{sign}(delta q) (dt/dx) / delta)   (Eq. flux_table)."""
    delta, dt_dx = Fraction(delta), Fraction(dt_dx)
    fp, fm = split(kind, param)
    f = fp if sign > 0 else fm
    return round_rational(f(delta * q) * dt_dx / delta, rounding)


def map_coefficients(kind: int, delta, dt_dx, sign: int, param=Fraction(1)):
    """Coefficients (c2, c1, den, support) with
    f^{sign}(delta q) (dt/dx)/delta = (c2 q^2 + c1 q)/den on the support.

    Obtained by exact interpolation of the paper's expression at q = +-1, +-2
    and verified at q = 0, +-3, +-7 (the expression is a polynomial of degree
    <= 2 on each sign half-line for every splitting above)."""
    delta, dt_dx = Fraction(delta), Fraction(dt_dx)
    fp, fm = split(kind, param)
    f = fp if sign > 0 else fm
    g = lambda q: f(delta * q) * dt_dx / delta
    if g(0) != 0:
        raise ValueError("map must vanish at q = 0")
    Ap = (g(2) - 2 * g(1)) / 2
    Bp = g(1) - Ap
    An = (g(-2) - 2 * g(-1)) / 2
    Bn = An - g(-1)
    for q in (3, 7, 11):
        assert g(q) == Ap * q * q + Bp * q
        assert g(-q) == An * q * q - Bn * q
    if (Ap, Bp) == (An, Bn):
        A, B, supp = Ap, Bp, SUPP_ALL
    elif An == 0 and Bn == 0:
        A, B, supp = Ap, Bp, SUPP_POS
    elif Ap == 0 and Bp == 0:
        A, B, supp = An, Bn, SUPP_NEG
    else:
        raise ValueError("map is not a single polynomial on a half-line")
    den = A.denominator * B.denominator // gcd(A.denominator, B.denominator)
    return int(A * den), int(B * den), int(den), supp


def kappa(kind: int, delta, dt_dx, param=Fraction(1)) -> Fraction:
    """The single rational coefficient of a LINEAR (kappa = a dt/dx) or
    BURGERS_EO (kappa = delta dt/dx / 2) map; for reporting/comparison."""
    delta, dt_dx = Fraction(delta), Fraction(dt_dx)
    if kind == LINEAR:
        return Fraction(param) * dt_dx
    if kind == BURGERS_EO:
        return delta * dt_dx / 2
    raise ValueError("kappa is defined for LINEAR and BURGERS_EO only")
