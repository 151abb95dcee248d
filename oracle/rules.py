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

and, for Thm transfer-operator equivalence, the quantised two-point
transfer rules  Phi(qL, qR) = round( F(delta qL, delta qR) (dt/dx) delta^{-1} )
(Eq. transfer_operator_equivalence_definition) of three classical
Burgers fluxes, each rounded ONCE:

    GODUNOV  F = f(u*(0; uL, uR)), u* the exact Riemann solution at x/t = 0
    EO2      F = f+(uL) + f-(uR) with the Engquist-Osher split  (rounded once,
             unlike the split rule's round(f+) + round(f-))
    LF2      F = (f(uL) + f(uR))/2 - alpha (uR - uL)/2
"""
from __future__ import annotations

from fractions import Fraction
from math import gcd
from typing import Callable, Tuple

LINEAR, BURGERS_EO, BURGERS_LF = 0, 1, 2
# two-point kinds (same codes as include/fqnm.h)
BURGERS_GODUNOV, BURGERS_EO2, BURGERS_LF2 = 5, 6, 7
TWO_POINT_KINDS = (BURGERS_GODUNOV, BURGERS_EO2, BURGERS_LF2)
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


# ---------------------------------------------------------------------------
# Quantised two-point transfer rules (Thm transfer-operator equivalence)

def burgers_f(u: Fraction) -> Fraction:
    return u * u / 2


def burgers_riemann_at_zero(uL: Fraction, uR: Fraction) -> Fraction:
    """u*(x/t = 0) of the exact entropy solution of the Burgers Riemann problem
    (textbook: a shock of speed (uL + uR)/2 if uL > uR, else a rarefaction fan
    u = x/t between uL and uR)."""
    if uL > uR:                       # shock
        s = (uL + uR) / 2
        return uL if s > 0 else (uR if s < 0 else uL)   # s = 0: f(uL) = f(uR), either
    if uL >= 0:                       # rarefaction moving right
        return uL
    if uR <= 0:                       # rarefaction moving left
        return uR
    return Fraction(0)                # transonic rarefaction: the sonic point


def two_point_flux(kind: int, uL: Fraction, uR: Fraction, param=Fraction(1)) -> Fraction:
    """The classical numerical flux F(uL, uR) of a two-point kind."""
    uL, uR = Fraction(uL), Fraction(uR)
    if kind == BURGERS_GODUNOV:
        return burgers_f(burgers_riemann_at_zero(uL, uR))
    if kind == BURGERS_EO2:
        zero = Fraction(0)
        return max(uL, zero) ** 2 / 2 + min(uR, zero) ** 2 / 2
    if kind == BURGERS_LF2:
        return (burgers_f(uL) + burgers_f(uR)) / 2 - Fraction(param) * (uR - uL) / 2
    raise ValueError(f"not a two-point kind: {kind}")


def two_point_phi(kind: int, delta, dt_dx, qL: int, qR: int, param=Fraction(1),
                  rounding: int = RHA) -> int:
    """Phi(qL, qR) = round(F(delta qL, delta qR) (dt/dx) / delta)."""
    delta, dt_dx = Fraction(delta), Fraction(dt_dx)
    return round_rational(two_point_flux(kind, delta * qL, delta * qR, param) * dt_dx / delta,
                          rounding)


def two_point_coefficients(kind: int, delta, dt_dx, param=Fraction(1)):
    """Integer coefficients (c2, c1, den) of the C oracle's evaluation:
    GODUNOV: Phi = round(c2 max(max(qL,0)^2, min(qR,0)^2) / den)
    EO2:     Phi = round(c2 (max(qL,0)^2 + min(qR,0)^2) / den)
    LF2:     Phi = round((c2 (qL^2 + qR^2) + c1 (qL - qR)) / den)
    derived from F(delta qL, delta qR) dt/dx / delta by exact interpolation and
    checked against the literal definition at sample points."""
    delta, dt_dx = Fraction(delta), Fraction(dt_dx)
    g = lambda a, b: two_point_flux(kind, delta * a, delta * b, param) * dt_dx / delta
    if kind in (BURGERS_GODUNOV, BURGERS_EO2):
        c2f, c1f = g(1, 0), Fraction(0)                     # = kappa = delta dt/dx / 2
    elif kind == BURGERS_LF2:
        # g(a, 0) = c2 a^2 + c1 a
        c2f = (g(2, 0) - 2 * g(1, 0)) / 2
        c1f = g(1, 0) - c2f
    else:
        raise ValueError(kind)
    den = c2f.denominator * c1f.denominator // gcd(c2f.denominator, c1f.denominator)
    c2, c1 = int(c2f * den), int(c1f * den)
    for a, b in ((3, -2), (-5, 4), (7, 7), (-3, -9), (0, 6), (6, 0), (2, -2)):
        if kind == BURGERS_GODUNOV:
            num = c2 * max(max(a, 0) ** 2, min(b, 0) ** 2)
        elif kind == BURGERS_EO2:
            num = c2 * (max(a, 0) ** 2 + min(b, 0) ** 2)
        else:
            num = c2 * (a * a + b * b) + c1 * (a - b)
        assert Fraction(num, den) == g(a, b), (kind, a, b)
    return c2, c1, den
