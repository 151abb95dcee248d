"""Float64 reference schemes and exact Riemann solutions — TEST INFRASTRUCTURE.

Used only by tests to check the oracle against the paper's theorems:

* `classical_step`  — the classical split finite-volume operator of
  Eq. classical_operator_definition in float64, the comparison
  object of Prop. 1 and the real-arithmetic scheme v^n of the
  convergence bound.
* `burgers_riemann_exact` — entropy solution of a Burgers top-hat on the
  periodic unit interval before wave interaction (closed form).
* `sod_exact` — exact Riemann solution of the Euler equations (textbook
  two-rarefaction/shock pressure function, solved by Newton + bisection).
"""
from __future__ import annotations

import math

import numpy as np

from .rules import BURGERS_EO, BURGERS_LF, LINEAR

PERIODIC, TRANSMISSIVE = 0, 1


def split_float(kind: int, param: float = 1.0):
    if kind == LINEAR:
        a = float(param)
        return (lambda u: max(a, 0.0) * u), (lambda u: min(a, 0.0) * u)
    if kind == BURGERS_EO:
        return (lambda u: np.maximum(u, 0.0) ** 2 / 2), (lambda u: np.minimum(u, 0.0) ** 2 / 2)
    if kind == BURGERS_LF:
        al = float(param)
        return (lambda u: (u * u / 2 + al * u) / 2), (lambda u: (u * u / 2 - al * u) / 2)
    raise ValueError(kind)


def classical_step(v: np.ndarray, kind: int, dt_dx: float, param: float = 1.0,
                   boundary: int = PERIODIC) -> np.ndarray:
    """v_i - (dt/dx) (F(v_i, v_{i+1}) - F(v_{i-1}, v_i)), F(uL,uR) = f+(uL) + f-(uR)."""
    fp, fm = split_float(kind, param)
    if boundary == PERIODIC:
        vl, vr = np.roll(v, 1), np.roll(v, -1)
    else:
        vl = np.concatenate([v[:1], v[:-1]])
        vr = np.concatenate([v[1:], v[-1:]])
    F_right = fp(v) + fm(vr)
    F_left = fp(vl) + fm(v)
    return v - dt_dx * (F_right - F_left)


def burgers_tophat_exact(x: np.ndarray, t: float, u_lo: float, u_hi: float,
                         a: float = 0.25, b: float = 0.75) -> np.ndarray:
    """Entropy solution of u_t + (u^2/2)_x = 0 on the periodic unit interval
    with u0 = u_hi on [a, b), u_lo elsewhere (u_lo < u_hi), before the
    rarefaction head meets the shock: a rarefaction fan u = (x - a)/t for
    u_lo t < x - a < u_hi t, and a shock at b + (u_lo + u_hi) t / 2."""
    s = b + 0.5 * (u_lo + u_hi) * t
    xx = np.mod(x - a - u_lo * t, 1.0) + a + u_lo * t   # unwrap to [a + u_lo t, a + u_lo t + 1)
    u = np.full_like(x, u_lo, dtype=np.float64)
    fan = (xx >= a + u_lo * t) & (xx < a + u_hi * t)
    u[fan] = (xx[fan] - a) / t
    plateau = (xx >= a + u_hi * t) & (xx < s)
    u[plateau] = u_hi
    return u


# ----------------------------------------------------------------------------
# exact Sod / Euler Riemann solution

def _fK(p, rho, pK, c, g):
    if p > pK:   # shock
        A = 2.0 / ((g + 1.0) * rho)
        B = (g - 1.0) / (g + 1.0) * pK
        f = (p - pK) * math.sqrt(A / (p + B))
        df = math.sqrt(A / (B + p)) * (1.0 - (p - pK) / (2.0 * (B + p)))
    else:        # rarefaction
        f = 2.0 * c / (g - 1.0) * ((p / pK) ** ((g - 1.0) / (2.0 * g)) - 1.0)
        df = 1.0 / (rho * c) * (p / pK) ** (-(g + 1.0) / (2.0 * g))
    return f, df


def riemann_star(left, right, g: float = 1.4):
    """(p*, u*) of the exact Riemann problem, left/right = (rho, u, p)."""
    rl, ul, pl = left
    rr, ur, pr = right
    cl, cr = math.sqrt(g * pl / rl), math.sqrt(g * pr / rr)
    p = 0.5 * (pl + pr)
    for _ in range(100):
        fl, dfl = _fK(p, rl, pl, cl, g)
        fr, dfr = _fK(p, rr, pr, cr, g)
        f = fl + fr + (ur - ul)
        pn = max(p - f / (dfl + dfr), 1e-12)
        if abs(pn - p) < 1e-15 * (pn + p):
            p = pn
            break
        p = pn
    fl, _ = _fK(p, rl, pl, cl, g)
    fr, _ = _fK(p, rr, pr, cr, g)
    u = 0.5 * (ul + ur) + 0.5 * (fr - fl)
    return p, u


def sod_exact(x: np.ndarray, t: float, left=(1.0, 0.0, 1.0), right=(0.125, 0.0, 0.1),
              x0: float = 0.5, g: float = 1.4):
    """Exact (rho, u, p) at points x and time t > 0 (left rarefaction, right shock case)."""
    rl, ul, pl = left
    rr, ur, pr = right
    cl, cr = math.sqrt(g * pl / rl), math.sqrt(g * pr / rr)
    ps, us = riemann_star(left, right, g)
    xi = (np.asarray(x, dtype=np.float64) - x0) / t
    rho = np.empty_like(xi); u = np.empty_like(xi); p = np.empty_like(xi)
    # left state / rarefaction
    rsl = rl * (ps / pl) ** (1.0 / g) if ps <= pl else rl * ((ps / pl + (g - 1) / (g + 1)) /
                                                              ((g - 1) / (g + 1) * ps / pl + 1))
    csl = cl * (ps / pl) ** ((g - 1.0) / (2.0 * g))
    head, tail = ul - cl, us - csl
    # right shock
    rsr = rr * ((ps / pr + (g - 1) / (g + 1)) / ((g - 1) / (g + 1) * ps / pr + 1))
    S = ur + cr * math.sqrt((g + 1) / (2 * g) * ps / pr + (g - 1) / (2 * g))
    for k, z in enumerate(xi):
        if z < head:
            rho[k], u[k], p[k] = rl, ul, pl
        elif z < tail:
            uu = 2.0 / (g + 1) * (cl + (g - 1) / 2 * ul + z)
            cc = 2.0 / (g + 1) * (cl + (g - 1) / 2 * (ul - z))
            rho[k] = rl * (cc / cl) ** (2.0 / (g - 1))
            u[k] = uu
            p[k] = pl * (cc / cl) ** (2.0 * g / (g - 1))
        elif z < us:
            rho[k], u[k], p[k] = rsl, us, ps
        elif z < S:
            rho[k], u[k], p[k] = rsr, us, ps
        else:
            rho[k], u[k], p[k] = rr, ur, pr
    return rho, u, p


def sod_wave_data(left=(1.0, 0.0, 1.0), right=(0.125, 0.0, 0.1), g: float = 1.4):
    """Star values and shock speed: (p*, u*, rho*L, rho*R, S)."""
    rl, ul, pl = left
    rr, ur, pr = right
    cr = math.sqrt(g * pr / rr)
    ps, us = riemann_star(left, right, g)
    rsl = rl * (ps / pl) ** (1.0 / g)
    rsr = rr * ((ps / pr + (g - 1) / (g + 1)) / ((g - 1) / (g + 1) * ps / pr + 1))
    S = ur + cr * math.sqrt((g + 1) / (2 * g) * ps / pr + (g - 1) / (2 * g))
    return ps, us, rsl, rsr, S
