"""FQNM CPU oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously correct CPU implementation of the FQNM update of
arXiv 2604.06947.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import this package.
It shares no code with the CUDA path and the product path never calls it.

* `rules.py`      — Eq. flux_table in exact Fraction arithmetic (the definition).
* `fqnm_oracle.c` — the stepping loops (flux-difference and four-term forms),
                    reconstruction and the componentwise-quantised Roe transfer,
                    in plain C with 128-bit integer intermediates and pinned,
                    uncontracted binary64 for the Roe path.
* `reference.py`  — float64 classical split finite-volume schemes and exact
                    Riemann solutions used to check the oracle against the
                    paper's theorems.

Parity status: every function is pinned by a
`-m "not gpu"` test except the absolute physical accuracy of the Euler/Roe
variant, which the paper gives no theorem for ("no complete
convergence theory for compressible Euler"): that property is checked only
heuristically against the exact Sod solution — "parity unpinned" for that
accuracy claim; its arithmetic is pinned (consistency, mirror symmetry,
upwind reduction, conservation, alternative Roe form).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from fractions import Fraction
from typing import Optional

import numpy as np

from . import rules
from .rules import (BURGERS_EO, BURGERS_EO2, BURGERS_GODUNOV, BURGERS_LF, BURGERS_LF2,
                    FLOOR, HALF_EVEN, LINEAR, RHA, map_coefficients)

PERIODIC, TRANSMISSIVE = 0, 1

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fqnm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC",
          "-std=gnu11"]


def build(force: bool = False) -> str:
    """Compile oracle/fqnm_oracle.c into oracle/liboracle.so (gcc)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Map(ctypes.Structure):
    _fields_ = [("c2", ctypes.c_int64), ("c1", ctypes.c_int64), ("den", ctypes.c_int64),
                ("support", ctypes.c_int32), ("rounding", ctypes.c_int32)]


class _Transfer(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("rounding", ctypes.c_int32),
                ("c2", ctypes.c_int64), ("c1", ctypes.c_int64), ("den", ctypes.c_int64),
                ("pp", _Map), ("pm", _Map)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P64 = ctypes.POINTER(ctypes.c_int64)
        PD = ctypes.POINTER(ctypes.c_double)
        PM = ctypes.POINTER(_Map)
        L.or_phi.restype = ctypes.c_int64
        L.or_phi.argtypes = [PM, ctypes.c_int64]
        L.or_phi_array.argtypes = [PM, P64, P64, ctypes.c_int64]
        L.or_step_scalar.argtypes = [PM, PM, ctypes.c_int, ctypes.c_int64, P64, P64]
        L.or_step_scalar_fourterm.argtypes = [PM, PM, ctypes.c_int64, P64, P64]
        L.or_run_scalar.argtypes = [PM, PM, ctypes.c_int, ctypes.c_int64, P64, ctypes.c_int64,
                                    ctypes.c_int]
        L.or_run_scalar_batch.argtypes = [PM, PM, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                          P64, ctypes.c_int64, ctypes.c_int]
        L.or_observe.argtypes = [ctypes.c_double, P64, PD, ctypes.c_int64]
        L.or_roe_transfer.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                      P64, P64, P64]
        L.or_step_euler.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_int64, P64, P64]
        L.or_run_euler.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                   ctypes.c_int64, P64, ctypes.c_int64, ctypes.c_int]
        L.or_step_euler_density.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                            ctypes.c_double, ctypes.c_int64, P64, P64]
        L.or_run_euler_density.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_int64, P64, ctypes.c_int64,
                                           ctypes.c_int]
        L.or_step_scalar_2d.argtypes = [PM, PM, PM, PM, ctypes.c_int, ctypes.c_int64,
                                        ctypes.c_int64, P64, P64]
        L.or_run_scalar_2d.argtypes = [PM, PM, PM, PM, ctypes.c_int, ctypes.c_int64,
                                       ctypes.c_int64, P64, ctypes.c_int64, ctypes.c_int]
        PT = ctypes.POINTER(_Transfer)
        L.or_transfer_eval.restype = ctypes.c_int64
        L.or_transfer_eval.argtypes = [PT, ctypes.c_int64, ctypes.c_int64]
        L.or_transfer_array.argtypes = [PT, P64, P64, P64, ctypes.c_int64]
        L.or_step_transfer.argtypes = [PT, ctypes.c_int, ctypes.c_int64, P64, P64]
        L.or_run_transfer.argtypes = [PT, ctypes.c_int, ctypes.c_int64, P64, ctypes.c_int64,
                                      ctypes.c_int]
        PPM = ctypes.POINTER(PM)
        L.or_step_scalar_3d.argtypes = [PPM, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_int64, P64, P64]
        L.or_run_scalar_3d.argtypes = [PPM, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int64, P64, ctypes.c_int64, ctypes.c_int]
        L.or_round_rational.restype = ctypes.c_int64
        L.or_round_rational.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.c_int64,
                                        ctypes.c_int]
        L.or_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p64(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


class Rule:
    """The pair of transfer maps (phi+, phi-) for a scalar flux kind, built
    from exact rationals delta and dt/dx (Fractions, or decimal strings)."""

    def __init__(self, kind: int, delta, dt_dx, param=Fraction(1), rounding: int = RHA):
        self.kind = kind
        self.delta = Fraction(delta)
        self.dt_dx = Fraction(dt_dx)
        self.param = Fraction(param)
        self.rounding = rounding
        cp = map_coefficients(kind, self.delta, self.dt_dx, +1, self.param)
        cm = map_coefficients(kind, self.delta, self.dt_dx, -1, self.param)
        self.coef_plus, self.coef_minus = cp, cm
        self._mp = _Map(cp[0], cp[1], cp[2], cp[3], rounding)
        self._mm = _Map(cm[0], cm[1], cm[2], cm[3], rounding)

    # --- maps -------------------------------------------------------------
    def phi_plus(self, q) -> np.ndarray:
        q = np.ascontiguousarray(np.atleast_1d(q), dtype=np.int64)
        out = np.empty_like(q)
        lib().or_phi_array(ctypes.byref(self._mp), _p64(q), _p64(out), q.size)
        return out

    def phi_minus(self, q) -> np.ndarray:
        q = np.ascontiguousarray(np.atleast_1d(q), dtype=np.int64)
        out = np.empty_like(q)
        lib().or_phi_array(ctypes.byref(self._mm), _p64(q), _p64(out), q.size)
        return out

    def interface_flux(self, qL, qR) -> np.ndarray:
        """F(qL, qR) = phi+(qL) + phi-(qR)  (Eq. numerical_count_flux_definition)."""
        return self.phi_plus(qL) + self.phi_minus(qR)

    # --- stepping -----------------------------------------------------------
    def step(self, q, boundary: int = PERIODIC) -> np.ndarray:
        q = np.ascontiguousarray(q, dtype=np.int64)
        out = np.empty_like(q)
        lib().or_step_scalar(ctypes.byref(self._mp), ctypes.byref(self._mm), boundary,
                             q.size, _p64(q), _p64(out))
        return out

    def step_fourterm(self, q) -> np.ndarray:
        q = np.ascontiguousarray(q, dtype=np.int64)
        out = np.empty_like(q)
        lib().or_step_scalar_fourterm(ctypes.byref(self._mp), ctypes.byref(self._mm),
                                      q.size, _p64(q), _p64(out))
        return out

    def run(self, q, nsteps: int, boundary: int = PERIODIC, nthreads: int = 0) -> np.ndarray:
        """q^{n+nsteps} (double-buffered explicit steps)."""
        q = np.array(q, dtype=np.int64, copy=True, order="C")
        if q.ndim == 1:
            lib().or_run_scalar(ctypes.byref(self._mp), ctypes.byref(self._mm), boundary,
                                q.size, _p64(q), nsteps, nthreads)
        else:
            B, N = q.shape
            lib().or_run_scalar_batch(ctypes.byref(self._mp), ctypes.byref(self._mm), boundary,
                                      B, N, _p64(q), nsteps, nthreads)
        return q


class TransferRule:
    """An interface transfer rule Phi(qL, qR) (Thm transfer-operator equivalence,
    P:262-280): either the paper's split rule phi+(qL) + phi-(qR) (kinds 0-2) or a
    quantised two-point rule round(F(delta qL, delta qR) dt/dx / delta) rounded once
    (kinds BURGERS_GODUNOV, BURGERS_EO2, BURGERS_LF2)."""

    def __init__(self, kind: int, delta, dt_dx, param=Fraction(1), rounding: int = RHA):
        self.kind = kind
        self.delta, self.dt_dx, self.param = Fraction(delta), Fraction(dt_dx), Fraction(param)
        self.rounding = rounding
        t = _Transfer()
        t.rounding = rounding
        if kind in rules.TWO_POINT_KINDS:
            t.kind = kind
            t.c2, t.c1, t.den = rules.two_point_coefficients(kind, delta, dt_dx, param)
        else:
            r = Rule(kind, delta, dt_dx, param, rounding)
            t.kind = 0
            t.pp, t.pm = r._mp, r._mm
        self._t = t

    def phi(self, qL, qR) -> np.ndarray:
        a = np.ascontiguousarray(np.atleast_1d(qL), dtype=np.int64)
        b = np.ascontiguousarray(np.broadcast_to(np.atleast_1d(qR), a.shape), dtype=np.int64)
        out = np.empty_like(a)
        lib().or_transfer_array(ctypes.byref(self._t), _p64(a), _p64(b), _p64(out), a.size)
        return out

    def _interfaces(self, q, boundary):
        """(qL, qR) of the interfaces i+1/2, i = -1 .. N-1 (N+1 values; periodic: the
        first equals the last)."""
        if boundary == PERIODIC:
            qL = np.concatenate([q[-1:], q])
            qR = np.concatenate([q[:1], q[1:], q[:1]])
        else:
            qL = np.concatenate([q[:1], q])
            qR = np.concatenate([q, q[-1:]])
        return qL, qR

    def step(self, q, boundary: int = PERIODIC) -> np.ndarray:
        q = np.ascontiguousarray(q, dtype=np.int64)
        out = np.empty_like(q)
        lib().or_step_transfer(ctypes.byref(self._t), boundary, q.size, _p64(q), _p64(out))
        return out

    def run(self, q, nsteps: int, boundary: int = PERIODIC, nthreads: int = 0) -> np.ndarray:
        q = np.array(q, dtype=np.int64, copy=True, order="C")
        lib().or_run_transfer(ctypes.byref(self._t), boundary, q.size, _p64(q), nsteps, nthreads)
        return q

    def equivalence(self, other: "TransferRule", q, nsteps: int, boundary: int = PERIODIC):
        """Steps q with THIS rule and evaluates `other` on every visited interface
        state (qL, qR) (the hypothesis of Thm P:274-280).  Returns (q_final, stats)
        with stats = interface_evals, mismatches, first_mismatch_step, visited_pairs,
        mismatched_pairs (distinct (qL, qR))."""
        q = np.array(q, dtype=np.int64, copy=True)
        evals = mism = 0
        first = -1
        visited, bad = set(), set()
        for s in range(nsteps):
            qL, qR = self._interfaces(q, boundary)
            if boundary == PERIODIC:            # N distinct interfaces
                qL, qR = qL[1:], qR[1:]
            Ta, Tb = self.phi(qL, qR), other.phi(qL, qR)
            evals += qL.size
            neq = Ta != Tb
            if neq.any() and first < 0:
                first = s
            mism += int(neq.sum())
            visited.update(zip(qL.tolist(), qR.tolist()))
            bad.update(zip(qL[neq].tolist(), qR[neq].tolist()))
            q = self.step(q, boundary)
        return q, {"interface_evals": evals, "mismatches": mism, "first_mismatch_step": first,
                   "visited_pairs": len(visited), "mismatched_pairs": len(bad)}


class Rule2D:
    """Directional composition in 2D (Thm P:364-401): one scalar Rule per direction
    (same flux kind and delta, dt/dx and dt/dy, per-direction speed param)."""

    def __init__(self, kind: int, delta, dt_dx, dt_dy, param_x=Fraction(1), param_y=Fraction(1),
                 rounding: int = RHA):
        self.rx = Rule(kind, delta, dt_dx, param_x, rounding)
        self.ry = Rule(kind, delta, dt_dy, param_y, rounding)

    def _maps(self):
        return (ctypes.byref(self.rx._mp), ctypes.byref(self.rx._mm),
                ctypes.byref(self.ry._mp), ctypes.byref(self.ry._mm))

    def step(self, q, boundary: int = PERIODIC) -> np.ndarray:
        q = np.ascontiguousarray(q, dtype=np.int64)
        ny, nx = q.shape
        out = np.empty_like(q)
        lib().or_step_scalar_2d(*self._maps(), boundary, nx, ny, _p64(q), _p64(out))
        return out

    def run(self, q, nsteps: int, boundary: int = PERIODIC, nthreads: int = 0) -> np.ndarray:
        q = np.array(q, dtype=np.int64, copy=True, order="C")
        ny, nx = q.shape
        lib().or_run_scalar_2d(*self._maps(), boundary, nx, ny, _p64(q), nsteps, nthreads)
        return q


class Rule3D:
    """Directional composition in 3D (Thm P:364-401, d = 3): one scalar Rule per
    direction (same flux kind and delta; dt/dx, dt/dy, dt/dz; per-direction param).
    State layout [nz][ny][nx] (x fastest)."""

    def __init__(self, kind: int, delta, dt_dx, dt_dy, dt_dz, params=(1, 1, 1),
                 rounding: int = RHA):
        self.rs = [Rule(kind, delta, l, Fraction(a), rounding)
                   for l, a in zip((dt_dx, dt_dy, dt_dz), params)]
        maps = []
        for r in self.rs:
            maps += [ctypes.pointer(r._mp), ctypes.pointer(r._mm)]
        self._maps = (ctypes.POINTER(_Map) * 6)(*maps)

    def step(self, q, boundary: int = PERIODIC) -> np.ndarray:
        q = np.ascontiguousarray(q, dtype=np.int64)
        nz, ny, nx = q.shape
        out = np.empty_like(q)
        lib().or_step_scalar_3d(self._maps, boundary, nx, ny, nz, _p64(q), _p64(out))
        return out

    def run(self, q, nsteps: int, boundary: int = PERIODIC, nthreads: int = 0) -> np.ndarray:
        q = np.array(q, dtype=np.int64, copy=True, order="C")
        nz, ny, nx = q.shape
        lib().or_run_scalar_3d(self._maps, boundary, nx, ny, nz, _p64(q), nsteps, nthreads)
        return q


def observe(q, delta: float) -> np.ndarray:
    """u = fl(delta * q)  (Eq. reconstruction_operator)."""
    q = np.ascontiguousarray(q, dtype=np.int64).ravel()
    u = np.empty(q.size, dtype=np.float64)
    lib().or_observe(float(delta), _p64(q), u.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                     q.size)
    return u


# --- Euler / Roe -------------------------------------------------------------

def euler_constants(delta: float, dt_dx: float, gamma: float = 1.4):
    """(s, g1) = (fl(dt/dx / delta), fl(gamma - 1))  (SURVEY §8(c)-C2 plan constants)."""
    return dt_dx / delta, gamma - 1.0


def roe_transfer(qL, qR, delta: float, dt_dx: float, gamma: float = 1.4) -> np.ndarray:
    """T(qL, qR) = RHA(fl(F_Roe(delta qL, delta qR) * s)) for one interface."""
    s, g1 = euler_constants(delta, dt_dx, gamma)
    a = np.ascontiguousarray(qL, dtype=np.int64)
    b = np.ascontiguousarray(qR, dtype=np.int64)
    T = np.empty(3, dtype=np.int64)
    lib().or_roe_transfer(delta, s, g1, _p64(a), _p64(b), _p64(T))
    return T


def euler_step(q, delta: float, dt_dx: float, gamma: float = 1.4) -> np.ndarray:
    q = np.ascontiguousarray(q, dtype=np.int64)
    s, g1 = euler_constants(delta, dt_dx, gamma)
    out = np.empty_like(q)
    lib().or_step_euler(delta, s, g1, q.shape[1], _p64(q), _p64(out))
    return out


def euler_run(q, nsteps: int, delta: float, dt_dx: float, gamma: float = 1.4,
              nthreads: int = 0) -> np.ndarray:
    q = np.array(q, dtype=np.int64, copy=True, order="C")
    s, g1 = euler_constants(delta, dt_dx, gamma)
    lib().or_run_euler(delta, s, g1, q.shape[1], _p64(q), nsteps, nthreads)
    return q


def pack_mixed(q_rho, m, E) -> np.ndarray:
    """[3][N] int64 buffer of the density-only variant: q_rho, then the float64 bit
    patterns of m and E."""
    out = np.empty((3, len(q_rho)), dtype=np.int64)
    out[0] = q_rho
    out[1] = np.asarray(m, dtype=np.float64).view(np.int64)
    out[2] = np.asarray(E, dtype=np.float64).view(np.int64)
    return out


def unpack_mixed(q):
    q = np.ascontiguousarray(q, dtype=np.int64)
    return q[0].copy(), q[1].view(np.float64).copy(), q[2].view(np.float64).copy()


def euler_density_step(q, delta: float, dt_dx: float, gamma: float = 1.4) -> np.ndarray:
    q = np.ascontiguousarray(q, dtype=np.int64)
    s, g1 = euler_constants(delta, dt_dx, gamma)
    out = np.empty_like(q)
    lib().or_step_euler_density(delta, s, dt_dx, g1, q.shape[1], _p64(q), _p64(out))
    return out


def euler_density_run(q, nsteps: int, delta: float, dt_dx: float, gamma: float = 1.4,
                      nthreads: int = 0) -> np.ndarray:
    """Density-only quantised Euler (the paper's Sod prototype)."""
    q = np.array(q, dtype=np.int64, copy=True, order="C")
    s, g1 = euler_constants(delta, dt_dx, gamma)
    lib().or_run_euler_density(delta, s, dt_dx, g1, q.shape[1], _p64(q), nsteps, nthreads)
    return q


def max_threads() -> int:
    return int(lib().or_max_threads())


def round_rational(num: int, den: int, rounding: int = RHA) -> int:
    """C-side rounding of num/den (128-bit numerator), for pinning tests."""
    hi = num >> 64
    lo = num & ((1 << 64) - 1)
    return int(lib().or_round_rational(hi, lo, den, rounding))
