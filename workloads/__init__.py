"""Seeded synthetic inputs for the FQNM configurations (shared by both sides).

This module is the ONLY code shared between the CUDA path's tests/bench and
the CPU oracle.  It holds no transfer-map, flux or stepping arithmetic: it
produces initial data q0 (reading D5 of SURVEY.md: q0 is generated once by the
harness and fed to both sides, so parity is a property of the stepper, not of
libm) and the scheme parameters (delta, dt/dx) each configuration states.

Configurations are BASELINE.json `configs` (BJ.cfg1..cfg5) plus the ensemble
ENS-1 of SURVEY.md §8(d)-D2.  Citations: P:a-b = PAPER.md lines, S:a-b =
SPEC.md lines.

Readings used here (listed in DESIGN.md):
  * cell centres x_i = (i + 1/2)/N              (A5; P:40 writes i*dx)
  * q0_i = RHA(fl(u0_i / delta))                 (Eq. quantisation, tie rule A1)
  * Courant nu = alpha * dt/dx                   (Eq. cfl_number, A3)
    with alpha = |a| (linear) or delta*max|q0| (Burgers, maximum principle P:211)
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Optional

import numpy as np

# ---------------------------------------------------------------------------
# flux kinds / boundaries: the integer codes of include/fqnm.h (plain data)
LINEAR, BURGERS_EO, BURGERS_LF, EULER_ROE = 0, 1, 2, 3
PERIODIC, TRANSMISSIVE = 0, 1


@dataclass
class Workload:
    name: str
    kind: int
    boundary: int
    n: int
    steps: int
    delta: Fraction            # exact decimal value of delta
    nu: Fraction               # Courant number as stated by the config
    batch: int = 1
    nvar: int = 1
    flux_param: Fraction = Fraction(1)   # a (linear), gamma (Euler)
    note: str = ""
    extra: dict = field(default_factory=dict)


def cfg(name: str, **over) -> Workload:
    """The named configuration, optionally with fields overridden (e.g. n=)."""
    w = _CONFIGS[name]
    d = dict(w.__dict__)
    d.update(over)
    d["extra"] = dict(w.extra)
    return Workload(**d)


_CONFIGS = {
    # BJ.cfg1: linear advection a=1, N=1024, periodic, delta=1e-4, Courant 0.5, 2000 steps
    "cfg1": Workload("cfg1", LINEAR, PERIODIC, 1024, 2000, Fraction("1e-4"), Fraction("0.5")),
    # BJ.cfg2: Burgers EO split, N=65536, periodic, delta=1e-5, Courant 0.4, 20000 steps
    "cfg2": Workload("cfg2", BURGERS_EO, PERIODIC, 65536, 20000, Fraction("1e-5"), Fraction("0.4")),
    # BJ.cfg3: high-frequency transport a=1, N=2^24, delta=1e-6, Courant 0.5, 1e4 steps
    "cfg3": Workload("cfg3", LINEAR, PERIODIC, 1 << 24, 10000, Fraction("1e-6"), Fraction("0.5")),
    # BJ.cfg4: Burgers single domain N=2^31, delta=1e-6, Courant 0.4, 1000 steps
    "cfg4": Workload("cfg4", BURGERS_EO, PERIODIC, 1 << 31, 1000, Fraction("1e-6"), Fraction("0.4"),
                     extra={"seed": 0, "nmodes": 64}),
    # BJ.cfg5: Sod, gamma=1.4, 3 x int64, N=2^26, delta=1e-7, CFL 0.4, transmissive, t=0.2
    "cfg5": Workload("cfg5", EULER_ROE, TRANSMISSIVE, 1 << 26, 0, Fraction("1e-7"), Fraction("0.4"),
                     nvar=3, flux_param=Fraction("1.4"), extra={"t_end": Fraction("0.2"),
                                                            "window_steps": 10000}),
    # 2^16 independent cfg1-like problems
    "ens1": Workload("ens1", LINEAR, PERIODIC, 1024, 2000, Fraction("1e-4"), Fraction("0.5"),
                     batch=1 << 16),
}

CONFIG_NAMES = tuple(_CONFIGS)


# ---------------------------------------------------------------------------
# helpers (input preparation only)

def cell_centres(n: int, offset: int = 0, count: Optional[int] = None) -> np.ndarray:
    """x_i = (i + 1/2)/N for i in [offset, offset+count)  (reading A5)."""
    if count is None:
        count = n - offset
    i = np.arange(offset, offset + count, dtype=np.float64)
    return (i + 0.5) / float(n)


def quantise(u, delta: float):
    """q = RHA(fl(u/delta)) elementwise (Eq. quantisation; tie rule A1).

    Works on numpy arrays and torch tensors (float64).  RHA is evaluated
    exactly on the double t = fl(u/delta): r = trunc(t); if |t - r| >= 1/2
    then r += sign(t) (t - trunc(t) is exact in binary64)."""
    try:
        import torch
        if isinstance(u, torch.Tensor):
            t = u / delta
            r = torch.trunc(t)
            r = r + torch.where((t - r).abs() >= 0.5, torch.sign(t), torch.zeros_like(t))
            return r.to(torch.int64)
    except ImportError:  # pragma: no cover
        pass
    u = np.asarray(u, dtype=np.float64)
    t = u / delta
    r = np.trunc(t)
    r = r + np.where(np.abs(t - r) >= 0.5, np.sign(t), 0.0)
    return r.astype(np.int64)


def dt_dx(w: Workload, qmax: Optional[int] = None) -> Fraction:
    """Exact dt/dx = nu / alpha for the configuration (reading A3/D3).

    linear: alpha = |a|; Burgers: alpha = delta * max|q0| (max principle P:211)."""
    if w.kind == LINEAR:
        return w.nu / abs(w.flux_param)
    if w.kind in (BURGERS_EO, BURGERS_LF):
        if qmax is None:
            raise ValueError("Burgers dt/dx needs max|q0|")
        return w.nu / (w.delta * qmax)
    raise ValueError("Euler dt/dx: use sod_steps_and_dt_dx")


def dt_dx_double(w: Workload, qmax: Optional[int] = None) -> float:
    """The double a user would pass to fqnm_plan: fl(nu / fl(alpha))."""
    if w.kind == LINEAR:
        return float(w.nu) / abs(float(w.flux_param))
    return float(w.nu) / (float(w.delta) * float(qmax))


# ---------------------------------------------------------------------------
# initial data

def u0_gaussian(x: np.ndarray, centre: float = 0.5, width: float = 0.05) -> np.ndarray:
    """BJ.cfg1: u0 = exp(-((x - 0.5)/0.05)^2)."""
    return np.exp(-((x - centre) / width) ** 2)


def q0_cfg1(n: int = 1024, centre: float = 0.5, delta: float = 1e-4) -> np.ndarray:
    return quantise(u0_gaussian(cell_centres(n), centre, 0.05), delta)


def q0_cfg2(n: int = 65536, delta: float = 1e-5) -> np.ndarray:
    """BJ.cfg2: u0 = 0.5 + sin(2 pi x)."""
    x = cell_centres(n)
    return quantise(0.5 + np.sin(2.0 * math.pi * x), delta)


def q0_cfg3(n: int = 1 << 24, delta: float = 1e-6, offset: int = 0,
            count: Optional[int] = None) -> np.ndarray:
    """BJ.cfg3: u0 = exp(-((x-0.5)/0.1)^2) * cos(2 pi x N/3).

    At cell centres cos(2 pi (i+1/2)/3) takes the exact values (0.5, -1, 0.5)
    for i mod 3 = 0, 1, 2; exact constants are used instead
    of libm cos of a huge argument."""
    x = cell_centres(n, offset, count)
    i = np.arange(offset, offset + len(x))
    c = np.array([0.5, -1.0, 0.5])[i % 3]
    return quantise(np.exp(-((x - 0.5) / 0.1) ** 2) * c, delta)


def cfg4_modes(seed: int = 0, nmodes: int = 64):
    """BJ.cfg4 'seeded sum of 64 random-phase sines with amplitudes ~U(0,1/64)'.

    Reading A7: numpy default_rng(seed); amplitudes drawn first, then phases."""
    rng = np.random.default_rng(seed)
    amp = rng.uniform(0.0, 1.0 / 64.0, nmodes)
    phase = rng.uniform(0.0, 2.0 * math.pi, nmodes)
    return amp, phase


def u0_cfg4_at(i, n: int, amp, phase):
    """u0 of BJ.cfg4 at integer cell indices i (float64 torch tensor of indices)."""
    import torch
    x = (i + 0.5) / float(n)
    u = torch.full_like(x, 0.2)
    for k in range(len(amp)):
        u += float(amp[k]) * torch.sin((2.0 * math.pi * (k + 1)) * x + float(phase[k]))
    return u


def q0_cfg4(n: int = 1 << 31, delta: float = 1e-6, seed: int = 0, nmodes: int = 64,
            device=None, offset: int = 0, count: Optional[int] = None,
            out=None, chunk: int = 1 << 25):
    """BJ.cfg4: u0 = 0.2 + sum_k a_k sin(2 pi k x + theta_k), summed in k order.

    Generated in float64 with torch (on `device`, chunked) into an int32
    tensor `out` (allocated if None).  Elementwise, so any sub-range (or
    `q0_cfg4_at`) reproduces the same integers bit for bit."""
    import torch
    amp, phase = cfg4_modes(seed, nmodes)
    if count is None:
        count = n - offset
    if out is None:
        out = torch.empty(count, dtype=torch.int32, device=device)
    dev = out.device
    for s in range(0, count, chunk):
        e = min(count, s + chunk)
        i = torch.arange(offset + s, offset + e, dtype=torch.float64, device=dev)
        out[s:e] = quantise(u0_cfg4_at(i, n, amp, phase), delta).to(torch.int32)
    return out


def q0_cfg4_at(idx, n: int = 1 << 31, delta: float = 1e-6, seed: int = 0, nmodes: int = 64,
               device=None):
    """q0 of BJ.cfg4 at arbitrary (e.g. wrapped window) indices; int64 numpy array."""
    import torch
    amp, phase = cfg4_modes(seed, nmodes)
    i = torch.as_tensor(np.asarray(idx) % n, dtype=torch.float64, device=device)
    return quantise(u0_cfg4_at(i, n, amp, phase), delta).cpu().numpy()


def q0_ensemble(batch: int, n: int = 1024, delta: float = 1e-4, first: int = 0,
                count: Optional[int] = None) -> np.ndarray:
    """ENS-1: problem b is cfg1 with centre 0.25 + 0.5 (b+1/2)/B."""
    if count is None:
        count = batch - first
    x = cell_centres(n)[None, :]
    b = np.arange(first, first + count, dtype=np.float64)[:, None]
    c = 0.25 + 0.5 * (b + 0.5) / float(batch)
    return quantise(np.exp(-((x - c) / 0.05) ** 2), delta)


# ---------------------------------------------------------------------------
# Sod (BJ.cfg5)

SOD_LEFT = (1.0, 0.0, 1.0)      # (rho, u, p)
SOD_RIGHT = (0.125, 0.0, 0.1)


def sod_q0(n: int, delta: Fraction = Fraction("1e-7"), gamma: Fraction = Fraction("1.4"),
           ) -> np.ndarray:
    """Conserved integer states [3][n] for the Sod tube (reading A13: cells with
    x_i < 1/2 are left).  E = p/(gamma-1) + rho u^2/2; with u = 0 the integers
    are exact: left (1e7, 0, 2.5e7), right (1.25e6, 0, 2.5e6) at delta = 1e-7."""
    def cons(rho, u, p):
        rho, u, p = Fraction(rho), Fraction(u), Fraction(p)
        E = p / (gamma - 1) + rho * u * u / 2
        vals = [rho / delta, rho * u / delta, E / delta]
        out = []
        for v in vals:
            r = int(abs(v) + Fraction(1, 2)) * (1 if v >= 0 else -1)
            out.append(r)
        return out
    L = cons(Fraction("1"), Fraction(0), Fraction("1"))
    R = cons(Fraction("0.125"), Fraction(0), Fraction("0.1"))
    q = np.empty((3, n), dtype=np.int64)
    nl = n // 2            # x_i = (i+1/2)/n < 1/2  <=>  i < (n-1)/2
    for c in range(3):
        q[c, :nl] = L[c]
        q[c, nl:] = R[c]
    return q


def sod_steps_and_dt_dx(n: int, t_end: float = 0.2, cfl: float = 0.4, gamma: float = 1.4):
    """Reading A11: nsteps = ceil(T c_L N / CFL) with c_L = sqrt(gamma p_L/rho_L),
    lambda = fl(fl(T N)/nsteps).  Returns (nsteps, dt/dx as double)."""
    c_l = math.sqrt(gamma * SOD_LEFT[2] / SOD_LEFT[0])
    nsteps = int(math.ceil(t_end * c_l * n / cfl))
    lam = (t_end * n) / nsteps
    return nsteps, lam


# ---------------------------------------------------------------------------
# generic seeded fuzz data (tests)

def random_states(rng: np.random.Generator, shape, lo: int, hi: int) -> np.ndarray:
    return rng.integers(lo, hi + 1, size=shape, dtype=np.int64)


def smooth_random(rng: np.random.Generator, n: int, amp: int, offset: int = 0,
                  nmodes: int = 8) -> np.ndarray:
    """Seeded smooth periodic integer data (sum of a few sines), for parity tests."""
    x = cell_centres(n)
    u = np.full(n, float(offset))
    for k in range(1, nmodes + 1):
        u += rng.uniform(0, amp / nmodes) * np.sin(2 * math.pi * k * x + rng.uniform(0, 2 * math.pi))
    return np.rint(u).astype(np.int64)
