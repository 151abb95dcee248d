"""Thin Python binding of libfqnm (include/fqnm.h) — argument marshalling only.

Every step of the FQNM hot path runs in the CUDA kernels of libfqnm.so
(paper_2604_06947_b200/csrc).  This module converts torch tensors to device
pointers, passes torch's current CUDA stream, and turns status codes into
exceptions.  There is no CPU fallback: importing it without the built library
raises, and every call needs CUDA tensors.

Names follow the C ABI: fqnm_plan, fqnm_plan_ex, fqnm_step, fqnm_step_block,
fqnm_observe, fqnm_step_host, fqnm_get_info, fqnm_transfer,
fqnm_transfer_device, fqnm_roe_transfer_device, fqnm_debug_override,
fqnm_launch_count, fqnm_destroy.  `Plan` is a small owning wrapper.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

__all__ = [
    "FqnmError", "Plan", "fqnm_plan", "fqnm_plan_ex", "fqnm_step", "fqnm_step_block",
    "fqnm_observe", "fqnm_step_host", "fqnm_get_info", "fqnm_transfer", "fqnm_transfer_device",
    "fqnm_roe_transfer_device", "fqnm_debug_override", "fqnm_debug_rcp_sqrt", "fqnm_launch_count", "fqnm_destroy",
    "fqnm_plan_validate", "fqnm_profile_enable", "fqnm_profile_read", "fqnm_halo_buffers",
    "fqnm_halo_connect", "fqnm_halo_owned", "fqnm_step_group", "fqnm_ipc_export",
    "fqnm_ipc_open", "fqnm_ipc_close", "owned_tensor", "fqnm_plan_2d", "fqnm_transfer2",
    "fqnm_transfer2_device", "fqnm_equivalence", "fqnm_plan_3d",
    "LINEAR", "BURGERS_EO", "BURGERS_LF", "EULER_ROE", "EULER_ROE_DENSITY", "PERIODIC", "TRANSMISSIVE", "HALO",
    "BURGERS_GODUNOV", "BURGERS_EO2", "BURGERS_LF2",
    "I32", "I64", "ROUND_HALF_AWAY", "ROUND_FLOOR", "ROUND_HALF_EVEN", "lib_path",
]

LINEAR, BURGERS_EO, BURGERS_LF, EULER_ROE, EULER_ROE_DENSITY = 0, 1, 2, 3, 4
BURGERS_GODUNOV, BURGERS_EO2, BURGERS_LF2 = 5, 6, 7      # two-point rules (Thm P:262-280)
PERIODIC, TRANSMISSIVE, HALO = 0, 1, 2
I32, I64 = 0, 1
ABI_VERSION = 3                                           # include/fqnm.h FQNM_ABI_VERSION
ROUND_HALF_AWAY, ROUND_FLOOR, ROUND_HALF_EVEN = 0, 1, 2
STATUS = {0: "FQNM_OK", 1: "FQNM_ERR_ARG", 2: "FQNM_ERR_CFL", 3: "FQNM_ERR_RANGE",
          4: "FQNM_ERR_CUDA", 5: "FQNM_ERR_UNSUPPORTED", 6: "FQNM_ERR_NOMEM"}

_HERE = os.path.dirname(os.path.abspath(__file__))


def lib_path() -> str:
    # FQNM_LIBPATH: alternative in-tree build (tools/tune.py variant sweeps only)
    return os.environ.get("FQNM_LIBPATH") or os.path.join(_HERE, "libfqnm.so")


class FqnmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class PlanDesc(ctypes.Structure):
    _fields_ = [
        ("n_local", ctypes.c_int64), ("n_global", ctypes.c_int64), ("offset", ctypes.c_int64),
        ("batch", ctypes.c_int64), ("nvar", ctypes.c_int32), ("dtype", ctypes.c_int32),
        ("delta", ctypes.c_double), ("dt_dx", ctypes.c_double), ("flux_kind", ctypes.c_int32),
        ("rounding", ctypes.c_int32), ("flux_param", ctypes.c_double),
        ("kappa_num", ctypes.c_int64), ("kappa_den", ctypes.c_int64),
        ("boundary", ctypes.c_int32), ("k", ctypes.c_int32),
        ("q_lo", ctypes.c_int64), ("q_hi", ctypes.c_int64), ("halo", ctypes.c_int64),
        ("check_range", ctypes.c_int32), ("p2p", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
    ]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("kappa_num", ctypes.c_int64), ("kappa_den", ctypes.c_int64),
        ("q_lo", ctypes.c_int64), ("q_hi", ctypes.c_int64),
        ("rule", ctypes.c_int32), ("k", ctypes.c_int32), ("cells_per_thread", ctypes.c_int32),
        ("kernel", ctypes.c_int32), ("scratch_bytes", ctypes.c_int64),
        ("s_euler", ctypes.c_double), ("g1_euler", ctypes.c_double),
        ("d8_lim", ctypes.c_int64), ("k2s_launches", ctypes.c_int64),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class LevelStats(ctypes.Structure):
    _fields_ = [("S", ctypes.c_double), ("N_eff", ctypes.c_double),
                ("occupied", ctypes.c_int64), ("outside", ctypes.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class TransitionStats(ctypes.Structure):
    _fields_ = [("before", LevelStats), ("after", LevelStats), ("rho", ctypes.c_double),
                ("dS", ctypes.c_double), ("nonzeros", ctypes.c_int64),
                ("overflow", ctypes.c_int64)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_}
        d["before"], d["after"] = self.before.as_dict(), self.after.as_dict()
        return d


class EquivalenceStats(ctypes.Structure):
    _fields_ = [("interface_evals", ctypes.c_int64), ("mismatches", ctypes.c_int64),
                ("first_mismatch_step", ctypes.c_int64), ("visited_pairs", ctypes.c_int64),
                ("mismatched_pairs", ctypes.c_int64), ("overflow", ctypes.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def _load():
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not os.path.exists(path):
        raise ImportError(f"libfqnm.so not built at {path}: run `python __graft_entry__.py build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    L.fqnm_plan.argtypes = [ctypes.POINTER(vp), i64, dbl, dbl, ctypes.c_int, ctypes.c_int]
    L.fqnm_plan_ex.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(PlanDesc)]
    L.fqnm_plan_2d.argtypes = [ctypes.POINTER(vp), i64, i64, dbl, dbl, dbl, ctypes.c_int,
                               ctypes.c_int, dbl, dbl]
    L.fqnm_plan_3d.argtypes = [ctypes.POINTER(vp), i64, i64, i64, dbl, dbl, dbl, dbl, ctypes.c_int,
                               ctypes.c_int, dbl, dbl, dbl]
    L.fqnm_desc_init.argtypes = [ctypes.POINTER(PlanDesc)]
    L.fqnm_desc_init.restype = None
    L.fqnm_destroy.argtypes = [vp]
    L.fqnm_destroy.restype = None
    L.fqnm_set_stream.argtypes = [vp, vp]
    L.fqnm_step.argtypes = [vp, vp, i64]
    L.fqnm_step_block.argtypes = [vp, vp, vp, i32]
    L.fqnm_observe.argtypes = [vp, vp, vp]
    L.fqnm_step_host.argtypes = [vp, vp, i64]
    L.fqnm_get_info.argtypes = [vp, ctypes.POINTER(PlanInfo)]
    L.fqnm_transfer.argtypes = [vp, i64, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.fqnm_transfer_device.argtypes = [vp, vp, vp, vp, i64]
    L.fqnm_roe_transfer_device.argtypes = [vp, vp, vp, vp, i64]
    L.fqnm_transfer2.argtypes = [vp, i64, i64, ctypes.POINTER(i64)]
    L.fqnm_transfer2_device.argtypes = [vp, vp, vp, vp, i64]
    L.fqnm_equivalence.argtypes = [vp, vp, vp, i64, i64, ctypes.POINTER(EquivalenceStats)]
    L.fqnm_debug_override.argtypes = [vp, i32, i32, i32]
    L.fqnm_debug_rcp_sqrt.argtypes = [i64, ctypes.c_uint64, i32, i32, ctypes.POINTER(ctypes.c_int64)]
    L.fqnm_plan_validate.argtypes = [ctypes.POINTER(PlanDesc), ctypes.POINTER(PlanInfo)]
    L.fqnm_profile_enable.argtypes = [vp, ctypes.c_int]
    L.fqnm_profile_read.argtypes = [vp, ctypes.POINTER(dbl), ctypes.POINTER(i64)]
    L.fqnm_halo_buffers.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp)]
    L.fqnm_halo_connect.argtypes = [vp, vp, vp, vp, i64, vp, vp, vp, i64]
    L.fqnm_halo_owned.argtypes = [vp, ctypes.POINTER(vp)]
    L.fqnm_step_group.argtypes = [ctypes.POINTER(vp), ctypes.c_int, i64]
    L.fqnm_ipc_export.argtypes = [vp, ctypes.c_char_p]
    L.fqnm_ipc_open.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
    L.fqnm_ipc_close.argtypes = [vp]
    L.fqnm_launch_count.argtypes = [vp]
    L.fqnm_levels.argtypes = [vp, vp, i64, i64, vp, ctypes.POINTER(LevelStats)]
    L.fqnm_transitions.argtypes = [vp, vp, vp, i64, i64, ctypes.POINTER(TransitionStats)]
    L.fqnm_launch_count.restype = i64
    L.fqnm_last_error.restype = ctypes.c_char_p
    L.fqnm_status_str.restype = ctypes.c_char_p
    L.fqnm_status_str.argtypes = [ctypes.c_int]
    L.fqnm_abi_version.restype = ctypes.c_int
    _lib = L
    return L


def _check(rc: int):
    if rc != 0:
        raise FqnmError(rc, _load().fqnm_last_error().decode())


def _stream_ptr(tensor=None):
    import torch
    dev = tensor.device if tensor is not None else None
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _dev_ptr(t, dtype=None, name="tensor"):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    return ctypes.c_void_p(t.data_ptr())


class Plan:
    """Owning handle of an fqnm_plan_t."""

    def __init__(self, handle: ctypes.c_void_p, desc: PlanDesc):
        self._h = handle
        self.desc = desc

    @property
    def handle(self):
        if not self._h:
            raise ValueError("plan destroyed")
        return self._h

    @property
    def dtype(self):
        import torch
        return torch.int64 if self.desc.dtype == I64 else torch.int32

    def state_shape(self):
        n = self.desc.n_local + (2 * self.desc.halo if self.desc.boundary == HALO else 0)
        shape = (self.desc.batch, self.desc.nvar, n)
        return tuple(s for s in shape[:-1] if s != 1) + (n,)

    def step(self, q, nsteps: int):
        return fqnm_step(self, q, nsteps)

    def step_block(self, src, dst, ksteps: int):
        return fqnm_step_block(self, src, dst, ksteps)

    def observe(self, q, u=None):
        return fqnm_observe(self, q, u)

    def info(self) -> dict:
        return fqnm_get_info(self)

    def launches(self) -> int:
        return fqnm_launch_count(self)

    def close(self):
        if self._h:
            _load().fqnm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def fqnm_plan(N: int, delta: float, dt_dx: float, flux_kind: int = LINEAR,
              boundary: int = PERIODIC) -> Plan:
    """North-star plan: one problem of N cells (include/fqnm.h fqnm_plan)."""
    L = _load()
    h = ctypes.c_void_p()
    _check(L.fqnm_plan(ctypes.byref(h), int(N), float(delta), float(dt_dx), int(flux_kind),
                       int(boundary)))
    d = PlanDesc()
    L.fqnm_desc_init(ctypes.byref(d))
    d.n_local = d.n_global = N
    d.delta, d.dt_dx, d.flux_kind, d.boundary = delta, dt_dx, flux_kind, boundary
    if flux_kind in (EULER_ROE, EULER_ROE_DENSITY):
        d.nvar, d.dtype = 3, I64
    d.check_range = 1 if flux_kind not in (EULER_ROE, EULER_ROE_DENSITY) else 0
    return Plan(h, d)


def fqnm_plan_2d(nx: int, ny: int, delta: float, dt_dx: float, dt_dy: float,
                 flux_kind: int = LINEAR, boundary: int = PERIODIC, param_x: float = 0.0,
                 param_y: float = 0.0) -> Plan:
    """2D directional-composition plan (include/fqnm.h fqnm_plan_2d); state [ny][nx] int32."""
    L = _load()
    h = ctypes.c_void_p()
    _check(L.fqnm_plan_2d(ctypes.byref(h), int(nx), int(ny), float(delta), float(dt_dx),
                          float(dt_dy), int(flux_kind), int(boundary), float(param_x),
                          float(param_y)))
    d = PlanDesc()
    L.fqnm_desc_init(ctypes.byref(d))
    d.n_local = d.n_global = nx * ny
    d.delta, d.dt_dx, d.flux_kind, d.boundary = delta, dt_dx, flux_kind, boundary
    d.check_range = 1
    return Plan(h, d)


def fqnm_plan_3d(nx: int, ny: int, nz: int, delta: float, dt_dx: float, dt_dy: float,
                 dt_dz: float, flux_kind: int = LINEAR, boundary: int = PERIODIC,
                 params=(0.0, 0.0, 0.0)) -> "Plan":
    """3D directional composition (Thm P:364-401, d = 3); state int32 [nz][ny][nx]."""
    L = _load()
    h = ctypes.c_void_p()
    _check(L.fqnm_plan_3d(ctypes.byref(h), int(nx), int(ny), int(nz), float(delta), float(dt_dx),
                          float(dt_dy), float(dt_dz), int(flux_kind), int(boundary),
                          float(params[0]), float(params[1]), float(params[2])))
    d = PlanDesc()
    L.fqnm_desc_init(ctypes.byref(d))
    d.n_local = d.n_global = int(nx) * int(ny) * int(nz)
    d.delta, d.dt_dx, d.flux_kind, d.boundary = delta, dt_dx, flux_kind, boundary
    d.check_range = 1
    return Plan(h, d)


def make_desc(n_local: int, delta: float, dt_dx: float, flux_kind: int = LINEAR,
              boundary: int = PERIODIC, *, batch: int = 1, nvar: Optional[int] = None,
              dtype: Optional[int] = None, flux_param: float = 0.0, kappa=None,
              rounding: int = ROUND_HALF_AWAY, q_range=None, k: int = 0, halo: int = 0,
              n_global: int = 0, offset: int = 0, check_range: bool = False,
              stream=None, p2p: bool = False) -> PlanDesc:
    L = _load()
    d = PlanDesc()
    L.fqnm_desc_init(ctypes.byref(d))
    euler = flux_kind in (EULER_ROE, EULER_ROE_DENSITY)
    d.n_local = n_local
    d.n_global = n_global or n_local
    d.offset = offset
    d.batch = batch
    d.nvar = nvar if nvar is not None else (3 if euler else 1)
    d.dtype = dtype if dtype is not None else (I64 if euler else I32)
    d.delta, d.dt_dx = float(delta), float(dt_dx)
    d.flux_kind, d.rounding = int(flux_kind), int(rounding)
    d.flux_param = float(flux_param)
    if kappa is not None:
        d.kappa_num, d.kappa_den = int(kappa[0]), int(kappa[1])
    d.boundary = int(boundary)
    d.k = int(k)
    if q_range is not None:
        d.q_lo, d.q_hi = int(q_range[0]), int(q_range[1])
    d.halo = int(halo)
    d.check_range = 1 if check_range else 0
    d.p2p = 1 if p2p else 0
    d.stream = stream
    return d


def fqnm_plan_ex(n_local: int, delta: float, dt_dx: float, flux_kind: int = LINEAR,
                 boundary: int = PERIODIC, **kw) -> Plan:
    """General plan (include/fqnm.h fqnm_plan_ex); kappa = (num, den) overrides."""
    d = make_desc(n_local, delta, dt_dx, flux_kind, boundary, **kw)
    h = ctypes.c_void_p()
    _check(_load().fqnm_plan_ex(ctypes.byref(h), ctypes.byref(d)))
    return Plan(h, d)


def fqnm_plan_validate(n_local: int, delta: float, dt_dx: float, flux_kind: int = LINEAR,
                       boundary: int = PERIODIC, **kw) -> dict:
    """Host-only rule building + kernel selection (no GPU needed)."""
    d = make_desc(n_local, delta, dt_dx, flux_kind, boundary, **kw)
    info = PlanInfo()
    _check(_load().fqnm_plan_validate(ctypes.byref(d), ctypes.byref(info)))
    return info.as_dict()


def fqnm_profile_enable(plan: Plan, enable: bool = True):
    _check(_load().fqnm_profile_enable(plan.handle, 1 if enable else 0))


def fqnm_profile_read(plan: Plan):
    """(summed device ms, number of bracketed stepping-kernel launches) since last read."""
    ms, n = ctypes.c_double(), ctypes.c_int64()
    _check(_load().fqnm_profile_read(plan.handle, ctypes.byref(ms), ctypes.byref(n)))
    return ms.value, n.value


def fqnm_step(plan: Plan, q, nsteps: int):
    """q <- q^{n+nsteps} in place (device tensor of the plan's dtype/layout).
    p2p split plans: q is None (the state lives in the plan's buffers)."""
    L = _load()
    if q is None:
        _check(L.fqnm_set_stream(plan.handle, _stream_ptr()))
        _check(L.fqnm_step(plan.handle, None, int(nsteps)))
        return None
    ptr = _dev_ptr(q, plan.dtype, "q")
    if q.numel() != _numel(plan):
        raise ValueError(f"q has {q.numel()} elements, plan expects {_numel(plan)}")
    _check(L.fqnm_set_stream(plan.handle, _stream_ptr(q)))
    _check(L.fqnm_step(plan.handle, ptr, int(nsteps)))
    return q


def fqnm_step_block(plan: Plan, src, dst, ksteps: int):
    L = _load()
    s = _dev_ptr(src, plan.dtype, "src")
    t = _dev_ptr(dst, plan.dtype, "dst")
    _check(L.fqnm_set_stream(plan.handle, _stream_ptr(src)))
    _check(L.fqnm_step_block(plan.handle, s, t, int(ksteps)))
    return dst


def fqnm_observe(plan: Plan, q, u=None):
    """u = fl(delta q) as a float64 device tensor of q's shape."""
    import torch
    L = _load()
    ptr = _dev_ptr(q, plan.dtype, "q")
    if u is None:
        u = torch.empty(q.shape, dtype=torch.float64, device=q.device)
    uptr = _dev_ptr(u, torch.float64, "u")
    _check(L.fqnm_set_stream(plan.handle, _stream_ptr(q)))
    _check(L.fqnm_observe(plan.handle, ptr, uptr))
    return u


def fqnm_step_host(plan: Plan, q_host, nsteps: int):
    """End-to-end: host buffer (pinned torch CPU tensor or numpy array) stepped in place.
    The C side copies state_elems x sizeof(dtype) bytes into and out of the pointer, so the
    buffer's element count and dtype are checked against the plan here."""
    L = _load()
    want = _numel(plan)
    is_i64 = plan.desc.dtype == I64
    try:
        import torch
        if isinstance(q_host, torch.Tensor):
            if q_host.is_cuda or not q_host.is_contiguous():
                raise ValueError("q_host must be a contiguous CPU tensor")
            if q_host.dtype != (torch.int64 if is_i64 else torch.int32):
                raise TypeError(f"q_host must be {'int64' if is_i64 else 'int32'}, got {q_host.dtype}")
            if q_host.numel() != want:
                raise ValueError(f"q_host has {q_host.numel()} elements, plan expects {want}")
            ptr = ctypes.c_void_p(q_host.data_ptr())
            _check(L.fqnm_set_stream(plan.handle, _stream_ptr()))
            _check(L.fqnm_step_host(plan.handle, ptr, int(nsteps)))
            return q_host
    except ImportError:  # pragma: no cover
        pass
    import numpy as np
    a = q_host
    if not (isinstance(a, np.ndarray) and a.flags.c_contiguous):
        raise TypeError("q_host must be a contiguous numpy array or CPU tensor")
    if a.dtype != (np.int64 if is_i64 else np.int32):
        raise TypeError(f"q_host must be {'int64' if is_i64 else 'int32'}, got {a.dtype}")
    if a.size != want:
        raise ValueError(f"q_host has {a.size} elements, plan expects {want}")
    _check(L.fqnm_step_host(plan.handle, ctypes.c_void_p(a.ctypes.data), int(nsteps)))
    return a


def fqnm_levels(plan: Plan, q, lo: int, hi: int, counts=None) -> dict:
    """Level histogram statistics of q (SI Eq. pk / discrete_entropy / neff):
    {S, N_eff, occupied, outside}; `counts` (optional uint32-sized int32 CUDA
    tensor of hi - lo + 1) receives c_k."""
    import torch
    L = _load()
    ptr = _dev_ptr(q, plan.dtype, "q")
    cptr = None
    if counts is not None:
        if counts.numel() != hi - lo + 1 or counts.element_size() != 4:
            raise ValueError("counts must hold hi - lo + 1 32-bit entries")
        cptr = _dev_ptr(counts, None, "counts")
    st = LevelStats()
    _check(L.fqnm_set_stream(plan.handle, _stream_ptr(q)))
    _check(L.fqnm_levels(plan.handle, ptr, int(lo), int(hi), cptr, ctypes.byref(st)))
    return st.as_dict()


def fqnm_transitions(plan: Plan, q0, q1, lo: int, hi: int) -> dict:
    """Level-transition statistics q0 -> q1 (SI Def. level_transition, row-sum
    defect rho): {before, after, rho, dS, nonzeros, overflow}."""
    L = _load()
    p0 = _dev_ptr(q0, plan.dtype, "q0")
    p1 = _dev_ptr(q1, plan.dtype, "q1")
    st = TransitionStats()
    _check(L.fqnm_set_stream(plan.handle, _stream_ptr(q0)))
    _check(L.fqnm_transitions(plan.handle, p0, p1, int(lo), int(hi), ctypes.byref(st)))
    return st.as_dict()


def _numel(plan: Plan) -> int:
    d = plan.desc
    n = d.n_local + (2 * d.halo if d.boundary == HALO else 0)
    return d.batch * d.nvar * n


def fqnm_get_info(plan: Plan) -> dict:
    info = PlanInfo()
    _check(_load().fqnm_get_info(plan.handle, ctypes.byref(info)))
    return info.as_dict()


def fqnm_transfer(plan: Plan, q: int):
    a, b = ctypes.c_int64(), ctypes.c_int64()
    _check(_load().fqnm_transfer(plan.handle, int(q), ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def fqnm_transfer_device(plan: Plan, q):
    import torch
    p = torch.empty_like(q)
    m = torch.empty_like(q)
    L = _load()
    qp = _dev_ptr(q, torch.int32, "q")
    _check(L.fqnm_set_stream(plan.handle, _stream_ptr(q)))
    _check(L.fqnm_transfer_device(plan.handle, qp, _dev_ptr(p), _dev_ptr(m), q.numel()))
    return p, m


def fqnm_transfer2(plan: Plan, qL: int, qR: int) -> int:
    """Host evaluation of the interface transfer Phi(qL, qR) of a scalar plan."""
    t = ctypes.c_int64()
    _check(_load().fqnm_transfer2(plan.handle, int(qL), int(qR), ctypes.byref(t)))
    return t.value


def fqnm_transfer2_device(plan: Plan, qL, qR):
    """The kernels' interface-transfer code on int32 device tensors qL, qR."""
    import torch
    T = torch.empty_like(qL)
    L = _load()
    a = _dev_ptr(qL, torch.int32, "qL")
    b = _dev_ptr(qR, torch.int32, "qR")
    if qR.numel() != qL.numel():
        raise ValueError("qL and qR must have the same size")
    _check(L.fqnm_set_stream(plan.handle, _stream_ptr(qL)))
    _check(L.fqnm_transfer2_device(plan.handle, a, b, _dev_ptr(T), qL.numel()))
    return T


def fqnm_equivalence(plan_a: Plan, plan_b: Plan, q, nsteps: int, pair_capacity: int = 0) -> dict:
    """Thm transfer-operator equivalence check: advance q (int32 device tensor, in
    place) by nsteps of plan_a's rule, evaluating plan_b's transfer on every visited
    interface state.  Synchronous; returns the statistics as a dict."""
    import torch
    L = _load()
    qp = _dev_ptr(q, torch.int32, "q")
    st = EquivalenceStats()
    _check(L.fqnm_set_stream(plan_a.handle, _stream_ptr(q)))
    _check(L.fqnm_equivalence(plan_a.handle, plan_b.handle, qp, int(nsteps), int(pair_capacity),
                              ctypes.byref(st)))
    return st.as_dict()


def fqnm_roe_transfer_device(plan: Plan, qL, qR):
    """qL, qR: [3][n] int64 device tensors; returns T [3][n]."""
    import torch
    T = torch.empty_like(qL)
    L = _load()
    a = _dev_ptr(qL, torch.int64, "qL")
    b = _dev_ptr(qR, torch.int64, "qR")
    _check(L.fqnm_set_stream(plan.handle, _stream_ptr(qL)))
    _check(L.fqnm_roe_transfer_device(plan.handle, a, b, _dev_ptr(T), qL.shape[-1]))
    return T


def fqnm_debug_override(plan: Plan, kernel: int = 0, k: int = 0, cells_per_thread: int = 0):
    _check(_load().fqnm_debug_override(plan.handle, int(kernel), int(k), int(cells_per_thread)))


def fqnm_debug_rcp_sqrt(n: int, seed: int = 0, e_lo: int = -60, e_hi: int = 60):
    """(rcp mismatches, sqrt mismatches, range flags, div mismatches) of the Euler kernel's
    own 1/x, sqrt and x/y sequences against the CUDA library's correctly rounded ones on n
    random doubles."""
    out = (ctypes.c_int64 * 4)()
    _check(_load().fqnm_debug_rcp_sqrt(int(n), int(seed), int(e_lo), int(e_hi), out))
    return int(out[0]), int(out[1]), int(out[2]), int(out[3])


# ---- fused peer-memory halo exchange --------------------------------------
def fqnm_halo_buffers(plan: Plan):
    """(buf0, buf1, flags) device pointers (ints) owned by a p2p split plan."""
    b0, b1, fl = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    _check(_load().fqnm_halo_buffers(plan.handle, ctypes.byref(b0), ctypes.byref(b1),
                                     ctypes.byref(fl)))
    return b0.value, b1.value, fl.value


def fqnm_halo_connect(plan: Plan, left, left_n: int, right, right_n: int):
    """left/right = (buf0, buf1, flags) device pointers of the ring neighbours."""
    _check(_load().fqnm_halo_connect(plan.handle, ctypes.c_void_p(left[0]), ctypes.c_void_p(left[1]),
                                     ctypes.c_void_p(left[2]), int(left_n),
                                     ctypes.c_void_p(right[0]), ctypes.c_void_p(right[1]),
                                     ctypes.c_void_p(right[2]), int(right_n)))


def fqnm_halo_owned(plan: Plan) -> int:
    """Device pointer (int) to the owned cells of the plan's current buffer."""
    o = ctypes.c_void_p()
    _check(_load().fqnm_halo_owned(plan.handle, ctypes.byref(o)))
    return o.value


def fqnm_step_group(plans, nsteps: int):
    """Step p2p plans of one device together (virtual ranks)."""
    arr = (ctypes.c_void_p * len(plans))(*[p.handle for p in plans])
    for p in plans:
        _check(_load().fqnm_set_stream(p.handle, _stream_ptr()))
    _check(_load().fqnm_step_group(arr, len(plans), int(nsteps)))


def fqnm_ipc_export(ptr: int) -> bytes:
    buf = ctypes.create_string_buffer(64)
    _check(_load().fqnm_ipc_export(ctypes.c_void_p(ptr), buf))
    return buf.raw


def fqnm_ipc_open(handle: bytes) -> int:
    o = ctypes.c_void_p()
    _check(_load().fqnm_ipc_open(ctypes.c_char_p(handle), ctypes.byref(o)))
    return o.value


def fqnm_ipc_close(ptr: int):
    _check(_load().fqnm_ipc_close(ctypes.c_void_p(ptr)))


def owned_tensor(plan: Plan):
    """torch view (int32, CUDA) of a p2p plan's owned cells (current buffer)."""
    import torch
    ptr = fqnm_halo_owned(plan)
    n = plan.desc.n_local
    dev = torch.cuda.current_device()
    # wrap the raw device pointer through a zero-copy DLPack-free path
    return _wrap_device(ptr, n, torch.int32, dev)


def _wrap_device(ptr: int, n: int, dtype, device: int):
    import torch

    class _CAI:
        def __init__(self):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i4", "data": (ptr, False),
                                             "version": 3, "strides": None}
    return torch.as_tensor(_CAI(), device=f"cuda:{device}")


def fqnm_launch_count(plan: Plan) -> int:
    return int(_load().fqnm_launch_count(plan.handle))


def fqnm_destroy(plan: Plan):
    plan.close()


def abi_version() -> int:
    return int(_load().fqnm_abi_version())
