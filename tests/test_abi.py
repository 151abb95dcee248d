"""CPU-only checks of the C-ABI library: it loads, exports every symbol that
include/fqnm.h declares, and its host-side rule builder (fqnm_plan_validate,
no GPU needed) derives the exact rules and rejects invalid ones."""
import ctypes
import os
import re
from fractions import Fraction

import pytest

import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def F():
    from paper_2604_06947_b200 import _build
    _build.build()
    import paper_2604_06947_b200 as F
    F._load()
    return F


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "fqnm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(fqnm_[a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_exports_every_declared_symbol(F):
    names = _declared_functions()
    assert len(names) >= 20
    lib = ctypes.CDLL(F.lib_path())
    for n in names:
        assert hasattr(lib, n), f"libfqnm.so does not export {n}"
    assert F.abi_version() == F.ABI_VERSION == 3


def test_library_is_sm100a_only(F):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", F.lib_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings(F):
    L = F._load()
    assert L.fqnm_status_str(0) == b"FQNM_OK"
    assert L.fqnm_status_str(2) == b"FQNM_ERR_CFL"


@pytest.mark.parametrize("name,qmax,expect", [
    ("cfg1", None, (1, 2)), ("cfg3", None, (1, 2)),
    ("cfg2", 150000, (1, 750000)), ("cfg4", 1_183_254, (1, 5 * 1_183_254))])
def test_kappa_rationalised_from_doubles(F, name, qmax, expect):
    """The plan recovers the exact kappa of the config from the double dt/dx a
    user passes (continued fraction), equal to the oracle's Fraction value."""
    import oracle.rules as R
    w = W.cfg(name)
    info = F.fqnm_plan_validate(w.n, float(w.delta), W.dt_dx_double(w, qmax), w.kind)
    k = R.kappa(w.kind, w.delta, W.dt_dx(w, qmax))
    assert (info["kappa_num"], info["kappa_den"]) == (k.numerator, k.denominator) == expect


def test_rule_and_kernel_selection(F):
    w4 = W.cfg("cfg4")
    info = F.fqnm_plan_validate(w4.n, 1e-6, W.dt_dx_double(w4, 1_200_000), F.BURGERS_EO)
    assert info["rule"] == 5 and info["kernel"] == 2           # EO fast path (P = 1), blocked kernel
    assert info["q_hi"] >= 2_400_000 and info["q_lo"] == -info["q_hi"]
    info = F.fqnm_plan_validate(1 << 24, 1e-5, 0.3, F.BURGERS_EO)   # kappa = 3/2e6, P = 3
    assert info["rule"] == 2 and info["kappa_num"] == 3
    info = F.fqnm_plan_validate(1 << 24, 1e-6, 0.5, F.LINEAR)
    assert info["rule"] == 1 and info["kernel"] == 2
    info = F.fqnm_plan_validate(1024, 1e-4, 0.5, F.LINEAR, batch=1 << 16)
    assert info["kernel"] == 3 and info["cells_per_thread"] == 32
    info = F.fqnm_plan_validate(1000, 1e-4, 0.5, F.LINEAR)
    assert info["kernel"] == 4
    info = F.fqnm_plan_validate(65536, 1e-5, 4 / 15, F.BURGERS_EO)      # cfg2: resident stepper
    assert info["kernel"] == 6
    # K6 geometry from the time model: the deepest halo whose warps still fit one per SM
    # sub-partition (4 x 148): n / (256 - 2k) <= 592 -> k = 72, P = 586
    assert info["k"] == 72 and info["cells_per_thread"] == 8
    assert -(-65536 // (256 - 2 * info["k"])) <= 4 * 148
    info = F.fqnm_plan_validate(150000, 1e-5, 4 / 15, F.BURGERS_EO)     # needs > 592 warps at any k
    assert info["kernel"] == 6 and 8 <= info["k"] <= 124 and info["k"] % 4 == 0
    assert -(-150000 // (256 - 2 * info["k"])) <= 8 * 148
    info = F.fqnm_plan_validate(1 << 26, 1e-7, 0.3, F.EULER_ROE, F.TRANSMISSIVE)
    assert info["kernel"] == 5 and info["s_euler"] == 0.3 / 1e-7 and info["g1_euler"] == 1.4 - 1.0
    assert info["cells_per_thread"] == 2                               # large problems: V = 2
    assert F.fqnm_plan_validate(4096, 1e-7, 0.3, F.EULER_ROE, F.TRANSMISSIVE)["cells_per_thread"] == 1


def test_d8_admissible_range_matches_oracle(F):
    """The derived symmetric range is exactly where the oracle's maps satisfy D8."""
    import numpy as np
    import oracle
    lam = Fraction(4, 15)
    info = F.fqnm_plan_validate(65536, 1e-5, float(lam), F.BURGERS_EO)
    A = info["q_hi"]
    r = oracle.Rule(oracle.BURGERS_EO, "1e-5", lam)
    q = np.arange(-A - 2, A + 3)
    dp, dm = np.diff(r.phi_plus(q)), np.diff(r.phi_minus(q))
    ok = (dp >= 0) & (dm <= 0) & (dp - dm <= 1)
    inner = ok[2:-2]                                  # steps q -> q+1 for q in [-A, A-1]
    assert inner.all()
    assert not ok[-2] or not ok[1]                     # D8 fails right outside [-A, A]


@pytest.mark.parametrize("kw,status", [
    (dict(n_local=1, delta=1e-4, dt_dx=0.5, flux_kind=0), 1),
    (dict(n_local=64, delta=-1.0, dt_dx=0.5, flux_kind=0), 1),
    (dict(n_local=64, delta=float("nan"), dt_dx=0.5, flux_kind=0), 1),
    (dict(n_local=64, delta=1e-4, dt_dx=0.0, flux_kind=0), 1),
    (dict(n_local=64, delta=1e-4, dt_dx=1.25, flux_kind=0), 2),              # nu > 1
    (dict(n_local=64, delta=1e-3, dt_dx=1 / 3, flux_kind=2, flux_param=1.2,
          q_range=(-1200, 1200)), 2),                                        # LF breaks D8
    (dict(n_local=64, delta=1e-4, dt_dx=0.5, flux_kind=9), 1),                # unknown kind
    (dict(n_local=64, delta=1e-4, dt_dx=0.5, flux_kind=7), 1),                # LF2 needs alpha
    (dict(n_local=64, delta=1e-4, dt_dx=0.5, flux_kind=0, boundary=9), 1),
    (dict(n_local=64, delta=1e-4, dt_dx=0.5, flux_kind=3), 1),               # Euler needs nvar 3
])
def test_invalid_plans_are_rejected(F, kw, status):
    n = kw.pop("n_local")
    d, lam, kind = kw.pop("delta"), kw.pop("dt_dx"), kw.pop("flux_kind")
    if kind == 3:
        kw.update(nvar=1, dtype=0)
    with pytest.raises(F.FqnmError) as e:
        F.fqnm_plan_validate(n, d, lam, kind, **kw)
    assert e.value.status == status


def test_gpu_entry_points_fail_loudly_without_gpu(F):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(F.FqnmError):
        F.fqnm_plan(1024, 1e-4, 0.5, F.LINEAR, F.PERIODIC)
    with pytest.raises(TypeError):
        q = torch.zeros(8, dtype=torch.int32)
        plan = F.Plan(ctypes.c_void_p(), F.make_desc(8, 1e-4, 0.5))
        F.fqnm_step(plan, q, 1)


def test_two_point_rules_validate(F):
    """Two-point kinds (Thm P:262-280) build R_TWOPOINT (6) with the admissible range
    of their split counterpart and the same kappa."""
    for kind, split in ((F.BURGERS_GODUNOV, F.BURGERS_EO), (F.BURGERS_EO2, F.BURGERS_EO)):
        info = F.fqnm_plan_validate(65536, 1e-5, 4 / 15, kind)
        ref = F.fqnm_plan_validate(65536, 1e-5, 4 / 15, split)
        assert info["rule"] == (7 if kind == F.BURGERS_GODUNOV else 6)   # Godunov: EO fast form
        assert (info["kappa_num"], info["kappa_den"]) == (ref["kappa_num"], ref["kappa_den"])
        assert (info["q_lo"], info["q_hi"]) == (ref["q_lo"], ref["q_hi"])
        assert info["kernel"] == ref["kernel"]
    info = F.fqnm_plan_validate(1 << 20, 1e-3, 0.5, F.BURGERS_LF2, flux_param=1.0)
    ref = F.fqnm_plan_validate(1 << 20, 1e-3, 0.5, F.BURGERS_LF, flux_param=1.0)
    assert info["rule"] == 6 and info["kernel"] == 2 and info["cells_per_thread"] == 8
    assert (info["q_lo"], info["q_hi"]) == (ref["q_lo"], ref["q_hi"])
