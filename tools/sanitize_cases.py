"""Small invocations of every stepping-kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).  Each case also
checks its result against the CPU oracle, so a run under the sanitizer is a parity run
too.  usage: compute-sanitizer --tool <t> python tools/sanitize_cases.py [case ...]"""
import os
import sys
from fractions import Fraction

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import oracle
import paper_2604_06947_b200 as F
import workloads as W

DEV = "cuda"
EO = (W.BURGERS_EO, "1e-5", Fraction(4, 15))


def dev(q):
    return torch.tensor(np.asarray(q), dtype=torch.int32, device=DEV)


def check(name, got, ref):
    ok = np.array_equal(got.cpu().numpy().astype(np.int64), ref)
    print(f"{name}: {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        sys.exit(1)


def data(n, signed=False, seed=0):
    rng = np.random.default_rng(seed)
    return W.smooth_random(rng, n, 100000, 0 if signed else 20000)


def k2(kernel=2, V=32, signed=True):
    n = 3 * 1024 + 77
    q0 = data(n, signed)
    plan = F.fqnm_plan_ex(n, 1e-5, float(EO[2]), W.BURGERS_EO)
    F.fqnm_debug_override(plan, kernel, 0, V if kernel == 2 else 0)
    q = dev(q0)
    F.fqnm_step(plan, q, 40)
    check(f"K{kernel} V={V} signed={signed}", q, oracle.Rule(*EO).run(q0, 40))


def k2_transmissive():
    n = 2 * 1024 + 5
    q0 = data(n, True, 3)
    plan = F.fqnm_plan_ex(n, 1e-5, float(EO[2]), W.BURGERS_EO, W.TRANSMISSIVE)
    F.fqnm_debug_override(plan, 2, 0, 16)
    q = dev(q0)
    F.fqnm_step(plan, q, 30)
    check("K2 transmissive", q, oracle.Rule(*EO).run(q0, 30, W.TRANSMISSIVE))


def k6():
    n = 20000 + 13
    q0 = data(n, True, 1)
    plan = F.fqnm_plan_ex(n, 1e-5, float(EO[2]), W.BURGERS_EO)
    assert plan.info()["kernel"] == 6
    q = dev(q0)
    F.fqnm_step(plan, q, 50)
    check("K6 resident", q, oracle.Rule(*EO).run(q0, 50))


def k2p():
    n = 8 * 1024 + 3
    q0 = data(n, False, 2)
    plan = F.fqnm_plan_ex(n, 1e-5, float(EO[2]), W.BURGERS_EO)
    F.fqnm_debug_override(plan, 12, 8, 0)
    q = dev(q0)
    F.fqnm_step(plan, q, 40)
    check("K2P persistent", q, oracle.Rule(*EO).run(q0, 40))


def p2p():
    from paper_2604_06947_b200 import halo
    n = 6000 + 7
    q0 = data(n, True, 4)
    ref = oracle.Rule(*EO).run(q0, 30)
    for P, H in [(2, 16), (3, 8)]:
        parts = [halo.partition(n, P, r) for r in range(P)]
        plans = [F.fqnm_plan_ex(nl, 1e-5, float(EO[2]), W.BURGERS_EO, F.HALO, halo=H,
                                n_global=n, offset=o, p2p=True) for o, nl in parts]
        ring = halo.P2PRing.virtual(plans)
        ring.load([dev(q0[o:o + nl]) for o, nl in parts])
        ring.step(30)
        got = torch.cat([ring.owned(i) for i in range(P)])
        check(f"K2 p2p virtual ranks P={P}", got, ref)


def k3_k4():
    for n, B in [(1024, 5), (3000, 3)]:
        rng = np.random.default_rng(n)
        q0 = np.stack([W.smooth_random(rng, n, 5000, 0) for _ in range(B)])
        rule = oracle.Rule(W.LINEAR, "1e-4", Fraction(1, 2))
        plan = F.fqnm_plan_ex(n, 1e-4, 0.5, W.LINEAR, batch=B)
        q = dev(q0).reshape(-1)
        F.fqnm_step(plan, q, 60)
        check(f"K{plan.info()['kernel']} ensemble n={n}", q.view(B, n), rule.run(q0, 60))


def k7_k9():
    ny, nx = 40, 300
    rng = np.random.default_rng(5)
    q0 = W.smooth_random(rng, ny * nx, 100000, 20000).reshape(ny, nx)
    lam = Fraction(2, 15)
    ref = oracle.Rule2D(W.BURGERS_EO, "1e-5", lam, lam).run(q0, 5)
    for kern in (9, 7):
        plan = F.fqnm_plan_2d(nx, ny, 1e-5, float(lam), float(lam), W.BURGERS_EO)
        F.fqnm_debug_override(plan, kern, 0, 0)
        q = dev(q0)
        F.fqnm_step(plan, q, 5)
        check(f"K{kern} 2D", q, ref)


def k8_k10():
    nz, ny, nx = 6, 20, 130
    rng = np.random.default_rng(6)
    q0 = W.smooth_random(rng, nz * ny * nx, 50000, 10000).reshape(nz, ny, nx)
    lam = Fraction(1, 15)
    ref = oracle.Rule3D(W.BURGERS_EO, "1e-5", lam, lam, lam).run(q0, 3)
    for kern in (8, 10):
        plan = F.fqnm_plan_3d(nx, ny, nz, 1e-5, float(lam), float(lam), float(lam), W.BURGERS_EO)
        F.fqnm_debug_override(plan, kern, 0, 0)
        q = dev(q0)
        F.fqnm_step(plan, q, 3)
        check(f"K{kern} 3D", q, ref)


def k5():
    n = 300
    nsteps, lam = W.sod_steps_and_dt_dx(n)
    q0 = W.sod_q0(n)
    plan = F.fqnm_plan(n, 1e-7, lam, F.EULER_ROE, F.TRANSMISSIVE)
    q = torch.tensor(q0, dtype=torch.int64, device=DEV)
    F.fqnm_step(plan, q, 20)
    check("K5 Euler/Roe", q, oracle.euler_run(q0, 20, 1e-7, lam))


CASES = {"k2": lambda: (k2(2, 32, True), k2(2, 8, False), k2_transmissive()),
         "k1": lambda: k2(1), "k6": k6, "k2p": k2p, "p2p": p2p, "ens": k3_k4,
         "2d": k7_k9, "3d": k8_k10, "euler": k5}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        CASES[nm]()
    torch.cuda.synchronize()
    print("all cases ok")
