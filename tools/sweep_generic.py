"""Throughput of the K2 paths planned without a register cap (minb = 0: LIN_FAST, GENERIC,
exact two-point) on a 2^26-cell slice of cfg4 data; FQNM_LIBPATH selects the build.
Prints GCUPS and a sha of the final state per rule."""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch
import paper_2604_06947_b200 as F
import workloads as W

n, steps = 1 << 26, 96
q0 = W.q0_cfg4(n=1 << 31, count=n, device="cuda")
qmax = int(q0.abs().max())
lam = W.dt_dx_double(W.cfg("cfg4"), qmax)
umax = qmax * 1e-6
for name, kind, lm, fp in (("linear_quarter", F.LINEAR, 0.25, 1.0),
                           ("burgers_lf", F.BURGERS_LF, lam / 2, umax),
                           ("burgers_eo2", F.BURGERS_EO2, lam, 0.0)):
    plan = F.fqnm_plan_ex(n, 1e-6, lm, kind, F.PERIODIC, flux_param=fp)
    q = q0.clone()
    F.fqnm_step(plan, q, steps)
    torch.cuda.synchronize()
    sha = hashlib.sha1(q.cpu().numpy().tobytes()).hexdigest()[:12]
    best = 1e30
    for _ in range(3):
        q.copy_(q0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        F.fqnm_step(plan, q, steps)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(json.dumps({"tag": os.environ.get("TAG", ""), "rule": name, "info_rule": plan.info()["rule"],
                      "GCUPS": round(n * steps / best / 1e6, 1), "sha": sha}), flush=True)
