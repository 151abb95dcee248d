"""cfg2 (K6) probe: the BJ data (sign-changing) against an all-positive state of the same
amplitude, to separate the cost of the mixed-sign windows (general step) from the rest."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2604_06947_b200 as F
import workloads as W

w = W.cfg("cfg2")
x = W.cell_centres(w.n)
for name, u in (("bj", 0.5 + np.sin(2 * np.pi * x)), ("positive", 1.6 + np.sin(2 * np.pi * x) * 0.0 + 0.5 * np.sin(2 * np.pi * x))):
    q0 = torch.tensor(W.quantise(u, 1e-5), dtype=torch.int32, device="cuda")
    qmax = int(q0.abs().max())
    plan = F.fqnm_plan(w.n, 1e-5, W.dt_dx_double(w, qmax), F.BURGERS_EO, F.PERIODIC)
    if os.environ.get("CFG2_K"):
        F.fqnm_debug_override(plan, 6, int(os.environ["CFG2_K"]), 8)
    q = q0.clone()
    F.fqnm_step(plan, q, w.steps)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        q.copy_(q0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); F.fqnm_step(plan, q, w.steps); e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(json.dumps({"data": name, "lib": os.path.basename(os.environ.get("FQNM_LIBPATH", "default")),
                      "ms": best, "k": plan.info()["k"], "kernel": plan.info()["kernel"]}))
