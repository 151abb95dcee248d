"""Small driver for ncu captures: one fqnm_step of a bench workload slice.
usage: python tools/prof_step.py eo|lin|euler|2d|3d [n] [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch
import paper_2604_06947_b200 as F
import workloads as W

which = sys.argv[1] if len(sys.argv) > 1 else "eo"
if which == "eo":
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 28
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 32
    q = W.q0_cfg4(n=1 << 31, count=n, device="cuda")
    qmax = int(q.abs().max())
    plan = F.fqnm_plan(n, 1e-6, W.dt_dx_double(W.cfg("cfg4"), qmax), F.BURGERS_EO, F.PERIODIC)
elif which == "lin":
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 24
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 128
    q = torch.tensor(W.q0_cfg3(n), dtype=torch.int32, device="cuda")
    plan = F.fqnm_plan(n, 1e-6, 0.5, F.LINEAR, F.PERIODIC)
elif which == "2d":
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    q = torch.randint(-100000, 100000, (n, n), dtype=torch.int32, device="cuda")
    plan = F.fqnm_plan_2d(n, n, 1e-5, 1 / 15, 1 / 15, F.BURGERS_EO, F.PERIODIC)
elif which == "3d":
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    q = torch.randint(-100000, 100000, (n, n, n), dtype=torch.int32, device="cuda")
    plan = F.fqnm_plan_3d(n, n, n, 1e-5, 1 / 15, 1 / 15, 1 / 15, F.BURGERS_EO, F.PERIODIC)
else:
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 22
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    _, lam = W.sod_steps_and_dt_dx(1 << 26)
    q = torch.tensor(W.sod_q0(n), dtype=torch.int64, device="cuda")
    plan = F.fqnm_plan(n, 1e-7, lam, F.EULER_ROE, F.TRANSMISSIVE)
F.fqnm_step(plan, q, steps)
torch.cuda.synchronize()
print(which, n, steps, plan.info())
