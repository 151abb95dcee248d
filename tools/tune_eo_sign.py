"""cfg4 slices through the range-checked north-star plan (so a one-signed state selects the
sign-specialised kernels): K2 (2), K2S (22), K2P voting (12), K2PS (32), auto (0).
usage: python tools/tune_eo_sign.py [log2 n] [steps] [fam,...]"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2604_06947_b200 as F
import workloads as W

ln = int(sys.argv[1]) if len(sys.argv) > 1 else 28
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 192
fams = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "0,2,22,12,32").split(",")]
n = 1 << ln
q0 = W.q0_cfg4(n=1 << 31, count=n, device="cuda")
qmax = int(q0.abs().max())
dt_dx = W.dt_dx_double(W.cfg("cfg4"), qmax)
for fam in fams:
    plan = F.fqnm_plan(n, 1e-6, dt_dx, F.BURGERS_EO, F.PERIODIC)
    if fam:
        F.fqnm_debug_override(plan, fam, int(os.environ.get("TUNE_K", 0)), 0)
    q = q0.clone()
    F.fqnm_step(plan, q, steps)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); F.fqnm_step(plan, q, steps); e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    sha = hashlib.sha256(q.cpu().numpy().tobytes()).hexdigest()[:16] if ln <= 28 else ""
    info = plan.info()
    print(json.dumps({"fam": fam, "log2n": ln, "steps": steps, "ms": best, "GCUPS": n * steps / best / 1e6,
                      "k": info["k"], "k2s_launches": info["k2s_launches"], "sha": sha}), flush=True)
    del q, plan
    torch.cuda.empty_cache()
