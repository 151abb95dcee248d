"""Sweep (V, k) of the temporally blocked kernel on the bench workloads (GPU).
Prints one JSON line per setting: GCUPS and kernel ms."""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch
import paper_2604_06947_b200 as F
import workloads as W


def run(plan, q, steps, reps=3):
    F.fqnm_step(plan, q, steps)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        F.fqnm_step(plan, q, steps)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "eo"
    if which == "eo":
        n = int(os.environ.get("TUNE_N", 1 << 30))
        steps = int(os.environ.get("TUNE_STEPS", 192))
        q0 = W.q0_cfg4(n=1 << 31, count=n, device="cuda")
        qmax = int(q0.abs().max())
        dt_dx = W.dt_dx_double(W.cfg("cfg4"), qmax)
        kind = F.BURGERS_EO
        Vs, ks = [8, 16, 32], [8, 12, 16, 24, 32]
    else:
        n = int(os.environ.get("TUNE_N", 1 << 24))
        steps = int(os.environ.get("TUNE_STEPS", 2048))
        q0 = torch.tensor(W.q0_cfg3(n), dtype=torch.int32, device="cuda")
        dt_dx = 0.5
        kind = F.LINEAR
        Vs, ks = [8, 16, 32], [8, 16, 32, 64, 96, 128]
    if os.environ.get("TUNE_V"):
        Vs = [int(x) for x in os.environ["TUNE_V"].split(",")]
    if os.environ.get("TUNE_K"):
        ks = [int(x) for x in os.environ["TUNE_K"].split(",")]
    fams = [int(x) for x in os.environ.get("TUNE_FAM", "2").split(",")]
    for fam in fams:
      for V in Vs:
        for k in ks:
            plan = F.fqnm_plan_ex(n, 1e-6, dt_dx, kind)
            try:
                F.fqnm_debug_override(plan, fam, 0, V)
                F.fqnm_debug_override(plan, 0, k, 0)
            except F.FqnmError as e:
                continue
            q = q0.clone()
            ms = run(plan, q, steps)
            digest = hashlib.sha256(q.cpu().numpy().tobytes()).hexdigest()[:16]
            print(json.dumps({"which": which, "lib": os.environ.get("FQNM_LIBPATH", "default"),
                              "fam": fam, "n": n, "steps": steps, "V": V, "k": k, "ms": ms,
                              "GCUPS": n * steps / ms / 1e6, "sha": digest}), flush=True)
            del q, plan
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
