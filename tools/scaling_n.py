"""SURVEY §8(d)-D6 / PAPER P:467-471 ("runtime per step is O(n)"): time the stepper
at fixed k for N = 2^20 .. 2^28 (cfg4 data slices, EO; cfg3-style data, linear) and
fit t = a + b N; prints one JSON line per point and one with the fit (R^2).
CUDA events, best of 3, after a warm-up."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch
import paper_2604_06947_b200 as F
import workloads as W


def timed(plan, q, steps, reps=3):
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
    for which in ("eo", "linear"):
        Ns, ts = [], []
        for e in range(20, 29, 2):
            n = 1 << e
            if which == "eo":
                q = W.q0_cfg4(n=1 << 31, count=n, device="cuda")
                qmax = int(q.abs().max())
                plan = F.fqnm_plan(n, 1e-6, W.dt_dx_double(W.cfg("cfg4"), qmax), F.BURGERS_EO,
                                   F.PERIODIC)
                steps = 96
            else:
                q = torch.tensor(W.q0_cfg3(n), dtype=torch.int32, device="cuda")
                plan = F.fqnm_plan(n, 1e-6, 0.5, F.LINEAR, F.PERIODIC)
                steps = 256
            if plan.info()["kernel"] != 2:
                F.fqnm_debug_override(plan, 2)
            ms = timed(plan, q, steps)
            Ns.append(n)
            ts.append(ms)
            print(json.dumps({"rule": which, "n": n, "steps": steps, "ms": ms,
                              "GCUPS": n * steps / ms / 1e6, "kernel": plan.info()["kernel"],
                              "k": plan.info()["k"], "V": plan.info()["cells_per_thread"]}), flush=True)
            del q, plan
            torch.cuda.empty_cache()
        N, t = np.array(Ns, float), np.array(ts, float)
        b, a = np.polyfit(N, t, 1)
        pred = a + b * N
        r2 = 1.0 - ((t - pred) ** 2).sum() / ((t - t.mean()) ** 2).sum()
        print(json.dumps({"rule": which, "fit": "t_ms = a + b N", "a_ms": a, "b_ms_per_cell": b,
                          "R2": r2, "asymptotic_GCUPS": steps / b / 1e6}), flush=True)


if __name__ == "__main__":
    main()
