"""Throughput of K8 (3D directional composition, one step per launch) on cubes:
GCUPS and achieved HBM GB/s (8 B algorithmic per cell-update). CUDA events."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch
import paper_2604_06947_b200 as F

for kind, lam, delta, amp, name in ((F.LINEAR, 0.25, 1e-3, 3000, "linear"),
                                    (F.BURGERS_EO, 1 / 15, 1e-5, 100000, "eo")):
    for n, kern in ((256, 8), (256, 10), (512, 8), (512, 10)):
        plan = F.fqnm_plan_3d(n, n, n, delta, lam, lam, lam, kind, F.PERIODIC)
        F.fqnm_debug_override(plan, kern)
        g = torch.Generator(device="cuda").manual_seed(0)
        q = torch.randint(-amp, amp, (n, n, n), dtype=torch.int32, device="cuda", generator=g)
        steps = 20
        F.fqnm_step(plan, q, 2)
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            F.fqnm_step(plan, q, steps)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        cu = n ** 3 * steps
        print(json.dumps({"kernel": "K8 k_step3d" if kern == 8 else "K10 k_step3d_s", "rule": name, "shape": [n, n, n], "steps": steps,
                          "ms": best, "GCUPS": cu / best / 1e6,
                          "hbm_GBs_alg": 8.0 * cu / best / 1e6, "info": plan.info()}), flush=True)
        del plan, q
        torch.cuda.empty_cache()
