"""Time every BASELINE.json configuration through the C ABI on one GPU (CUDA
events, after a warm-up run) and report GCUPS; bench.py's headline is cfg4.
usage: python tools/bench_configs.py [cfg ...]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch
import paper_2604_06947_b200 as F
import workloads as W


def timed(plan, q0, steps, reps=3):
    q = q0.clone()
    F.fqnm_step(plan, q, steps)                      # warm-up
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        q.copy_(q0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        F.fqnm_step(plan, q, steps)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best, q


def main():
    names = sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "ens1", "cfg5"]
    for name in names:
        w = W.cfg(name) if name in W.CONFIG_NAMES else None
        if name == "cfg1":
            q0 = torch.tensor(W.q0_cfg1(), dtype=torch.int32, device="cuda")
            plan = F.fqnm_plan(w.n, 1e-4, W.dt_dx_double(w), F.LINEAR, F.PERIODIC)
            steps, cells = w.steps, w.n
        elif name == "cfg2":
            q0 = torch.tensor(W.q0_cfg2(), dtype=torch.int32, device="cuda")
            plan = F.fqnm_plan(w.n, 1e-5, W.dt_dx_double(w, 150000), F.BURGERS_EO, F.PERIODIC)
            if os.environ.get("CFG2_K") or os.environ.get("CFG2_V"):
                F.fqnm_debug_override(plan, 6, int(os.environ.get("CFG2_K", 16)),
                                      int(os.environ.get("CFG2_V", 8)))
            steps, cells = w.steps, w.n
        elif name == "cfg3":
            q0 = torch.tensor(W.q0_cfg3(), dtype=torch.int32, device="cuda")
            plan = F.fqnm_plan(w.n, 1e-6, W.dt_dx_double(w), F.LINEAR, F.PERIODIC)
            steps, cells = w.steps, w.n
        elif name == "ens1":
            q0 = torch.tensor(W.q0_ensemble(w.batch), dtype=torch.int32, device="cuda")
            plan = F.fqnm_plan_ex(w.n, 1e-4, W.dt_dx_double(w), F.LINEAR, batch=w.batch)
            steps, cells = w.steps, w.n * w.batch
        elif name == "cfg5":
            _, lam = W.sod_steps_and_dt_dx(w.n)
            q0 = torch.tensor(W.sod_q0(w.n), dtype=torch.int64, device="cuda")
            plan = F.fqnm_plan(w.n, 1e-7, lam, F.EULER_ROE, F.TRANSMISSIVE)
            if os.environ.get("EULER_V"):
                F.fqnm_debug_override(plan, 0, 0, int(os.environ["EULER_V"]))
            steps, cells = int(os.environ.get("CFG5_STEPS", 2000)), w.n
        elif name in ("eo2d", "lin2d"):
            # 2D directional composition (NEXT-f3): 8192 x 8192 cells, 200 steps
            nx = ny = int(os.environ.get("N2D", 8192))
            rng = np.random.default_rng(5)
            x = W.cell_centres(nx)[None, :]
            y = W.cell_centres(ny)[:, None]
            if name == "eo2d":
                u = 0.2 + 0.5 * np.sin(2 * np.pi * x) * np.cos(2 * np.pi * y)
                q0 = torch.tensor(W.quantise(u, 1e-6), dtype=torch.int32, device="cuda")
                qmax = int(q0.abs().max())
                lam = 0.4 / (1e-6 * qmax) / 2          # nu = 0.4 per direction, split over 2 dims
                plan = F.fqnm_plan_2d(nx, ny, 1e-6, lam, lam, F.BURGERS_EO, F.PERIODIC)
            else:
                u = np.exp(-((x - 0.5) ** 2 + (y - 0.5) ** 2) / 0.01)
                q0 = torch.tensor(W.quantise(u, 1e-6), dtype=torch.int32, device="cuda")
                plan = F.fqnm_plan_2d(nx, ny, 1e-6, 0.25, 0.25, F.LINEAR, F.PERIODIC)
            if os.environ.get("K2D"):
                F.fqnm_debug_override(plan, int(os.environ.get("KERN2D", 0)), int(os.environ["K2D"]), 0)
            steps, cells = 200, nx * ny
        elif name in ("godunov2", "godunov26"):
            # quantised two-point Godunov rule (Thm P:262-280) on cfg2 data (K6) and on
            # a 2^26-cell slice of cfg4 data (K2, int64 exact evaluation)
            if name == "godunov2":
                w = W.cfg("cfg2")
                q0 = torch.tensor(W.q0_cfg2(), dtype=torch.int32, device="cuda")
                plan = F.fqnm_plan(w.n, 1e-5, W.dt_dx_double(w, 150000), F.BURGERS_GODUNOV,
                                   F.PERIODIC)
                steps, cells = w.steps, w.n
            else:
                n = 1 << 26
                q0 = W.q0_cfg4(n=1 << 31, count=n, device="cuda")
                qmax = int(q0.abs().max())
                plan = F.fqnm_plan(n, 1e-6, W.dt_dx_double(W.cfg("cfg4"), qmax),
                                   F.BURGERS_GODUNOV, F.PERIODIC)
                steps, cells = 96, n
        elif name in ("eo3d", "lin3d"):
            # 3D directional composition (NEXT-f3, d = 3), 512^3 cells, 20 steps
            n3 = int(os.environ.get("N3D", 512))
            g = torch.Generator(device="cuda").manual_seed(0)
            amp = 100000 if name == "eo3d" else 3000
            q0 = torch.randint(-amp, amp, (n3, n3, n3), dtype=torch.int32, device="cuda", generator=g)
            if name == "eo3d":
                plan = F.fqnm_plan_3d(n3, n3, n3, 1e-5, 1 / 15, 1 / 15, 1 / 15, F.BURGERS_EO)
            else:
                plan = F.fqnm_plan_3d(n3, n3, n3, 1e-3, 0.25, 0.25, 0.25, F.LINEAR)
            steps, cells = 20, n3 ** 3
        else:
            raise SystemExit(f"unknown config {name}")
        ms, q = timed(plan, q0, steps, reps=1 if name == "cfg5" else 3)
        info = plan.info()
        print(json.dumps({"config": name, "cells": cells, "steps": steps, "ms": ms,
                          "GCUPS": cells * steps / ms / 1e6, "kernel": info["kernel"],
                          "V": info["cells_per_thread"], "k": info["k"]}), flush=True)
        del q, q0, plan
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
