#!/usr/bin/env python
"""FQNM bench: integer cell-updates/s of the B200 stepper on BASELINE.json's
single-domain Burgers configuration (BJ.cfg4: N = 2^31 cells, int32, EO split,
delta = 1e-6, Courant 0.4, 1000 time steps), split contiguously across the
ranks for N > 1 GPUs (strong scaling: total work fixed).

One bench "step" = one pass of the whole hot path over the workload: the
1000 explicit time steps of cfg4 (every row of SURVEY §8(a): plan constants,
staging, map evaluation, interface transfer, update, temporal blocks, write
back, halo exchange for N > 1), continuing from the previous state.

Contract (see task): W >= 3 warm-up steps, K timed steps bracketed by a
barrier + synchronize on both sides, CUDA-event time on the launching stream,
max over ranks, one JSON line from rank 0.  `--impl reference` times the CPU
oracle (the paper has no reference implementation) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np

METRIC = "integer cell-updates/sec (GCUPS)"
UNIT = "GCUPS"
# Algorithmic operations per cell-update (DESIGN.md §6 "ops_alg"): the exact closed form's
# own operations, not counting redundant halo work, shuffles, loads/stores or loop control.
# EO with P = 1 (every BJ Burgers config): int->float, q^2 (FMUL), estimate (FFMA), remainder
# (2 IMAD), correction (LEA), sign mask (SHF), phi- (LOP3), interface transfer + update
# (2 IADD3) = 10.  SURVEY §8(d)-D3's a-priori 16 over-counts this closed form (it made the
# fraction exceed 1.0).  General P adds one IMAD (11).  Linear kappa = 1/2: 4.
OPS_ALG = {"burgers_eo": 10, "burgers_eo_general_p": 11, "linear": 4}
RULE_NAMES = {1: "LIN_HALF", 2: "EO_FAST", 3: "GENERIC", 4: "LIN_FAST", 5: "EO_P1"}
SM_COUNT = 148
LANES_PER_SM_CLK = 128                          # 4 SMSPs x 32 lanes, 1 warp-instr/clk each


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return mp, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if self.proc is None:
            return out
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            try:
                pw.append(float(parts[3]))
            except ValueError:
                pass
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        if sm:
            out.update(sm_mhz=statistics.median(sm), sm_max_mhz=max(mx), reasons=sorted(reasons),
                       samples=len(sm))
            if pw:
                out["power_w"] = statistics.median(pw)
        return out


def ncu_traffic(n_local: int):
    """Per-launch DRAM bytes of the dominant kernel from the latest committed
    `ncu --set full` capture (profiles/*_bench_kernel_ncu.json, written by
    tools/ncu_traffic.py), scaled to this run's cells per launch."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_bench_kernel_ncu.json")))
    if not files:
        return None, None
    with open(files[-1]) as f:
        cap = json.load(f)
    scale = n_local / float(1 << 31)           # the capture is of the N = 2^31 bench launch
    return cap["dram_bytes_per_launch"] * scale, os.path.relpath(files[-1], ROOT)


def init_dist():
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    return rank, world, local


def cpu_oracle_rate(q_sample: np.ndarray, qmax: int, target_s: float = 12.0):
    """The oracle as it stands, on host cores, on a bounded periodic slice of cfg4."""
    import oracle
    import workloads as W
    w = W.cfg("cfg4")
    rule = oracle.Rule(oracle.BURGERS_EO, w.delta, W.dt_dx(w, qmax))
    n = len(q_sample)
    t = time.perf_counter()
    rule.run(q_sample, 2)
    dt = max(time.perf_counter() - t, 1e-6)
    steps = max(2, int(target_s / (dt / 2)))
    t = time.perf_counter()
    rule.run(q_sample, steps)
    dt = time.perf_counter() - t
    return n * steps / dt / 1e9, steps, dt, oracle.max_threads()


def state_invariants(q, chunk=1 << 28):
    """Sum (int64), min, max and periodic total variation of a 1-D int32 CUDA state,
    by plain torch reductions in chunks (independent of the FQNM kernels)."""
    import torch
    n = q.numel()
    tot, mn, mx, tv = 0, None, None, 0
    for i in range(0, n, chunk):
        c = q[i:i + chunk]
        tot += int(c.sum(dtype=torch.int64))
        cmin, cmax = int(c.min()), int(c.max())
        mn = cmin if mn is None else min(mn, cmin)
        mx = cmax if mx is None else max(mx, cmax)
        j = min(i + chunk + 1, n)
        seg = q[i:j].to(torch.int64)
        tv += int((seg[1:] - seg[:-1]).abs().sum())
    tv += abs(int(q[0]) - int(q[n - 1]))
    return {"sum": tot, "min": mn, "max": mx, "tv": tv}


def run_reference(args):
    """--impl reference: the CPU oracle timed on host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import oracle
    import workloads as W
    import torch
    w = W.cfg("cfg4")
    n_sample = 1 << 20
    q = W.q0_cfg4(n=w.n, count=n_sample).numpy().astype(np.int64)
    qmax = 344848                      # max |q0| of cfg4 (the GPU arm's kappa = 1/(5 Q_max) = 1/1724240)
    rule = oracle.Rule(oracle.BURGERS_EO, w.delta, W.dt_dx(w, qmax))
    steps_per = 1000                   # the time steps of one cfg4 bench step
    for _ in range(args.warmup):
        q = rule.run(q, 1)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        q = rule.run(q, steps_per)
        times.append(time.perf_counter() - t)
    tot = sum(times)
    val = n_sample * steps_per * args.steps / tot / 1e9
    cores = oracle.max_threads()
    sample = f"cfg4 slice of {n_sample} cells x {steps_per} time steps per bench step (periodic)"
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": {"workload": "cfg4", "sample_cells": n_sample,
                                             "time_steps_per_step": steps_per},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fqnm", choices=["fqnm", "reference"])
    ap.add_argument("--n", type=int, default=1 << 31, help="cells (default: BJ.cfg4 2^31)")
    ap.add_argument("--time-steps", type=int, default=1000, help="time steps per bench step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--halo", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1: fused peer-memory halo exchange inside the kernel (p2p) "
                         "or torch.distributed NCCL send/recv between launches")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_2604_06947_b200 as F
    from paper_2604_06947_b200 import halo
    import workloads as W

    rank, world, local = init_dist()
    halo_mode = "none"
    dev = torch.device("cuda", local)
    w = W.cfg("cfg4")
    N = args.n
    T = args.time_steps
    off, n_local = halo.partition(N, world, rank)

    # ---- inputs (seeded, synthetic, generated on the device; D5) ----
    q = W.q0_cfg4(n=N, offset=off, count=n_local, device=dev)
    qmax_t = q.abs().max().to(torch.int64)
    if world > 1:
        dist.all_reduce(qmax_t, op=dist.ReduceOp.MAX)
    qmax = int(qmax_t)
    dt_dx = W.dt_dx_double(w, qmax)           # Courant 0.4 with alpha = delta max|q0| (A3)

    # ---- plan (the public C-ABI entry points) ----
    if world == 1:
        plan = F.fqnm_plan(N, 1e-6, dt_dx, F.BURGERS_EO, F.PERIODIC)     # north-star signature
        info = plan.info()
        k = info["k"]

        def do_step():
            F.fqnm_step(plan, q, T)
        stepper_plans = [plan]
    else:
        probe = F.fqnm_plan_validate(N, 1e-6, dt_dx, F.BURGERS_EO)
        k = probe["k"]
        halo_mode = args.halo
        ring = None
        if halo_mode == "p2p":
            ring, why = halo.P2PRing.distributed(
                lambda: F.fqnm_plan_ex(n_local, 1e-6, dt_dx, F.BURGERS_EO, F.HALO, halo=k,
                                       n_global=N, offset=off, p2p=True), None, dev)
            if ring is None:                         # no peer access somewhere: NCCL for all
                if rank == 0:
                    print(f"[bench] p2p halo unavailable ({why}); using nccl", file=sys.stderr)
                halo_mode = "nccl"
            else:
                plan = ring.plans[0]
                ring.load([q])
        if halo_mode == "nccl":
            plan = F.fqnm_plan_ex(n_local, 1e-6, dt_dx, F.BURGERS_EO, F.HALO, halo=k,
                                  n_global=N, offset=off)
            sd = halo.SplitDomain([n_local], k, halo.DistTransport(), [plan.step_block],
                                  lambda m: torch.zeros(m, dtype=torch.int32, device=dev))
            sd.load([q])
        info = plan.info()
        del q
        torch.cuda.empty_cache()

        def owned():
            return ring.owned(0) if ring is not None else sd.owned(0)

        def do_step():
            if ring is not None:
                ring.step(T)
            else:
                sd.step(T)
        stepper_plans = [plan]

    # invariants of the initial state (independent torch reductions)
    inv0 = state_invariants(q) if world == 1 else None

    # ---- warm-up ----
    for _ in range(max(args.warmup, 0)):
        do_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # ---- timed region ----
    clocks = Clocks(local)
    launches0 = sum(p.launches() for p in stepper_plans)
    F.fqnm_profile_enable(plan, True)
    F.fqnm_profile_read(plan)                  # reset accumulators
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        do_step()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    kern_ms, kern_launches = F.fqnm_profile_read(plan)
    F.fqnm_profile_enable(plan, False)
    launches = sum(p.launches() for p in stepper_plans) - launches0
    t = torch.tensor([ms, kern_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, kern_ms_max = float(t[0]), float(t[1])

    cell_updates = N * T * args.steps
    value = cell_updates / (ms_max / 1e3) / 1e9

    # ---- roofline of the dominant kernel (k_blocked, EO fast path) ----
    peaks, peak_src = _peaks()
    f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    peak_ops = SM_COUNT * LANES_PER_SM_CLK * f_max                    # int lane-ops/s at max clock
    per_launch_ms = kern_ms / max(kern_launches, 1)
    updates_per_launch = n_local * T * args.steps / max(kern_launches, 1)
    ops_alg = OPS_ALG["burgers_eo"] if info["rule"] == 5 else OPS_ALG["burgers_eo_general_p"]
    achieved_ops = ops_alg * updates_per_launch / (per_launch_ms / 1e3)
    hbm_bytes_per_launch = 8.0 * n_local                               # read + write int32 once per block
    roofline = {
        "bound": "alu", "kernel": "k_blocked<%s,V=%d>" % (RULE_NAMES.get(info["rule"], "?"),
                                                           info["cells_per_thread"]),
        "achieved": achieved_ops / 1e12, "peak": peak_ops / 1e12, "unit": "Tops/s",
        "frac": achieved_ops / peak_ops,
        "ops_alg_per_cell_update": ops_alg,
        "peak_basis": "148 SMs x 128 int lanes/clk x sm_max_mhz (%s)" % peak_src,
        "traffic": None,
        "traffic_source": None,
        "algorithmic_bytes_per_launch": hbm_bytes_per_launch,
        "kernel_ms_per_launch": per_launch_ms, "kernel_launches": kern_launches,
        "kernel_share_of_step": kern_ms / ms if ms > 0 else None,
        "hbm_achieved_gbs": hbm_bytes_per_launch / (per_launch_ms / 1e3) / 1e9,
        "hbm_peak_gbs": float(peaks.get("hbm_gbs", 6650.0)),
        "k": info["k"], "V": info["cells_per_thread"],
    }

    tr, tr_src = ncu_traffic(n_local)
    if tr is not None:
        roofline["traffic"] = tr
        roofline["traffic_source"] = tr_src
        roofline["traffic_over_algorithmic"] = tr / hbm_bytes_per_launch

    inv1 = state_invariants(q) if world == 1 else None

    # ---- end-to-end through the public API with host buffers (H2D + steps + D2H) ----
    e2e = None
    if not args.no_e2e:
        if world == 1:
            qh = torch.empty(N, dtype=torch.int32, pin_memory=True)
            qh.copy_(q.cpu())
            F.fqnm_step_host(plan, qh, T)              # warm (allocates the e2e buffer)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                F.fqnm_step_host(plan, qh, T)          # synchronous: H2D, T steps, D2H
            e2e_s = time.perf_counter() - t0
            del qh
            e2e = {"value": N * T * args.steps / e2e_s / 1e9, "unit": UNIT,
                   "h2d_bytes_per_step": 4 * N, "d2h_bytes_per_step": 4 * N}
        else:
            qh = torch.empty(n_local, dtype=torch.int32, pin_memory=True)
            qh.copy_(owned().cpu())
            dist.barrier()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                owned().copy_(qh, non_blocking=True)
                do_step()
                qh.copy_(owned(), non_blocking=True)
                torch.cuda.synchronize()
            e2e_s = time.perf_counter() - t0
            tt = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e = {"value": N * T * args.steps / float(tt) / 1e9, "unit": UNIT,
                   "h2d_bytes_per_step": 4 * N, "d2h_bytes_per_step": 4 * N}

    # ---- parity spot check (light-cone windows vs the oracle; rank 0) ----
    parity = None
    if rank == 0 and not args.no_parity and world == 1:
        try:
            import oracle
            total = T * (args.warmup + args.steps)
            parity = {"checked_windows": 0, "ok": True, "time_steps": total}
            if total <= 20000:
                rule = oracle.Rule(oracle.BURGERS_EO, w.delta, W.dt_dx(w, qmax))
                for a in (0, N // 3, N - 2048):
                    a = (a // 4) * 4
                    lo, hi = a - total, a + 2048 + total
                    qin = W.q0_cfg4_at(np.arange(lo, hi) % N, n=N, device=dev)
                    ref = rule.run(qin, total)[total:total + 2048]
                    got = q[a:a + 2048].cpu().numpy()
                    parity["checked_windows"] += 1
                    parity["ok"] &= bool(np.array_equal(ref, got))
        except Exception as ex:       # never let the spot check kill the bench line
            parity = {"ok": None, "error": str(ex)[:200]}
        if inv0 is not None and inv1 is not None:
            # exact conservation, maximum principle and TVD of the whole 2^31-cell state
            # after warm-up + timed steps (Lemma P:197-238, Thm conservation)
            parity["invariants"] = {
                "sum_conserved": inv1["sum"] == inv0["sum"],
                "max_principle": inv1["min"] >= inv0["min"] and inv1["max"] <= inv0["max"],
                "tv_nonincreasing": inv1["tv"] <= inv0["tv"],
                "initial": inv0, "final": inv1}
            parity["ok"] = bool(parity["ok"]) and all(
                parity["invariants"][k] for k in ("sum_conserved", "max_principle", "tv_nonincreasing"))

    # ---- CPU baseline (oracle on host cores; rank 0, N = 1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        sample = W.q0_cfg4(n=N, count=1 << 20).numpy().astype(np.int64)
        rate, steps_c, secs, cores = cpu_oracle_rate(sample, qmax)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"periodic cfg4 slice of 2^20 cells x {steps_c} time steps ({secs:.1f} s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int32", "data": "synthetic",
            "config": {"workload": "cfg4", "n_cells": N, "time_steps_per_step": T,
                       "flux": "burgers_eo", "delta": 1e-6, "courant": 0.4, "kappa": [
                           info["kappa_num"], info["kappa_den"]], "k": info["k"],
                       "l2": "inputs larger than L2 (state %.1f GiB > 126 MB)" % (4 * N / 2**30),
                       "parallelism": ("domain split x%d, %s halo" % (world, halo_mode))
                       if world > 1 else "single domain"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "gpu_launches": launches, "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
