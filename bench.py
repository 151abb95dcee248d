#!/usr/bin/env python
"""FQNM bench: integer cell-updates/s of the B200 stepper.

Workloads (`--workload`):
  cfg4 (default, the headline)  BASELINE.json's single-domain Burgers configuration
        (BJ.cfg4: N = 2^31 cells, int32, EO split, delta = 1e-6, Courant 0.4, 1000 time
        steps per bench step), split contiguously across the ranks for N > 1 GPUs
        (strong scaling: total work fixed; one k-deep halo exchange per temporal block).
  ens1  SURVEY §8(d)-D2 ENS-1, the north star's batched-ensemble mode: 2^16 independent
        cfg1-like problems (1024 cells, linear kappa = 1/2, 2000 time steps) PER GPU;
        rank r owns problems [r B, (r+1) B) of a P B-problem ensemble, no data-path
        collective (weak scaling, SURVEY §8(e) "Ensembles").

One bench "step" = one pass of the whole hot path over the workload (every row of
SURVEY §8(a): plan constants, staging, map evaluation, interface transfer, update,
temporal blocks, write back, halo exchange for N > 1), continuing from the previous
state.

Contract (see task): W >= 3 warm-up steps, K timed steps bracketed by a barrier +
synchronize on both sides, CUDA-event time on the launching stream, max over ranks, one
JSON line from rank 0.  Every run is then verified against the CPU oracle (parity
windows / sampled problems, bit-exact) and by whole-state invariants, at any N.
`--impl reference` times the CPU oracle (the paper has no reference implementation) on
a bounded sample.
"""
from __future__ import annotations

import argparse
import json
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
# EO with P = 1 (every BJ Burgers config), mixed-sign data: int->float, q^2 (FMUL), estimate
# (FFMA), remainder (2 IMAD), correction (LEA), sign mask (SHF), phi- (LOP3), interface
# transfer + update (2 IADD3) = 10.  Sign-uniform data (every cell >= 0, as BJ.cfg4's
# u0 = 0.2 + ... > 0; DESIGN §K2 "sign-uniform windows"): phi- = 0, the transfer is g alone:
# int->float, FMUL, FFMA, 2 IMAD, LEA, one IADD3 = 7.  General P adds one IMAD.
# Linear kappa = 1/2: 4.  SURVEY §8(d)-D3's a-priori 16 over-counts these closed forms.
OPS_ALG = {"burgers_eo": 10, "burgers_eo_general_p": 11, "burgers_eo_sign_uniform": 7,
           "burgers_eo_sign_uniform_general_p": 8, "linear": 4}
# The sign-uniform P = 1 step in float64 (maps.cuh eo_g_dp; K2S / K2PS and the sign-uniform
# windows of K2 / K2P): IMAD.WIDE, DFMA, DADD + the IADD3 update = 4 instructions per
# cell-update.  Two bounds coincide: instruction issue (128 lanes / 4) and the FP64 pipe
# (64 lanes / 2 for DFMA + DADD) both allow 32 cell-updates/clk/SM = 9.3 TCUPS at 1.965 GHz.
# The microbenchmarks (profiles/r02_micro.json) show the four instruction classes as
# independent streams reach 0.94 of issue (grp_dfma_dadd_imadwide_iadd), but the step's own
# dataflow (IMAD.WIDE -> DFMA -> DADD -> IADD3) tops out at 19.0 cell-updates/clk/SM
# (eo_dp_step: 0.59 of issue; ncu: dispatch stalls on the FP64 instructions), which is what
# `mix_ceiling` reports.
EO_DP_INSTR = 4
RULE_NAMES = {1: "LIN_HALF", 2: "EO_FAST", 3: "GENERIC", 4: "LIN_FAST", 5: "EO_P1"}
SM_COUNT = 148
LANES_PER_SM_CLK = 128                          # 4 SMSPs x 32 lanes, 1 warp-instr/clk each
WINDOW = 2048                                   # cells per parity window
# float64-pipe instructions (DMUL + DADD + DFMA + DSETP) the Euler kernel executes per
# cell-update, counted by ncu on the V = 2 branch-free path (profiles/r02_summary.md;
# 305 thread instructions in all): the basis of cfg5's FP64-issue roofline
FP64_PER_CELL_EULER = 122


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return mp, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def _micro_peaks():
    """Per-pipe issue rates measured on a B200 by tools/micro.py (committed under
    profiles/*_micro.json): lane-operations per second at the clock they ran at."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_micro.json")))
    if not files:
        return None, None
    with open(files[-1]) as f:
        return json.load(f), os.path.relpath(files[-1], ROOT)


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
    scale = n_local / float(cap.get("n_cells", 1 << 31))
    return cap["dram_bytes_per_launch"] * scale, os.path.relpath(files[-1], ROOT)


def init_dist():
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def host_cpu():
    """Host CPU model and sockets (lscpu), for the oracle timing context."""
    info = {"model": None, "sockets": None, "affinity_cores": len(os.sched_getaffinity(0))}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() == "Model name":
                info["model"] = v.strip()
            elif k.strip() == "Socket(s)":
                info["sockets"] = int(v.strip()) if v.strip().isdigit() else v.strip()
    except Exception:
        pass
    return info


def time_oracle(run, cells: int, target_s: float):
    """Cell-updates/s of run(steps) on `cells` cells, sized to about target_s seconds."""
    t = time.perf_counter()
    run(2)
    dt = max(time.perf_counter() - t, 1e-6)
    steps = max(2, int(target_s / (dt / 2)))
    t = time.perf_counter()
    run(steps)
    dt = time.perf_counter() - t
    return cells * steps / dt / 1e9, steps, dt


def cpu_baseline_cfg4(qmax: int):
    """The oracle as it stands on the host: all cores (OpenMP) on a periodic 2^20-cell slice
    of cfg4 and one thread on a 2^17-cell slice."""
    import oracle
    import workloads as W
    w = W.cfg("cfg4")
    rule = oracle.Rule(oracle.BURGERS_EO, w.delta, W.dt_dx(w, qmax))
    qa = W.q0_cfg4(n=w.n, count=1 << 20).numpy().astype(np.int64)
    q1 = qa[:1 << 17].copy()
    cores = oracle.max_threads()              # the OpenMP default the all-core run uses
    rate, steps, secs = time_oracle(lambda s: rule.run(qa, s, nthreads=cores), qa.size, 12.0)
    rate1, steps1, secs1 = time_oracle(lambda s: rule.run(q1, s, nthreads=1), q1.size, 5.0)
    return {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"periodic cfg4 slice of 2^20 cells x {steps} time steps ({secs:.1f} s)",
            "one_thread": {"value": rate1, "unit": UNIT,
                           "sample": f"2^17 cells x {steps1} time steps ({secs1:.1f} s)"},
            "host": host_cpu()}


# ---------------------------------------------------------------------------
# --impl reference: the CPU oracle (rank 0 only)
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import oracle
    import workloads as W
    cores = oracle.max_threads()
    if args.workload == "ens1":
        w = W.cfg("ens1")
        B = 64                               # problems per sample (the GPU arm: 2^16 per GPU)
        q = W.q0_ensemble(1 << 16, n=w.n, count=B).astype(np.int64)
        rule = oracle.Rule(oracle.LINEAR, w.delta, W.dt_dx(w))
        steps_per = w.steps
        cells = B * w.n
        sample = f"ens1: {B} of the 2^16 problems x {w.n} cells x {steps_per} time steps per bench step"
        config = {"workload": "ens1", "sample_problems": B, "n_cells": w.n,
                  "time_steps_per_step": steps_per}
    else:
        w = W.cfg("cfg4")
        cells = 1 << 20
        q = W.q0_cfg4(n=w.n, count=cells).numpy().astype(np.int64)
        qmax = 344848                  # max |q0| of cfg4 (the GPU arm's kappa = 1/(5 Q_max) = 1/1724240)
        rule = oracle.Rule(oracle.BURGERS_EO, w.delta, W.dt_dx(w, qmax))
        steps_per = 1000                   # the time steps of one cfg4 bench step
        sample = f"cfg4 slice of {cells} cells x {steps_per} time steps per bench step (periodic)"
        config = {"workload": "cfg4", "sample_cells": cells, "time_steps_per_step": steps_per}
    for _ in range(args.warmup):
        q = rule.run(q, 1)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        q = rule.run(q, steps_per)
        times.append(time.perf_counter() - t)
    tot = sum(times)
    val = cells * steps_per * args.steps / tot / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak" if args.workload == "ens1" else "strong",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic", "config": config,
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": sample, "host": host_cpu()},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def timed(do_step, args, world, local, plan, stepper_plans):
    """W untimed warm-up steps, then exactly K steps between barrier + sync, CUDA events
    on the launching stream; device time max over ranks."""
    import torch
    import torch.distributed as dist
    import paper_2604_06947_b200 as F
    for _ in range(max(args.warmup, 0)):
        do_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
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
    dev = torch.device("cuda", local)
    t = torch.tensor([ms, kern_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0]), float(t[1]), kern_ms, kern_launches, launches, clk, ms


def alu_roofline(kernel: str, ops_alg: int, updates_per_launch: float, per_launch_ms: float,
                 hbm_bytes_per_launch: float, extra: dict, mix_ceiling_key: str = "",
                 pipe_lanes: int = 0, pipe_name: str = ""):
    """ops_alg operations per cell-update against 148 SMs x lanes/clk x f: the whole SM's
    instruction issue (128 lanes) by default, or the one pipe that binds (pipe_lanes)."""
    peaks, peak_src = _peaks()
    f_max = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    lanes = pipe_lanes if pipe_lanes else LANES_PER_SM_CLK
    peak_ops = SM_COUNT * lanes * f_max                               # lane-ops/s at max clock
    achieved_ops = ops_alg * updates_per_launch / (per_launch_ms / 1e3)
    roof = {
        "bound": "alu", "kernel": kernel,
        "achieved": achieved_ops / 1e12, "peak": peak_ops / 1e12, "unit": "Tops/s",
        "frac": achieved_ops / peak_ops,
        "ops_alg_per_cell_update": ops_alg,
        "peak_basis": ("148 SMs x %d lanes/clk (%s) x sm_max_mhz (%s)" % (
            lanes, pipe_name if pipe_lanes else "instruction issue: 4 schedulers x 32", peak_src)),
        "traffic": None, "traffic_source": None,
        "algorithmic_bytes_per_launch": hbm_bytes_per_launch,
        "kernel_ms_per_launch": per_launch_ms,
        "hbm_achieved_gbs": hbm_bytes_per_launch / (per_launch_ms / 1e3) / 1e9,
        "hbm_peak_gbs": float(peaks.get("hbm_gbs", 6650.0)),
    }
    roof.update(extra)
    micro, src = _micro_peaks()
    if micro:
        # the same achieved rate against the issue rate measured on a B200 by
        # microbenchmarks (the mixed ALU + FMA integer stream, scaled to sm_max_mhz)
        m = micro.get("dfma_dadd" if pipe_lanes else "mixed_alu_fma_int", {})
        if m.get("lane_ops_per_clk_per_sm"):
            mp = m["lane_ops_per_clk_per_sm"] * SM_COUNT * f_max
            roof["measured_issue_peak"] = mp / 1e12
            roof["frac_vs_measured_issue_peak"] = achieved_ops / mp
            roof["measured_peak_source"] = src
        # and against the compute-only ceiling of the kernel's own instruction mix: the
        # sign-uniform EO step on register data (no loads/stores), same occupancy
        e = micro.get(mix_ceiling_key, {}) if mix_ceiling_key else {}
        if e.get("lane_ops_per_clk_per_sm"):
            # micro reports instructions; convert to cell-updates with its instructions per cell
            per_cell = {"eo_sign_step": 7.0, "eo_dp_step": 4.0}[mix_ceiling_key]
            ceil_cups = e["lane_ops_per_clk_per_sm"] / per_cell * SM_COUNT * f_max
            cups = updates_per_launch / (per_launch_ms / 1e3)
            roof["mix_ceiling"] = {"what": "the kernel's own step on register data, no loads/stores "
                                           "(tools/micro.cu k_%s, %g instr/cell)" % (mix_ceiling_key, per_cell),
                                   "achieved_frac": cups / ceil_cups,
                                   "ceiling_tcups": ceil_cups / 1e12}
    return roof


# ---------------------------------------------------------------------------
def run_cfg4(args):
    import torch
    import torch.distributed as dist
    import paper_2604_06947_b200 as F
    from paper_2604_06947_b200 import checks, halo
    import workloads as W

    rank, world, local = init_dist()
    halo_mode = "none"
    dev = torch.device("cuda", local)
    w = W.cfg("cfg4")
    N = args.n
    T = args.time_steps
    off, n_local = halo.partition(N, world, rank)
    offsets = [halo.partition(N, world, r)[0] for r in range(world)]

    # ---- inputs (seeded, synthetic, generated on the device; D5) ----
    q = W.q0_cfg4(n=N, offset=off, count=n_local, device=dev)
    qmax_t = q.abs().max().to(torch.int64)
    if world > 1:
        dist.all_reduce(qmax_t, op=dist.ReduceOp.MAX)
    qmax = int(qmax_t)
    dt_dx = W.dt_dx_double(w, qmax)           # Courant 0.4 with alpha = delta max|q0| (A3)
    # invariants of the initial state (independent torch reductions, all ranks)
    inv0 = checks.invariants(q)

    # ---- plan (the public C-ABI entry points) ----
    ring = sd = None
    if world == 1:
        plan = F.fqnm_plan(N, 1e-6, dt_dx, F.BURGERS_EO, F.PERIODIC)     # north-star signature
        info = plan.info()

        def do_step():
            F.fqnm_step(plan, q, T)

        def owned():
            return q
    else:
        probe = F.fqnm_plan_validate(N, 1e-6, dt_dx, F.BURGERS_EO)
        k = probe["k"]
        halo_mode = args.halo
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

    ms_max, kern_ms_max, kern_ms, kern_launches, launches, clk, ms = timed(
        do_step, args, world, local, plan, [plan])
    cell_updates = N * T * args.steps
    value = cell_updates / (ms_max / 1e3) / 1e9

    # ---- roofline of the dominant kernel (k_blocked, EO fast path) ----
    per_launch_ms = kern_ms / max(kern_launches, 1)
    updates_per_launch = n_local * T * args.steps / max(kern_launches, 1)
    # the K2 path every window takes: sign-uniform when the whole state is >= 0 (or <= 0),
    # which the maximum principle keeps for the whole run (Lemma CFL)
    uniform = inv0["min"] >= 0 or inv0["max"] <= 0
    ops_key = ("burgers_eo_sign_uniform" if uniform else "burgers_eo") + (
        "" if info["rule"] == 5 else "_general_p")
    ops_alg = OPS_ALG[ops_key]
    hbm_bytes_per_launch = 8.0 * n_local                               # read + write int32 once per block
    # which K2 ran: the sign-specialised K2S (V = 48) when the range check proved the sign
    k2s = plan.info()["k2s_launches"] > 0
    Vk = 48 if k2s else info["cells_per_thread"]
    kname = "k_blocked<%s,V=%d%s>" % (RULE_NAMES.get(info["rule"], "?"), Vk, ",sign" if k2s else "")
    # P = 1 sign-uniform state: the float64 step, bound by the FP64 pipe
    dp = uniform and info["rule"] == 5
    if dp:
        ops_key = "burgers_eo_sign_uniform_f64"
    roofline = alu_roofline(
        kname, EO_DP_INSTR if dp else ops_alg, updates_per_launch, per_launch_ms, hbm_bytes_per_launch,
        {"kernel_launches": kern_launches, "kernel_share_of_step": kern_ms / ms if ms > 0 else None,
         "k": info["k"], "V": Vk, "ops_basis": ops_key,
         "instructions_per_cell_update": EO_DP_INSTR if dp else ops_alg,
         # K2S windows carry a halo on one side only (a one-signed state moves one way)
         "windows_redundancy": 32.0 * Vk / (32.0 * Vk - (1 if k2s else 2) * ((info["k"] + 3) // 4 * 4))},
        mix_ceiling_key="eo_dp_step" if dp else ("eo_sign_step" if ops_key == "burgers_eo_sign_uniform" else ""))
    # the same rate on the bases used before: the float32 form's 7 operations (the kernel of
    # the earlier bench lines) and SURVEY 8(d)-D3's a-priori 16 operations per EO cell-update
    cups = updates_per_launch / (per_launch_ms / 1e3)
    issue = SM_COUNT * LANES_PER_SM_CLK * float(_peaks()[0].get("sm_max_mhz", 1965.0)) * 1e6
    roofline["frac_on_7op_float32_form_basis"] = cups * 7 / issue
    roofline["frac_on_survey_16op_basis"] = cups * 16 / issue
    tr, tr_src = ncu_traffic(n_local)
    if tr is not None:
        roofline["traffic"] = tr
        roofline["traffic_source"] = tr_src
        roofline["traffic_over_algorithmic"] = tr / hbm_bytes_per_launch

    # ---- verification of the benchmarked state (every run, any N) ----
    total = T * (args.warmup + args.steps)
    parity = None
    if not args.no_parity:
        parity = verify_cfg4(args, owned(), off, n_local, N, offsets, total, qmax, inv0, dev, world,
                             rank)

    # ---- end-to-end through the public API with host buffers (H2D + steps + D2H) ----
    e2e = None
    if not args.no_e2e:
        if world == 1:
            qh = torch.empty(N, dtype=torch.int32, pin_memory=True)
            qh.copy_(q.cpu())
            F.fqnm_step_host(plan, qh, T)              # warm (allocates the e2e pipeline)
            torch.cuda.synchronize()
            eclk = Clocks(local)
            eclk.start()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                F.fqnm_step_host(plan, qh, T)          # synchronous: H2D, T steps, D2H
            e2e_s = time.perf_counter() - t0
            ec = eclk.stop()
            del qh
            e2e = {"value": N * T * args.steps / e2e_s / 1e9, "unit": UNIT,
                   "h2d_bytes_per_step": 4 * N, "d2h_bytes_per_step": 4 * N,
                   "clocks": ec}
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

    # ---- CPU baseline (oracle on host cores; rank 0, N = 1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_cfg4(qmax)

    # ---- the other BASELINE configurations, timed + parity-checked (rank 0, N = 1 only) ----
    others = None
    if rank == 0 and world == 1 and not args.no_configs:
        del q, plan
        torch.cuda.empty_cache()
        others = run_other_configs(dev, args.seed)

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
            "gpu_launches": launches, "parity": parity, "other_configs": others,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def verify_cfg4(args, q, off, n_local, N, offsets, total, qmax, inv0, dev, world, rank):
    """Bit-exact light-cone windows vs the oracle (wrap, every split point, middle, random;
    SURVEY §8(c)-C6, §8(e)), whole-domain invariants before/after (with the cross-rank
    edge pairs), and the number of cells the run changed.  Collective over the ranks;
    the oracle runs on rank 0."""
    import torch
    import torch.distributed as dist
    from paper_2604_06947_b200 import checks
    import workloads as W
    out = {"time_steps": total, "checked_windows": 0, "ok": True}
    try:
        inv1 = checks.invariants(q)
        changed = checks.changed_cells(
            q, lambda i, m: W.q0_cfg4(n=N, offset=off + i, count=m, device=dev))
        starts = checks.window_starts(N, offsets, WINDOW, n_random=1, seed=args.seed)
        got = checks.gather_windows(q, off, N, starts, WINDOW).cpu().numpy()
        if rank == 0:
            import oracle
            w = W.cfg("cfg4")
            rule = oracle.Rule(oracle.BURGERS_EO, w.delta, W.dt_dx(w, qmax))
            mism = []
            t0 = time.perf_counter()
            for i, a in enumerate(starts):
                # dependence cone: `total` cells on each side; the oracle's periodic wrap
                # inside the window buffer only corrupts cells outside [total, total + W)
                idx = np.arange(a - total, a + WINDOW + total)
                qin = W.q0_cfg4_at(idx % N, n=N, device=dev)
                ref = rule.run(qin, total)[total:total + WINDOW]
                out["checked_windows"] += 1
                if not np.array_equal(ref, got[i]):
                    mism.append({"start": int(a), "cells": int((ref != got[i]).sum())})
            out["oracle_s"] = time.perf_counter() - t0
            out["window_starts"] = [int(s) for s in starts]
            out["window_cells"] = WINDOW
            out["mismatches"] = mism
            out["ok"] = not mism
            out["cells_changed"] = changed
            out["invariants"] = {
                "sum_conserved": inv1["sum"] == inv0["sum"],
                "max_principle": inv1["min"] >= inv0["min"] and inv1["max"] <= inv0["max"],
                "tv_nonincreasing": inv1["tv"] <= inv0["tv"],
                "initial": inv0, "final": inv1,
                "tv_includes": "all adjacent pairs incl. %d cross-rank edges and the periodic wrap"
                               % max(world - 1, 0)}
            out["ok"] = bool(out["ok"]) and changed > 0 and all(
                out["invariants"][k] for k in ("sum_conserved", "max_principle", "tv_nonincreasing"))
    except Exception as ex:       # never let the check kill the bench line
        out = {"ok": None, "error": repr(ex)[:300]}
    if world > 1:
        dist.barrier()
    return out


# ---------------------------------------------------------------------------
def run_other_configs(dev, seed: int):
    """The other BASELINE.json configurations, timed and parity-checked beside the headline
    (N = 1 only; outside the timed region of the bench line): cfg1, cfg2 (full runs vs the
    oracle), cfg3 and a cfg5 window (light-cone windows vs the oracle), ENS-1 (sampled
    problems).  Each entry: best of 3 repetitions by CUDA events on the launching stream,
    after one warm-up run; roofline fraction on SURVEY 8(d)-D3's basis where one applies."""
    import torch
    import oracle
    import paper_2604_06947_b200 as F
    import workloads as W
    out = []
    rng = np.random.default_rng(seed)

    def best_ms(plan, q0, steps, reps=3):
        q = q0.clone()
        F.fqnm_step(plan, q, steps)
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

    def entry(name, plan, cells, steps, ms, ok, what, bound=None):
        info = plan.info()
        e = {"config": name, "cells": cells, "time_steps": steps, "ms": ms,
             "GCUPS": cells * steps / ms / 1e6, "kernel": info["kernel"], "V": info["cells_per_thread"],
             "k": info["k"], "parity": {"ok": bool(ok), "what": what}}
        if bound:
            e["roofline"] = dict(bound, frac=e["GCUPS"] / bound["peak_gcups"])
        out.append(e)

    def windows_ok(run, q0h, qh, n, steps, periodic, width=1024, count=2, axis=-1):
        ok = True
        for a in [0] + [int(x) for x in rng.integers(0, n - width, count)]:
            if periodic:
                idx = np.arange(a - steps, a + width + steps) % n
                ref = run(np.ascontiguousarray(np.take(q0h, idx, axis=axis)))
                ref = np.take(ref, np.arange(steps, steps + width), axis=axis)
            else:
                lo, hi = max(0, a - steps), min(n, a + width + steps)
                ref = run(np.ascontiguousarray(np.take(q0h, np.arange(lo, hi), axis=axis)))
                ref = np.take(ref, np.arange(a - lo, a - lo + width), axis=axis)
            ok = ok and np.array_equal(ref, np.take(qh, np.arange(a, a + width), axis=axis))
        return ok

    sm_ghz = _peaks()[0].get("sm_max_mhz", 1965.0) / 1e3
    issue4 = {"bound": "alu", "ops_alg_per_cell_update": 4, "peak_gcups": 148 * 128 * sm_ghz / 4}
    try:
        # cfg1: linear advection, N = 1024, 2000 steps (one warp, K3)
        w = W.cfg("cfg1")
        q0h = W.q0_cfg1()
        plan = F.fqnm_plan(w.n, float(w.delta), W.dt_dx_double(w), F.LINEAR, F.PERIODIC)
        ms, q = best_ms(plan, torch.tensor(q0h, dtype=torch.int32, device=dev), w.steps)
        ref = oracle.Rule(oracle.LINEAR, w.delta, W.dt_dx(w)).run(q0h, w.steps)
        entry("cfg1", plan, w.n, w.steps, ms, np.array_equal(q.cpu().numpy(), ref), "full state vs oracle")
        # cfg2: Burgers EO, N = 65536, 20000 steps (resident stepper, K6)
        w = W.cfg("cfg2")
        q0h = W.q0_cfg2()
        qmax = int(np.abs(q0h).max())
        plan = F.fqnm_plan(w.n, float(w.delta), W.dt_dx_double(w, qmax), F.BURGERS_EO, F.PERIODIC)
        ms, q = best_ms(plan, torch.tensor(q0h, dtype=torch.int32, device=dev), w.steps)
        ref = oracle.Rule(oracle.BURGERS_EO, w.delta, W.dt_dx(w, qmax)).run(q0h, w.steps)
        entry("cfg2", plan, w.n, w.steps, ms, np.array_equal(q.cpu().numpy(), ref), "full state vs oracle")
        # cfg3: linear kappa = 1/2, N = 2^24, 10^4 steps (K2P)
        w = W.cfg("cfg3")
        q0h = W.q0_cfg3()
        plan = F.fqnm_plan(w.n, float(w.delta), W.dt_dx_double(w), F.LINEAR, F.PERIODIC)
        ms, q = best_ms(plan, torch.tensor(q0h, dtype=torch.int32, device=dev), w.steps)
        rule = oracle.Rule(oracle.LINEAR, w.delta, W.dt_dx(w))
        qh = q.cpu().numpy()
        ok = windows_ok(lambda x: rule.run(x, w.steps), q0h, qh, w.n, w.steps, True)
        ok = ok and int(qh.astype(np.int64).sum()) == int(q0h.astype(np.int64).sum())
        entry("cfg3", plan, w.n, w.steps, ms, ok, "3 light-cone windows of 1024 cells + exact sum", issue4)
        del q, qh, q0h
        # ENS-1: 2^16 independent cfg1-like problems (K3)
        w = W.cfg("ens1")
        q0h = W.q0_ensemble(w.batch)
        plan = F.fqnm_plan_ex(w.n, float(w.delta), W.dt_dx_double(w), F.LINEAR, batch=w.batch)
        ms, q = best_ms(plan, torch.tensor(q0h, dtype=torch.int32, device=dev), w.steps)
        pick = np.unique(np.concatenate([[0, w.batch - 1], rng.integers(0, w.batch, 14)]))
        ref = oracle.Rule(oracle.LINEAR, w.delta, W.dt_dx(w)).run(q0h[pick], w.steps)
        entry("ens1", plan, w.n * w.batch, w.steps, ms, np.array_equal(q[pick].cpu().numpy(), ref),
              "%d sampled problems vs oracle" % len(pick), issue4)
        del q, q0h
        # cfg5: Sod, 3 x int64, N = 2^26, a 300-step window at the configuration's dt/dx
        w = W.cfg("cfg5")
        S5 = 300
        _, lam = W.sod_steps_and_dt_dx(w.n)
        q0h = W.sod_q0(w.n)
        plan = F.fqnm_plan(w.n, 1e-7, lam, F.EULER_ROE, F.TRANSMISSIVE)
        ms, q = best_ms(plan, torch.tensor(q0h, dtype=torch.int64, device=dev), S5)
        qh = q.cpu().numpy()
        ok = True
        for a in (0, w.n - 1024, w.n // 2 - 512, int(rng.integers(0, w.n - 1024))):
            lo, hi = max(0, a - S5), min(w.n, a + 1024 + S5)
            ref = oracle.euler_run(np.ascontiguousarray(q0h[:, lo:hi]), S5, 1e-7, lam)
            ok = ok and np.array_equal(ref[:, a - lo:a - lo + 1024], qh[:, a:a + 1024])
        micro = _micro_peaks()[0] or {}
        dfma = micro.get("dfma", {}).get("lane_ops_per_clk_per_sm", 64.0)   # measured DFMA rate
        entry("cfg5", plan, w.n, S5, ms, ok, "4 light-cone windows (walls, diaphragm, random)",
              {"bound": "fp64", "fp64_instr_per_cell_update": FP64_PER_CELL_EULER,
               "peak_gcups": 148 * dfma * sm_ghz / FP64_PER_CELL_EULER})
    except Exception as ex:                 # never let the side measurements kill the bench line
        out.append({"error": repr(ex)[:300]})
    return out


# ---------------------------------------------------------------------------
def run_ens1(args):
    """ENS-1: B = 2^16 independent cfg1-like problems per GPU (weak scaling)."""
    import torch
    import torch.distributed as dist
    import paper_2604_06947_b200 as F
    from paper_2604_06947_b200 import shard
    import workloads as W

    rank, world, local = init_dist()
    dev = torch.device("cuda", local)
    w = W.cfg("ens1")
    B = args.batch
    Bt = B * world
    n = w.n
    T = args.time_steps if args.time_steps_set else w.steps
    first, cnt = shard.ensemble_range(Bt, world, rank)   # [r B, (r+1) B): no communication
    assert cnt == B
    q0 = W.q0_ensemble(Bt, n=n, first=first, count=B)
    q = torch.tensor(q0, dtype=torch.int32, device=dev).reshape(-1)
    plan = F.fqnm_plan_ex(n, float(w.delta), W.dt_dx_double(w), F.LINEAR, F.PERIODIC, batch=B)
    info = plan.info()

    def do_step():
        F.fqnm_step(plan, q, T)

    ms_max, _, kern_ms, kern_launches, launches, clk, ms = timed(do_step, args, world, local,
                                                                 plan, [plan])
    value = Bt * n * T * args.steps / (ms_max / 1e3) / 1e9
    per_launch_ms = kern_ms / max(kern_launches, 1)
    updates_per_launch = B * n * T * args.steps / max(kern_launches, 1)
    roofline = alu_roofline("k_warp_ensemble<LIN_HALF,V=%d>" % info["cells_per_thread"],
                            OPS_ALG["linear"], updates_per_launch, per_launch_ms, 8.0 * B * n,
                            {"kernel_launches": kern_launches,
                             "kernel_share_of_step": kern_ms / ms if ms > 0 else None})

    # ---- verification: sampled problems vs the oracle (bit-exact) + per-problem sums ----
    total = T * (args.warmup + args.steps)
    parity = None
    if not args.no_parity:
        parity = {"time_steps": total, "ok": True}
        try:
            import oracle
            qv = q.view(B, n)
            sums_ok = bool(torch.equal(qv.sum(1, dtype=torch.int64),
                                       torch.tensor(q0, device=dev).sum(1)))
            rng = np.random.default_rng(args.seed + rank)
            pick = np.unique(np.concatenate([[0, B - 1], rng.integers(0, B, 30)]))
            ref = oracle.Rule(oracle.LINEAR, w.delta, W.dt_dx(w)).run(q0[pick], total)
            got = qv[torch.as_tensor(pick, device=dev)].cpu().numpy().astype(np.int64)
            ok = bool(np.array_equal(ref, got)) and sums_ok
            flag = torch.tensor([0 if ok else 1, len(pick)], dtype=torch.int64, device=dev)
            if world > 1:
                dist.all_reduce(flag)
            parity.update(ok=int(flag[0]) == 0, checked_problems=int(flag[1]),
                          per_problem_sums_conserved=sums_ok if world == 1 else None)
        except Exception as ex:
            parity = {"ok": None, "error": repr(ex)[:300]}

    e2e = None
    if not args.no_e2e:
        qh = torch.empty(B * n, dtype=torch.int32, pin_memory=True)
        qh.copy_(q.cpu())
        F.fqnm_step_host(plan, qh, T)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            F.fqnm_step_host(plan, qh, T)
        e2e_s = shard.max_over_ranks(time.perf_counter() - t0, dev)
        e2e = {"value": Bt * n * T * args.steps / e2e_s / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 4 * Bt * n, "d2h_bytes_per_step": 4 * Bt * n}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle
        qs = q0[:64].astype(np.int64)
        rule = oracle.Rule(oracle.LINEAR, w.delta, W.dt_dx(w))
        rate, steps_c, secs = time_oracle(lambda s: rule.run(qs, s), qs.size, 10.0)
        cpu = {"value": rate, "unit": UNIT, "cores": oracle.max_threads(), "kind": "oracle",
               "sample": f"64 problems x {n} cells x {steps_c} time steps ({secs:.1f} s)",
               "host": host_cpu()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int32", "data": "synthetic",
            "config": {"workload": "ens1", "problems": Bt, "problems_per_gpu": B, "n_cells": n,
                       "time_steps_per_step": T, "flux": "linear", "kappa": [1, 2],
                       "l2": "state %.0f MiB per GPU, HBM touched once per bench step "
                             "(all time steps in registers)" % (4 * B * n / 2**20),
                       "parallelism": "ensemble shard x%d (no data-path collective)" % world},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "gpu_launches": launches, "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fqnm", choices=["fqnm", "reference"])
    ap.add_argument("--workload", default="cfg4", choices=["cfg4", "ens1"])
    ap.add_argument("--n", type=int, default=1 << 31, help="cfg4 cells (default: BJ.cfg4 2^31)")
    ap.add_argument("--batch", type=int, default=1 << 16, help="ens1 problems per GPU")
    ap.add_argument("--time-steps", type=int, default=None,
                    help="time steps per bench step (cfg4 1000, ens1 2000)")
    ap.add_argument("--seed", type=int, default=0, help="seed of the random parity samples")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the side measurements of cfg1/2/3/5 and ENS-1 (N = 1)")
    ap.add_argument("--halo", default="p2p", choices=["p2p", "nccl"],
                    help="cfg4, N > 1: fused peer-memory halo exchange inside the kernel (p2p) "
                         "or torch.distributed NCCL send/recv between launches")
    args = ap.parse_args()
    args.time_steps_set = args.time_steps is not None
    if args.time_steps is None:
        args.time_steps = 1000
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "ens1":
        return run_ens1(args)
    return run_cfg4(args)


if __name__ == "__main__":
    main()
