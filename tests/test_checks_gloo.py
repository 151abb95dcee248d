"""The N > 1 verification and ensemble-sharding host logic on CPU (gloo, world_size 2
and 3):

* `checks.invariants` of a domain split over the ranks equals the single-domain sum /
  min / max / periodic TV, including the cross-rank edge pairs and the wrap;
* `checks.gather_windows` assembles windows that straddle split points and the wrap;
* `checks.changed_cells` counts over all ranks;
* `shard.ensemble_range` partitions B problems contiguously (no gaps, no overlap), and a
  sharded ensemble run (oracle as the per-rank stepper: CPU tests launch no kernels)
  equals the unsharded run with no data-path collective, only the timing max.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from fractions import Fraction

import oracle
import workloads as W
from paper_2604_06947_b200 import checks, halo, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ref_invariants(q):
    q = q.astype(np.int64)
    return {"sum": int(q.sum()), "min": int(q.min()), "max": int(q.max()),
            "tv": int(np.abs(q - np.roll(q, 1)).sum())}


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _checks_worker(rank, world, port, q, q0, starts, width, out):
    _init(rank, world, port)
    try:
        N = q.size
        off, nl = halo.partition(N, world, rank)
        mine = torch.from_numpy(q[off:off + nl].astype(np.int32))
        inv = checks.invariants(mine, chunk=97)             # small chunks: seams inside ranks
        win = checks.gather_windows(mine, off, N, starts, width)
        changed = checks.changed_cells(
            mine, lambda i, m: torch.from_numpy(q0[off + i:off + i + m].astype(np.int32)),
            chunk=101)
        t = shard.max_over_ranks(float(rank + 1))
        if rank == 0:
            out["inv"] = inv
            out["win"] = win.numpy()
            out["changed"] = changed
            out["tmax"] = t
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("N", [1000, 4099])
def test_split_verification_matches_single_domain(world, N):
    rng = np.random.default_rng(N + world)
    q0 = rng.integers(-5000, 5000, N)
    q = q0.copy()
    q[rng.integers(0, N, N // 3)] += rng.integers(1, 9, N // 3)   # "stepped" cells
    offsets = [halo.partition(N, world, r)[0] for r in range(world)]
    width = 64
    starts = checks.window_starts(N, offsets, width, n_random=2, seed=3)
    # windows straddle the wrap and every split point
    assert starts[0] + width > N
    for o in offsets[1:]:
        assert any(s < o < s + width for s in starts)
    out = mp.Manager().dict()
    port = _free_port()
    mp.spawn(_checks_worker, args=(world, port, q, q0, starts, width, out), nprocs=world)
    assert out["inv"] == _ref_invariants(q)
    ref_win = np.stack([q[(s + np.arange(width)) % N] for s in starts])
    assert np.array_equal(out["win"], ref_win)
    assert out["changed"] == int((q != q0).sum())
    assert out["tmax"] == float(world)


def test_single_process_verification():
    rng = np.random.default_rng(1)
    q = rng.integers(-100, 100, 777)
    t = torch.from_numpy(q.astype(np.int32))
    assert checks.invariants(t, chunk=50) == _ref_invariants(q)
    w = checks.gather_windows(t, 0, 777, [770, 5], 20).numpy()
    assert np.array_equal(w[0], q[(770 + np.arange(20)) % 777])


@pytest.mark.parametrize("B,P", [(10, 3), (7, 7), (65536 * 2, 2), (1001, 8)])
def test_ensemble_range_partition(B, P):
    ranges = [shard.ensemble_range(B, P, r) for r in range(P)]
    covered = np.concatenate([np.arange(f, f + c) for f, c in ranges])
    assert np.array_equal(covered, np.arange(B))                  # contiguous, no overlap
    counts = [c for _, c in ranges]
    assert max(counts) - min(counts) <= 1
    with pytest.raises(ValueError):
        shard.ensemble_range(B, P, P)
    with pytest.raises(ValueError):
        shard.ensemble_range(P - 1, P, 0)


def _ens_worker(rank, world, port, Bt, n, nsteps, out):
    _init(rank, world, port)
    try:
        first, cnt = shard.ensemble_range(Bt, world, rank)
        w = W.cfg("ens1")
        q0 = W.q0_ensemble(Bt, n=n, first=first, count=cnt).astype(np.int64)
        rule = oracle.Rule(oracle.LINEAR, w.delta, W.dt_dx(w))
        q = rule.run(q0, nsteps)                                     # no communication
        tmax = shard.max_over_ranks(0.5 * (rank + 1))                # the one collective
        out[rank] = (first, q, tmax)
    finally:
        dist.destroy_process_group()


def test_ensemble_shard_equals_unsharded():
    Bt, n, nsteps, world = 9, 1024, 50, 2
    out = mp.Manager().dict()
    mp.spawn(_ens_worker, args=(world, _free_port(), Bt, n, nsteps, out), nprocs=world)
    w = W.cfg("ens1")
    ref = oracle.Rule(oracle.LINEAR, w.delta, W.dt_dx(w)).run(
        W.q0_ensemble(Bt, n=n).astype(np.int64), nsteps)
    got = np.concatenate([out[r][1] for r in range(world)])
    assert [out[r][0] for r in range(world)] == [0, 5]
    assert np.array_equal(got, ref)
    assert all(out[r][2] == 1.0 for r in range(world))
