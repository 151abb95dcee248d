"""Split-domain (halo-exchange) path on CPU: world_size-2 and 3 `gloo` process
groups run the real torch.distributed transport (`halo.DistTransport`) and the
block loop of `halo.SplitDomain`; the per-block stepper is the oracle (CPU
tests may not launch kernels).  The gathered state must equal the
single-domain oracle run bit for bit (decomposition invariance)."""
import os
import socket
from fractions import Fraction

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads as W
from paper_2604_06947_b200 import halo

CASES = {
    "eo": (oracle.BURGERS_EO, "1e-5", Fraction(4, 15), 1, 100000, 20000),
    "lin": (oracle.LINEAR, "1e-4", Fraction(1, 2), 1, 5000, 0),
    "lin_left": (oracle.LINEAR, "1e-3", Fraction(1, 3), -1, 3000, 100),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_block(rule, H):
    def fn(src, dst, k):
        n = src.numel() - 2 * H
        out = rule.run(src.numpy().astype(np.int64), k)     # periodic wrap stays in the halos
        dst[H:H + n] = torch.from_numpy(out[H:H + n].astype(np.int32))
    return fn


def _worker(rank, world, port, case, n, H, nsteps, q0, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        kind, delta, lam, param, _, _ = CASES[case]
        rule = oracle.Rule(kind, delta, lam, Fraction(param))
        off, nl = halo.partition(n, world, rank)
        sd = halo.SplitDomain([nl], H, halo.DistTransport(), [_oracle_block(rule, H)],
                              lambda m: torch.zeros(m, dtype=torch.int32))
        sd.load([torch.from_numpy(q0[off:off + nl].astype(np.int32))])
        sd.step(nsteps)
        parts = [torch.zeros(halo.partition(n, world, r)[1], dtype=torch.int32)
                 for r in range(world)]
        mine = sd.owned(0).clone()
        if rank == 0:
            for r in range(1, world):
                dist.recv(parts[r], src=r)
            parts[0] = mine
            result[:] = torch.cat(parts)
        else:
            dist.send(mine, dst=0)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world,H,nsteps", [("eo", 2, 8, 37), ("lin", 2, 16, 40),
                                                 ("lin_left", 3, 4, 21), ("eo", 3, 12, 30)])
def test_split_domain_gloo_matches_single_domain(case, world, H, nsteps):
    kind, delta, lam, param, amp, off = CASES[case]
    n = 997
    rng = np.random.default_rng(11)
    q0 = W.smooth_random(rng, n, amp, off)
    ref = oracle.Rule(kind, delta, lam, Fraction(param)).run(q0, nsteps)
    result = torch.zeros(n, dtype=torch.int32).share_memory_()
    mp.start_processes(_worker, args=(world, _free_port(), case, n, H, nsteps, q0, result),
                       nprocs=world, join=True, start_method="fork")
    assert np.array_equal(result.numpy().astype(np.int64), ref)


def test_partition_and_schedule():
    for n in (10, 997, 1 << 20):
        for P in (1, 2, 3, 7, 8):
            parts = [halo.partition(n, P, r) for r in range(P)]
            assert parts[0][0] == 0 and sum(nl for _, nl in parts) == n
            for (o1, n1), (o2, _) in zip(parts, parts[1:]):
                assert o1 + n1 == o2
            assert max(nl for _, nl in parts) - min(nl for _, nl in parts) <= 1
    assert halo.block_schedule(50, 16) == [16, 16, 16, 2]
    assert halo.block_schedule(0, 8) == []


def test_local_transport_virtual_ranks_cpu():
    """Virtual ranks in one process (the GPU test uses the same transport with kernels)."""
    kind, delta, lam, param, amp, off = CASES["eo"]
    rule = oracle.Rule(kind, delta, lam)
    n, H = 500, 8
    rng = np.random.default_rng(3)
    q0 = W.smooth_random(rng, n, amp, off)
    ref = rule.run(q0, 29)
    for P in (1, 2, 4):
        parts = [halo.partition(n, P, r) for r in range(P)]
        sd = halo.SplitDomain([nl for _, nl in parts], H, halo.LocalTransport(),
                              [_oracle_block(rule, H)] * P,
                              lambda m: torch.zeros(m, dtype=torch.int32))
        sd.load([torch.from_numpy(q0[o:o + nl].astype(np.int32)) for o, nl in parts])
        sd.step(29)
        got = torch.cat([sd.owned(i) for i in range(P)]).numpy().astype(np.int64)
        assert np.array_equal(got, ref)


def _p2p_fallback_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def factory():
            if rank == 1:
                raise RuntimeError("no peer access on rank 1")
            raise RuntimeError("no GPU in the CPU test")
        ring, why = halo.P2PRing.distributed(factory, None, "cpu")
        out[rank] = 1 if (ring is None and "rank 1" in why) else 0
    finally:
        dist.destroy_process_group()


def test_p2p_setup_failure_is_collective():
    """If the fused peer-memory setup fails on any rank, every rank falls back
    (returns None) instead of waiting in a collective the failed rank skipped."""
    out = torch.zeros(2, dtype=torch.int32).share_memory_()
    mp.start_processes(_p2p_fallback_worker, args=(2, _free_port(), out), nprocs=2, join=True,
                       start_method="fork")
    assert out.tolist() == [1, 1]
