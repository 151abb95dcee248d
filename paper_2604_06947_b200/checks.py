"""Run verification of a (possibly split) 1D periodic state, by plain torch reductions
that share nothing with the FQNM kernels (SURVEY §8(c)-C6, §8(e) "Verification").

Rank r of P holds the owned cells [off_r, off_r + n_r) of one periodic domain of N
cells (contiguous split, `halo.partition`).  Everything here works on CUDA tensors
under NCCL and on CPU tensors under gloo (the CPU tests), and with no process group
at all (P = 1).

* `invariants`: exact integer sum, min, max and periodic total variation of the whole
  domain.  The TV includes the P cross-rank edge pairs |q[off_{r+1}] - q[off_{r+1} - 1]|
  (and the periodic wrap |q_0 - q_{N-1}|), gathered from every rank's first and last
  cell.  The theorems they check: exact conservation (Lemma discrete Green/Stokes,
  P:309-333), maximum principle and TVD (Lemma CFL).
* `gather_windows`: cells at arbitrary global windows (which may straddle split points
  and the periodic wrap), assembled on every rank by a SUM all-reduce of zero-filled
  buffers (each cell is owned by exactly one rank).
* `changed_cells`: the number of cells that differ from the initial data, a cheap proof
  that the timed run really moved the state (a no-op kernel would keep the
  invariants).
* `window_starts`: the parity windows of a run: the periodic wrap, every split point,
  the middle and seeded random positions.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence

import numpy as np


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def _allreduce(t, op: str, group=None):
    d = _dist()
    if d is None:
        return t
    ops = {"sum": d.ReduceOp.SUM, "min": d.ReduceOp.MIN, "max": d.ReduceOp.MAX}
    d.all_reduce(t, op=ops[op], group=group)
    return t


def invariants(q, chunk: int = 1 << 28, group=None) -> dict:
    """Whole-domain {sum, min, max, tv} of the owned part q (1-D int32/int64 tensor) of a
    periodic domain split contiguously in rank order over the group."""
    import torch
    n = q.numel()
    tot = torch.zeros((), dtype=torch.int64, device=q.device)
    tv = torch.zeros((), dtype=torch.int64, device=q.device)
    mn = torch.full((), np.iinfo(np.int64).max, dtype=torch.int64, device=q.device)
    mx = torch.full((), np.iinfo(np.int64).min, dtype=torch.int64, device=q.device)
    for i in range(0, n, chunk):
        c = q[i:i + chunk]
        tot += c.sum(dtype=torch.int64)
        mn = torch.minimum(mn, c.min().to(torch.int64))
        mx = torch.maximum(mx, c.max().to(torch.int64))
        seg = q[i:min(i + chunk + 1, n)].to(torch.int64)            # pairs inside the rank
        tv += (seg[1:] - seg[:-1]).abs().sum()
    _allreduce(tot, "sum", group)
    _allreduce(tv, "sum", group)
    _allreduce(mn, "min", group)
    _allreduce(mx, "max", group)
    # cross-rank edge pairs and the periodic wrap: every rank's (first, last) cell
    d = _dist()
    P = d.get_world_size(group) if d is not None else 1
    r = d.get_rank(group) if d is not None else 0
    ends = torch.zeros(2 * P, dtype=torch.int64, device=q.device)
    ends[2 * r] = q[0].to(torch.int64)
    ends[2 * r + 1] = q[n - 1].to(torch.int64)
    _allreduce(ends, "sum", group)
    e = ends.view(P, 2)
    first_next = torch.roll(e[:, 0], -1)                 # first cell of rank r+1 (wraps)
    tv += (first_next - e[:, 1]).abs().sum()
    return {"sum": int(tot), "min": int(mn), "max": int(mx), "tv": int(tv)}


def gather_windows(q, off: int, N: int, starts: Sequence[int], width: int, group=None):
    """[len(starts), width] int64 tensor of the global cells (start + j) mod N, on every
    rank; q is this rank's owned part, which begins at global cell `off`."""
    import torch
    n = q.numel()
    out = torch.zeros((len(starts), width), dtype=torch.int64, device=q.device)
    j = torch.arange(width, dtype=torch.int64, device=q.device)
    for w, a in enumerate(starts):
        g = (int(a) + j) % N                              # global indices of the window
        loc = g - off
        mine = (loc >= 0) & (loc < n)
        if bool(mine.any()):
            out[w, mine] = q[loc[mine]].to(torch.int64)
    return _allreduce(out, "sum", group)


def changed_cells(q, q0_fn: Callable[[int, int], "object"], chunk: int = 1 << 27,
                  group=None) -> int:
    """Number of cells (whole domain) where q differs from the initial data;
    q0_fn(start, count) regenerates the initial cells [start, start + count) of this
    rank's part (same device and dtype as q)."""
    import torch
    n = q.numel()
    cnt = torch.zeros((), dtype=torch.int64, device=q.device)
    for i in range(0, n, chunk):
        m = min(chunk, n - i)
        cnt += (q[i:i + m] != q0_fn(i, m)).sum()
    return int(_allreduce(cnt, "sum", group))


def window_starts(N: int, offsets: Sequence[int], width: int, n_random: int = 1,
                  seed: int = 0) -> List[int]:
    """Windows of `width` cells: straddling the periodic wrap, straddling each split point
    offsets[1:], in the middle of the domain, and n_random seeded random positions."""
    starts = [(N - width // 2) % N]
    starts += [(o - width // 2) % N for o in offsets[1:]]
    starts.append(N // 2 + 12345 if N > 2 * width + 12345 else N // 2)
    rng = np.random.default_rng(seed)
    starts += [int(rng.integers(0, N)) for _ in range(n_random)]
    out, seen = [], set()
    for s in starts:
        s = (s // 4) * 4 % N
        if s not in seen:
            seen.add(s)
            out.append(s)
    return out
