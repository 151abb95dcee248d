"""Halo-exchange layer: one periodic 1D domain split contiguously across ranks.

Rank r owns global cells [r*N/P, (r+1)*N/P).  Its device buffer
holds  [H halo | n_local owned | H halo]  int32 cells.  Per temporal block of
k <= H steps there is exactly one exchange (the only data-path communication
of the method, "nearest-neighbour communication pattern"):

  left  halo  <- the H owned cells at the right end of rank r-1
  right halo  <- the H owned cells at the left end of rank r+1

followed by one fqnm_step_block launch that advances the owned cells by k
steps (overlapped trapezoids: the halo supplies the light cone).

Transports
  * `DistTransport`  torch.distributed point-to-point (NCCL over NVLink on the
                     GPU box; gloo in the CPU tests), periodic ring.
  * `LocalTransport` several subdomains in one process (virtual ranks), halos
                     filled by tensor copies - lets one GPU test the split path
                     without kernels that wait on each other.

The block stepper is injected (`block_fn(src, dst, k)`): the product uses the
C-ABI kernel `fqnm_step_block`; CPU tests inject the oracle.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence


def partition(n_global: int, nranks: int, rank: int):
    """(offset, n_local) of rank's contiguous block; blocks differ by at most one cell."""
    base, rem = divmod(n_global, nranks)
    off = rank * base + min(rank, rem)
    return off, base + (1 if rank < rem else 0)


def block_schedule(nsteps: int, k: int) -> List[int]:
    """Split nsteps into blocks of at most k steps (all but possibly the last are k)."""
    out = []
    left = nsteps
    while left > 0:
        out.append(min(k, left))
        left -= out[-1]
    return out


class DistTransport:
    """Periodic ring exchange with torch.distributed P2P ops (backend-agnostic)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def exchange(self, bufs: Sequence, n_locals: Sequence[int], H: int):
        (buf,), (n,) = bufs, n_locals
        dist = self.dist
        if self.size == 1:
            buf[:H].copy_(buf[n:n + H])
            buf[n + H:n + 2 * H].copy_(buf[H:2 * H])
            return
        left = (self.rank - 1) % self.size
        right = (self.rank + 1) % self.size
        gl = dist.get_global_rank(self.group, left) if self.group is not None else left
        gr = dist.get_global_rank(self.group, right) if self.group is not None else right
        # Order and tags pair the messages even when left == right (P = 2):
        # tag 1 = a right edge travelling right, tag 2 = a left edge travelling left.
        ops = [
            dist.P2POp(dist.isend, buf[n:n + H], gr, self.group, 1),          # right edge -> right
            dist.P2POp(dist.isend, buf[H:2 * H], gl, self.group, 2),          # left edge -> left
            dist.P2POp(dist.irecv, buf[:H], gl, self.group, 1),               # left halo
            dist.P2POp(dist.irecv, buf[n + H:n + 2 * H], gr, self.group, 2),  # right halo
        ]
        for r in dist.batch_isend_irecv(ops):
            r.wait()


class LocalTransport:
    """All subdomains live in this process (virtual ranks on one device)."""

    def exchange(self, bufs: Sequence, n_locals: Sequence[int], H: int):
        P = len(bufs)
        for r in range(P):
            lb, ln = bufs[(r - 1) % P], n_locals[(r - 1) % P]
            rb = bufs[(r + 1) % P]
            b, n = bufs[r], n_locals[r]
            b[:H].copy_(lb[ln:ln + H])
            b[n + H:n + 2 * H].copy_(rb[H:2 * H])


class SplitDomain:
    """Owned state of one or more subdomains (virtual ranks) plus the block loop.

    Parameters
      n_locals   owned cells of each subdomain held by this process
      H          halo width (>= steps per block, multiple of 4)
      transport  DistTransport or LocalTransport
      block_fn   callable(src, dst, k) advancing owned cells of one subdomain
                 buffer by k steps; the i-th subdomain uses block_fns[i]
      alloc      callable(n_cells) -> zero-initialised 1-D buffer
    """

    def __init__(self, n_locals: Sequence[int], H: int, transport, block_fns: Sequence[Callable],
                 alloc: Callable):
        if H < 1:
            raise ValueError("halo must be >= 1")
        for n in n_locals:
            if n < H:
                raise ValueError(f"subdomain of {n} cells is smaller than the halo {H}")
        self.n_locals = list(n_locals)
        self.H = H
        self.transport = transport
        self.block_fns = list(block_fns)
        self.bufs = [[alloc(n + 2 * H), alloc(n + 2 * H)] for n in self.n_locals]
        self.cur = 0

    def owned(self, i: int = 0):
        n, H = self.n_locals[i], self.H
        return self.bufs[i][self.cur][H:H + n]

    def load(self, parts: Sequence):
        self.cur = 0
        for i, q in enumerate(parts):
            self.owned(i).copy_(q)

    def step(self, nsteps: int, k: Optional[int] = None):
        k = self.H if k is None else min(k, self.H)
        for kb in block_schedule(nsteps, k):
            src = [b[self.cur] for b in self.bufs]
            dst = [b[self.cur ^ 1] for b in self.bufs]
            self.transport.exchange(src, self.n_locals, self.H)
            for i in range(len(self.bufs)):
                self.block_fns[i](src[i], dst[i], kb)
            self.cur ^= 1


class P2PRing:
    """Fused peer-memory halo exchange (FQNM_HALO plans with p2p = 1).

    The stepping kernel itself writes each rank's H edge cells into its ring
    neighbours' next buffers (NVLink peer stores, CUDA IPC across processes) and
    releases a block tag; no NCCL call and no host round trip per block.

    * virtual ranks: `P2PRing.virtual(plans)` connects plans of one device in a
      ring and `step` interleaves their launches (fqnm_step_group).
    * one rank per GPU: `P2PRing.distributed(plan, group)` exchanges CUDA IPC
      handles of the plan buffers with torch.distributed and connects the plan;
      every rank then calls `step(nsteps)` (collective)."""

    def __init__(self, plans, opened=()):
        self.plans = list(plans)
        self._opened = list(opened)

    @classmethod
    def virtual(cls, plans):
        import paper_2604_06947_b200 as F
        P = len(plans)
        bufs = [F.fqnm_halo_buffers(p) for p in plans]
        for i, p in enumerate(plans):
            l, r = (i - 1) % P, (i + 1) % P
            F.fqnm_halo_connect(p, bufs[l], plans[l].desc.n_local, bufs[r], plans[r].desc.n_local)
        return cls(plans)

    @classmethod
    def distributed(cls, plan_factory, group=None, device=None):
        """Collective and failure-safe: every rank builds its p2p plan with
        `plan_factory()`, exports CUDA IPC handles, all-gathers them, opens its
        neighbours'; if any rank fails anywhere, every rank gets None (the
        caller falls back to the NCCL transport) - no rank is left waiting."""
        import torch
        import torch.distributed as dist
        import paper_2604_06947_b200 as F
        rank, size = dist.get_rank(group), dist.get_world_size(group)
        plan, handles, n_local, err = None, None, 0, ""
        try:
            plan = plan_factory()
            mine = F.fqnm_halo_buffers(plan)
            handles = [F.fqnm_ipc_export(x) for x in mine]
            n_local = plan.desc.n_local
        except Exception as ex:                              # noqa: BLE001
            err = str(ex)[:200]
        info = [None] * size
        dist.all_gather_object(info, (handles, n_local, err), group=group)
        opened, ok = [], all(i[0] is not None for i in info)
        if ok:
            try:
                cache = {}

                def ptrs(r):
                    if r == rank:
                        return mine
                    if r not in cache:
                        cache[r] = tuple(F.fqnm_ipc_open(h) for h in info[r][0])
                        opened.extend(cache[r])
                    return cache[r]
                l, r = (rank - 1) % size, (rank + 1) % size
                F.fqnm_halo_connect(plan, ptrs(l), info[l][1], ptrs(r), info[r][1])
            except Exception as ex:                          # noqa: BLE001
                ok, err = False, str(ex)[:200]
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        if int(flag) == 0:
            for ptr in opened:
                try:
                    F.fqnm_ipc_close(ptr)
                except Exception:                            # noqa: BLE001
                    pass
            errs = [i[2] for i in info if i[2]] + ([err] if err else [])
            return None, "; ".join(errs) or "peer setup failed on another rank"
        dist.barrier(group)
        return cls([plan], opened), ""

    def load(self, parts):
        import paper_2604_06947_b200 as F
        for p, q in zip(self.plans, parts):
            F.owned_tensor(p).copy_(q)

    def owned(self, i: int = 0):
        import paper_2604_06947_b200 as F
        return F.owned_tensor(self.plans[i])

    def step(self, nsteps: int):
        import paper_2604_06947_b200 as F
        if len(self.plans) == 1:
            F.fqnm_step(self.plans[0], None, nsteps)
        else:
            F.fqnm_step_group(self.plans, nsteps)

    def close(self):
        import paper_2604_06947_b200 as F
        for ptr in self._opened:
            F.fqnm_ipc_close(ptr)
        self._opened = []
