"""Batch x head sharding across the GPUs of one box.

Every (b, head) unit of the reference loop nest (attention.cpp:158-159) is
independent, so the path shards with NO collective in the compute: each rank
runs the same kernel on a disjoint block of units.  Collectives (NCCL over
NVLink/NVSwitch on GPUs, gloo in the CPU tests) appear only to scatter the
inputs from and gather the outputs to a root rank, for verification.

Plan rules (contiguous blocks, so a shard is one strided BSHD view):
  * L % world == 0      -> split the batch
  * h % world == 0      -> split the heads (all batches; strided view)
  * L >= world          -> uneven batch split (sizes differ by at most 1)
  * otherwise           -> uneven head split; ranks beyond L*h... get nothing
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List


@dataclass(frozen=True)
class Shard:
    rank: int
    b0: int
    b1: int
    h0: int
    h1: int

    @property
    def empty(self) -> bool:
        return self.b1 <= self.b0 or self.h1 <= self.h0

    @property
    def units(self) -> int:
        return 0 if self.empty else (self.b1 - self.b0) * (self.h1 - self.h0)


def _split(n: int, parts: int) -> List[tuple]:
    base, extra = divmod(n, parts)
    out, s = [], 0
    for i in range(parts):
        e = s + base + (1 if i < extra else 0)
        out.append((s, e))
        s = e
    return out


def plan(L: int, h: int, world: int) -> List[Shard]:
    if world < 1:
        raise ValueError("world must be >= 1")
    if L % world == 0 or (L >= world and h % world != 0):
        return [Shard(r, b0, b1, 0, h) for r, (b0, b1) in enumerate(_split(L, world))]
    return [Shard(r, 0, L, h0, h1) for r, (h0, h1) in enumerate(_split(h, world))]


def view(t, s: Shard):
    """The shard's BSHD view of a (L, N, h, d) tensor (torch or numpy)."""
    return t[s.b0:s.b1, :, s.h0:s.h1, :]


def lse_view(t, s: Shard):
    """The shard's view of an (L, h, N) LSE tensor."""
    return t[s.b0:s.b1, s.h0:s.h1, :]


def scatter_gather(q, k, v, compute: Callable, L: int, N: int, h: int, d: int, make_empty: Callable,
                   root: int = 0):
    """Scatter Q/K/V from `root`, run `compute(q_s, k_s, v_s) -> (o_s, lse_s)`
    on every rank's shard, gather O and LSE back to `root`.

    q/k/v are full tensors on the root (ignored elsewhere).  `make_empty(shape,
    kind)` allocates a contiguous tensor on this rank's device ("x" for 16-bit
    activations, "f32" for LSE).  Uses torch.distributed point-to-point ops
    (NCCL send/recv over NVLink for CUDA tensors, gloo for CPU tensors).
    Returns (O, LSE) on the root, (None, None) elsewhere."""
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    shards = plan(L, h, world)
    mine = shards[rank]

    def shape_of(s):
        return (s.b1 - s.b0, N, s.h1 - s.h0, d)

    # scatter
    if rank == root:
        for s in shards:
            if s.rank == root or s.empty:
                continue
            for t in (q, k, v):
                dist.send(view(t, s).contiguous(), dst=s.rank)
        local = [view(t, mine).contiguous() for t in (q, k, v)] if not mine.empty else None
    else:
        local = None
        if not mine.empty:
            local = [make_empty(shape_of(mine), "x") for _ in range(3)]
            for t in local:
                dist.recv(t, src=root)
    # compute (no collective)
    out = compute(*local) if local is not None else None
    # gather
    if rank == root:
        O = make_empty((L, N, h, d), "x")
        LSE = make_empty((L, h, N), "f32")
        for s in shards:
            if s.empty:
                continue
            if s.rank == root:
                view(O, s)[...] = out[0]
                lse_view(LSE, s)[...] = out[1]
            else:
                o_s = make_empty(shape_of(s), "x")
                l_s = make_empty((s.b1 - s.b0, s.h1 - s.h0, N), "f32")
                dist.recv(o_s, src=s.rank)
                dist.recv(l_s, src=s.rank)
                view(O, s)[...] = o_s
                lse_view(LSE, s)[...] = l_s
        return O, LSE
    if out is not None:
        dist.send(out[0].contiguous(), dst=root)
        dist.send(out[1].contiguous(), dst=root)
    return None, None
