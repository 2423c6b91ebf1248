"""Batch x head sharding on CPU: the plan covers every
(b, head) unit exactly once, and a world_size-2 gloo scatter -> compute ->
gather reproduces the single-process oracle bit for bit."""
import os
import socket

import numpy as np
import pytest

from paper_2312_11918_b200 import shard


@pytest.mark.parametrize("L,h,world", [(8, 32, 1), (8, 32, 2), (8, 32, 8), (4, 16, 8), (3, 5, 2),
                                       (1, 12, 8), (1, 3, 8), (16, 12, 3), (2, 8, 4)])
def test_plan_partitions_units(L, h, world):
    sh = shard.plan(L, h, world)
    assert len(sh) == world and [s.rank for s in sh] == list(range(world))
    cover = np.zeros((L, h), np.int32)
    for s in sh:
        if not s.empty:
            cover[s.b0:s.b1, s.h0:s.h1] += 1
    assert (cover == 1).all()
    sizes = [s.units for s in sh]
    assert max(sizes) - min(sizes) <= max(L, h)  # contiguous, near-balanced
    if L % world == 0:
        assert all(s.h0 == 0 and s.h1 == h for s in sh)  # batch split: dense shards


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, L, N, h, d, out_path):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from oracle import oracle as orc
    from paper_2312_11918_b200 import shard as sh

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    q = k = v = None
    if rank == 0:
        q, k, v = (torch.from_numpy(x) for x in orc.problem(L, N, h, d, 42, dtype="f16"))

    def compute(qs, ks, vs):  # stands in for the GPU kernel on this rank
        o, lse = orc.fmha_forward(qs.numpy(), ks.numpy(), vs.numpy(), 64, 64, threads=1)
        return torch.from_numpy(o), torch.from_numpy(lse)

    def make_empty(shape, kind):
        return torch.empty(shape, dtype=torch.float32)

    O, LSE = sh.scatter_gather(q, k, v, compute, L, N, h, d, make_empty)
    if rank == 0:
        np.savez(out_path, O=O.numpy(), LSE=LSE.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("L,h", [(2, 3), (1, 4), (3, 1)])
def test_gloo_world2_scatter_compute_gather(tmp_path, oracle, L, h):
    import torch.multiprocessing as mp
    N, d = 128, 32
    out = str(tmp_path / "out.npz")
    mp.start_processes(_worker, args=(2, _free_port(), L, N, h, d, out), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(out)
    q, k, v = oracle.problem(L, N, h, d, 42, dtype="f16")
    o, lse = oracle.fmha_forward(q, k, v, 64, 64)
    np.testing.assert_array_equal(got["O"], o)
    np.testing.assert_array_equal(got["LSE"], lse)
