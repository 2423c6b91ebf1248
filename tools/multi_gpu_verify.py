#!/usr/bin/env python
"""Multi-GPU run of the FMHA forward, sharded over batch x heads
(SURVEY.md 8(e)): rank 0 owns the full Q/K/V, NCCL point-to-point sends
scatter each rank's contiguous (b, head) block over NVLink, every rank runs
the sm_100a kernel on its shard with no collective in the compute, and the
O / LSE shards are gathered back to rank 0, which checks them bit for bit
against a single-GPU run of the same problem.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/multi_gpu_verify.py \
        [--batch 8 --heads 32 --seqlen 16384 --headdim 128 --dtype bf16]

Prints one JSON line on rank 0: per-rank compute time (max over ranks),
aggregate TFLOP/s, scatter/gather times (outside the compute), and the
parity verdict.
"""
import argparse
import json
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2312_11918_b200 as fm  # noqa: E402
from paper_2312_11918_b200 import shard  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--heads", type=int, default=32)
    ap.add_argument("--seqlen", type=int, default=16384)
    ap.add_argument("--headdim", type=int, default=128)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--iterations", type=int, default=5)
    a = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    td = torch.bfloat16 if a.dtype == "bf16" else torch.float16
    L, N, h, d = a.batch, a.seqlen, a.heads, a.headdim
    q = k = v = None
    if rank == 0:
        g = torch.Generator(device=dev).manual_seed(7)
        q, k, v = (torch.randn((L, N, h, d), generator=g, device=dev).to(td) for _ in range(3))

    times = {}

    def compute(qs, ks, vs):
        o, lse = fm.fmha_fwd(qs, ks, vs)  # warm-up / result
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iterations):
            fm.fmha_fwd(qs, ks, vs, o=o, lse=lse)
        e1.record()
        torch.cuda.synchronize()
        times["ms"] = e0.elapsed_time(e1) / a.iterations
        return o, lse

    def make_empty(shape, kind):
        return torch.empty(shape, dtype=td if kind == "x" else torch.float32, device=dev)

    dist.barrier()
    t0 = time.perf_counter()
    O, LSE = shard.scatter_gather(q, k, v, compute, L, N, h, d, make_empty)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    mine = shard.plan(L, h, world)[rank]
    my_flops = 4 * mine.units * N * N * d
    t = torch.tensor([times.get("ms", 0.0)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        o_ref, lse_ref = fm.fmha_fwd(q, k, v)
        torch.cuda.synchronize()
        same = bool(torch.equal(O, o_ref)) and bool(torch.equal(LSE, lse_ref))
        total = 4 * L * h * N * N * d
        print(json.dumps({
            "world": world, "L": L, "h": h, "N": N, "d": d, "dtype": a.dtype,
            "plan": [s.__dict__ for s in shard.plan(L, h, world)],
            "compute_ms_max_over_ranks": float(t.item()),
            "aggregate_tflops": total / (float(t.item()) * 1e-3) / 1e12,
            "rank0_shard_tflops": my_flops / (times["ms"] * 1e-3) / 1e12,
            "scatter_compute_gather_wall_s": wall,
            "bitwise_equal_to_single_gpu": same,
        }), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
