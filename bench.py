#!/usr/bin/env python
"""bench.py -- FMHA forward TFLOP/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c1|c2|c3|c4|c5]

A step is one FMHA forward (one kernel launch) over the configured problem,
inputs resident in HBM.  Default workload: config 3 of BASELINE.json
(L=4, h=16, N=4096, d=128, fp16: the paper's / FA2 benchmark shape and the
north-star target shape d=128, N>=4k).  Under torchrun each rank runs its own
batch shard of a global batch of 4*N (weak scaling, no collective in the data
path: SURVEY.md 8(e)); ``--config c5`` instead shards config 5's batch of 8
over the ranks (strong scaling).

FLOPs = 4*L*h*N^2*d (attention_flops, attention.cpp:191-193).  Timing: CUDA
events on the launching stream around every step, barrier + synchronize on
both sides of the timed loop, max over ranks.  Rank 0 prints ONE JSON line.
"""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": dict(L=1, h=1, N=512, d=64, dtype="fp16", desc="config 1: L=1,h=1,N=512,d=64 fp16 (CPU-oracle case)"),
    "c2": dict(L=16, h=12, N=512, d=64, dtype="fp16", desc="config 2: distilbert-like L=16,h=12,N=512,d=64 fp16"),
    "c3": dict(L=4, h=16, N=4096, d=128, dtype="fp16", desc="config 3: L=4,h=16,N=4096,d=128 fp16 (FA2/paper shape)"),
    "c4": dict(L=2, h=8, N=8192, d=256, dtype="fp16", desc="config 4: L=2,h=8,N=8192,d=256 fp16"),
    "c5": dict(L=8, h=32, N=16384, d=128, dtype="bf16", desc="config 5: L=8,h=32,N=16384,d=128 bf16"),
}
L2_BYTES = 126 * 2 ** 20
FALLBACK_PEAK_TFLOPS = 1590.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=120.0,
                    help="reference arm: CPU-time budget for the whole --warmup + --steps run")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def flops(L, N, h, d):
    return 4 * L * h * N * N * d


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["bf16_tflops"]), float(j.get("bf16_tflops_sustained", j["bf16_tflops"])), "measured"
    return FALLBACK_PEAK_TFLOPS, 1400.0, "fallback"


def workload(cfg_name, world, rank):
    """Per-rank problem shape and the global description."""
    c = dict(CONFIGS[cfg_name])
    if cfg_name == "c5" and world > 1:
        if c["L"] % world:
            raise SystemExit(f"c5 batch {c['L']} not divisible by {world} GPUs")
        local = dict(c, L=c["L"] // world)
        scaling = "strong"
        global_L = c["L"]
    else:
        local = c
        scaling = "weak"
        global_L = c["L"] * world
    return c, local, scaling, global_L


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML while the timed region runs."""

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - NVML optional
            self.nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self.nv
        names = {}
        if nv is not None:
            for attr, name in (("nvmlClocksEventReasonHwSlowdown", "hw_slowdown"),
                               ("nvmlClocksEventReasonHwThermalSlowdown", "hw_thermal_slowdown"),
                               ("nvmlClocksEventReasonSwThermalSlowdown", "sw_thermal_slowdown"),
                               ("nvmlClocksEventReasonSwPowerCap", "sw_power_cap"),
                               ("nvmlClocksEventReasonGpuIdle", None)):
                if hasattr(nv, attr):
                    names[getattr(nv, attr)] = name
        while not self._stop.is_set():
            if nv is not None:
                try:
                    self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    for bit, name in names.items():
                        if name and (r & bit):
                            self.reasons.add(name)
                except Exception:  # noqa: BLE001
                    pass
            time.sleep(0.005)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join()

    def summary(self):
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


def cpu_baseline(cfg, threads=None, budget_s=20.0, mode="heads"):
    """Reference CPU path on this host's cores over a bounded sample of the
    workload: oracle/_ref (the reference compiled from its sources) when
    present, else the oracle port.  Returns the cpu_baseline dict."""
    import numpy as np
    from oracle import oracle as orc
    threads = threads or orc.default_threads()
    N, d = cfg["N"], cfg["d"]
    n_heads_total = cfg["L"] * cfg["h"]
    rng = np.random.default_rng(0)
    kind = "reference" if orc.ref_available() else "port"
    qdt = "bf16" if cfg["dtype"] == "bf16" else "f16"
    if mode == "heads":
        heads = min(threads, n_heads_total)
        qh, kh, vh = (orc.quantize(rng.standard_normal((heads, N, d), dtype=np.float32), qdt) for _ in range(3))
        t0 = time.perf_counter()
        if kind == "reference":
            orc.ref_fmha_forward_heads(qh, kh, vh, 128, 128, threads=threads)
        else:
            orc.fmha_forward(qh.reshape(heads, N, 1, d), kh.reshape(heads, N, 1, d),
                             vh.reshape(heads, N, 1, d), 128, 128, threads=threads, want_lse=False)
        dt = time.perf_counter() - t0
        fl = heads * 4 * N * N * d
        sample = (f"{heads} whole (b,h) heads of {cfg['desc']}, fmha_forward ExactF32 tile 128x128 "
                  f"(reference flags -O2), one head per thread")
    else:  # tiles: `mode` tiles per thread through the restated per-tile driver
        ntiles = max(1, int(mode)) * threads
        q, k, v = (orc.quantize(rng.standard_normal((1, N, 1, d), dtype=np.float32), qdt) for _ in range(3))
        tiles = [(0, 0, i % (N // 128)) for i in range(ntiles)]
        t0 = time.perf_counter()
        if kind == "reference":
            orc.ref_fmha_tiles(q, k, v, tiles, 128, 128, threads=threads)
        else:
            orc.fmha_tiles(q, k, v, tiles, 128, 128, threads=threads)
        dt = time.perf_counter() - t0
        fl = ntiles * 4 * 128 * N * d
        sample = (f"{ntiles} 128-row Q tiles of {cfg['desc']} through the reference's "
                  f"gemm_nt_accumulate/online_softmax_step (restated tile driver), {threads} threads")
    return {"value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": kind,
            "sample": sample, "seconds": round(dt, 3), "gflop": round(fl / 1e9, 2),
            "host_cpus": os.cpu_count()}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as orc
    if not os.path.exists(orc.LIB_PATH):
        orc.build()
    cfg, local, scaling, global_L = workload(args.config, 1, 0)
    threads = orc.default_threads()
    # per-step sample sized so W + K steps stay within ~2 minutes
    per_step_budget = args.ref_seconds / max(1, args.steps + args.warmup)
    probe = cpu_baseline(cfg, threads, mode="1")
    tiles_per_thread = max(1, int(per_step_budget / max(probe["seconds"], 1e-3)))
    for _ in range(args.warmup):
        cpu_baseline(cfg, threads, mode=str(tiles_per_thread))
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_baseline(cfg, threads, mode=str(tiles_per_thread)))
    wall = time.perf_counter() - t0
    total_fl = sum(v["gflop"] for v in vals) * 1e9
    value = total_fl / wall / 1e12
    cb = dict(vals[-1])
    cb["value"] = value
    line = {
        "impl": "reference", "metric": "FMHA forward TFLOP/s (fp16, non-causal)", "value": value,
        "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall / args.steps * 1e3, "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic N(0,1) rounded to the 16-bit type",
        "config": {"workload": cfg["desc"], "L": global_L, "h": cfg["h"], "N": cfg["N"], "d": cfg["d"],
                   "causal": False, "parallelism": "host threads"},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2312_11918_b200 as fm

    rank, world, local_rank = dist_env()
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg, loc, scaling, global_L = workload(args.config, world, rank)
    L, N, h, d = loc["L"], loc["N"], loc["h"], loc["d"]
    td = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float16
    g = torch.Generator(device=dev).manual_seed(42 + rank)
    q, k, v = (torch.randn((L, N, h, d), generator=g, device=dev, dtype=torch.float32).to(td) for _ in range(3))
    o = torch.empty_like(q)
    lse = torch.empty((L, h, N), dtype=torch.float32, device=dev)
    work_bytes = 4 * q.numel() * q.element_size() + lse.numel() * 4
    flush = None
    if work_bytes < 2 * L2_BYTES:
        flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        fm.fmha_fwd(q, k, v, o=o, lse=lse, stream=stream)
        return fm.launch_count()

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        wall0 = time.perf_counter()
        for i in range(args.steps):
            if flush is not None:
                flush.zero_()  # L2 flush between timed steps (outside the events)
            starts[i].record(stream)
            launches += step()
            ends[i].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    if world > 1:
        dist.barrier()
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    per_rank_flops = flops(L, N, h, d)
    value = world * per_rank_flops * args.steps / (ms_max * 1e-3) / 1e12
    per_launch_ms = ms_max / args.steps
    peak, peak_sus, peak_kind = peaks()
    achieved = per_rank_flops / (per_launch_ms * 1e-3) / 1e12

    # ---- end to end through the public host API (pinned host buffers) ----
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(fm, q, k, v, cfg, args, world, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(cfg)
        except Exception as ex:  # noqa: BLE001
            cpu = {"value": None, "error": str(ex)}

    if rank == 0:
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
        if os.path.exists(prof):
            with open(prof) as f:
                j = json.load(f)
            traffic = j.get(args.config, {}).get("dram_bytes_per_launch")
        line = {
            "metric": "FMHA forward TFLOP/s (fp16, non-causal)", "value": value, "unit": "TFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": cfg["dtype"],
            "data": "synthetic: device-side seeded N(0,1) rounded to the 16-bit type",
            "config": {"workload": cfg["desc"], "L": global_L, "h": h, "N": N, "d": d, "causal": False,
                       "per_gpu_L": L, "parallelism": f"batch-shard x{world} (no collective)",
                       "kernel": fm.kernel_for(L, N, h, d, cfg["dtype"]),
                       "l2": ("inputs %.0f MB per GPU > 126 MB L2" % (work_bytes / 2 ** 20)) if flush is None
                       else "L2 flushed (256 MB write) between timed steps"},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "peak_kind": f"{peak_kind} bf16 dense (burst)",
                         "frac_of_sustained": achieved / peak_sus, "frac_of_datasheet_2250": achieved / 2250.0,
                         "traffic": traffic,
                         "algorithmic_flops_per_launch": per_rank_flops,
                         "algorithmic_bytes_per_launch": 8 * L * h * N * d + 4 * L * h * N},
            "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
            "wall_s_timed": wall,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def measure_e2e(fm, q, k, v, cfg, args, world, dev):
    """Same metric through fmha_fwd_host: pinned host fp16 buffers, H2D of
    Q/K/V, kernel, D2H of O and LSE inside the timed region, every step."""
    import torch
    import torch.distributed as dist
    L, N, h, d = q.shape
    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    ho = torch.empty_like(hq).pin_memory()
    hl = torch.empty((L, h, N), dtype=torch.float32).pin_memory()
    p = fm.dense_params(L, N, h, d, fm.BF16 if q.dtype == torch.bfloat16 else fm.F16)
    lib = fm.lib()
    idx = dev.index

    def call():
        st = lib.fmha_fwd_host(C.byref(p), hq.data_ptr(), hk.data_ptr(), hv.data_ptr(), ho.data_ptr(),
                               hl.data_ptr(), idx)
        if st:
            raise RuntimeError(lib.fmha_last_error().decode())

    for _ in range(2):
        call()
    steps = max(3, min(args.steps, 20))
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        call()
    dt = time.perf_counter() - t0
    tt = torch.tensor([dt], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    dt = float(tt.item())
    bi = 3 * hq.numel() * hq.element_size()
    bo = ho.numel() * ho.element_size() + hl.numel() * 4
    # the e2e roofline: host->device copy of the inputs at this box's measured
    # pinned H2D rate (the D2H of O/LSE overlaps it; PCIe is full duplex)
    pcie = measure_h2d_gbps(dev, hq)
    bound_ms = bi / (pcie * 1e9) * 1e3
    return {"value": world * flops(L, N, h, d) * steps / dt / 1e12, "unit": "TFLOP/s",
            "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo, "steps": steps,
            "ms_per_step": dt / steps * 1e3,
            "roofline": {"bound": "pcie_h2d", "h2d_GBps_measured": pcie, "bound_ms": bound_ms,
                         "frac": bound_ms / (dt / steps * 1e3)},
            "api": "fmha_fwd_host (C ABI, pinned host 16-bit buffers; 3-stream H2D/kernel/D2H pipeline)"}


def measure_h2d_gbps(dev, host, reps=5):
    """Pinned host->device copy rate on this box (GB/s): contiguous copies of
    `host` (a pinned buffer the e2e loop already used), timed with CUDA events
    after warm-up."""
    import torch
    dbuf = torch.empty(host.numel() * host.element_size(), dtype=torch.uint8, device=dev)
    src = host.view(-1).view(torch.uint8)
    for _ in range(3):
        dbuf.copy_(src, non_blocking=True)
    torch.cuda.synchronize(dev)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        dbuf.copy_(src, non_blocking=True)
    e.record()
    torch.cuda.synchronize(dev)
    return reps * src.numel() / (s.elapsed_time(e) * 1e-3) / 1e9


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
