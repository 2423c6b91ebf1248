"""SM clock / power / throttle reasons while a config runs back to back for ~2 s."""
import os, sys, threading, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2312_11918_b200 as fm
import pynvml
pynvml.nvmlInit()
hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
cfgs = {"c3": (4, 16, 4096, 128, torch.float16), "c5": (8, 32, 16384, 128, torch.bfloat16),
        "c4": (2, 8, 8192, 256, torch.float16), "c2": (16, 12, 512, 64, torch.float16)}
for name in sys.argv[1:] or ["c3"]:
    L, h, N, d, dt = cfgs[name]
    q, k, v = (torch.randn(L, N, h, d, device="cuda", dtype=dt) for _ in range(3))
    o = torch.empty_like(q); lse = torch.empty(L, h, N, device="cuda")
    for _ in range(3): fm.fmha_fwd(q, k, v, o=o, lse=lse)
    torch.cuda.synchronize()
    samples = []; stop = threading.Event()
    def sample():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(hnd) / 1000.0,
                            pynvml.nvmlDeviceGetCurrentClocksEventReasons(hnd)))
            time.sleep(0.01)
    th = threading.Thread(target=sample); th.start()
    n = 0; t0 = time.perf_counter()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    while time.perf_counter() - t0 < 2.0:
        for _ in range(20): fm.fmha_fwd(q, k, v, o=o, lse=lse)
        n += 20
        torch.cuda.synchronize()
    b.record(); torch.cuda.synchronize()
    stop.set(); th.join()
    ms = a.elapsed_time(b) / n
    s = sorted(x[0] for x in samples[len(samples) // 4:])
    p = sorted(x[1] for x in samples[len(samples) // 4:])
    caps = sum(1 for x in samples if x[2] & pynvml.nvmlClocksEventReasonSwPowerCap)
    print(f"{name}: {ms:.4f} ms/launch {4*L*h*N*N*d/ms/1e9:.1f} TF | sm clock median {s[len(s)//2]} MHz "
          f"(min {s[0]}, max {s[-1]}) | power median {p[len(p)//2]:.0f} W max {p[-1]:.0f} W | "
          f"sw_power_cap in {caps}/{len(samples)} samples", flush=True)
