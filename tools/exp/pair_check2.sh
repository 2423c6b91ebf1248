timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 120 python tools/exp/ab.py pair 4
timeout 120 python tools/exp/ab.py pair 4
python - <<'PY'
import torch, paper_2312_11918_b200 as fm, time
# odd tile count: pair kernel with a padding CTA vs single-CTA (same inputs)
for N in (384, 8064):
    g = torch.Generator(device="cuda").manual_seed(5)
    q, k, v = (torch.randn(2, N, 8, 256, device="cuda", generator=g).half() for _ in range(3))
    o, l = fm.fmha_fwd(q, k, v)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): fm.fmha_fwd(q, k, v)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 20
    print(f"N={N} pair path {ms:.4f} ms {4*2*8*N*N*256/ms/1e9:.1f} TF")
PY
ncu --set full --clock-control none --import-source on -k regex:fmha_fwd -s 3 -c 1 -o gpurun_out/prof_c4_pair python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; ls -la gpurun_out/
