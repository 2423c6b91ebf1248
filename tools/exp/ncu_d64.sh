cat > gpurun_out/d64run.py <<'PY'
import torch, paper_2312_11918_b200 as fm
q, k, v = (torch.randn(4, 4096, 32, 64, device="cuda").half() for _ in range(3))
for _ in range(5):
    fm.fmha_fwd(q, k, v)
torch.cuda.synchronize()
PY
ncu --set full --clock-control none --import-source on -k regex:fmha_fwd_d64 -s 3 -c 1 -o gpurun_out/prof_t1d64 env PYTHONPATH=. python gpurun_out/d64run.py > gpurun_out/ncu_t1d64.log 2>&1; tail -3 gpurun_out/ncu_t1d64.log
