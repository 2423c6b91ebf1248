timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 compute-sanitizer --tool memcheck python -c "
import torch, paper_2312_11918_b200 as fm
for N in (8192, 8320):
    q,k,v=(torch.randn(1,N,2,128,device='cuda').half() for _ in range(3)); o=fm.fmha_fwd(q,k,v)
torch.cuda.synchronize(); print('memcheck ok')" 2>&1 | tail -2
timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | cut -c1-200
FMHA_TUNE_PAIR=0 timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | cut -c1-200
timeout 300 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | cut -c1-200
