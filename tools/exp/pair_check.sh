timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 compute-sanitizer --tool memcheck python -c "
import torch, paper_2312_11918_b200 as fm
for N in (512, 1000, 384):
    q,k,v=(torch.randn(1,N,2,256,device='cuda').half() for _ in range(3)); o=fm.fmha_fwd(q,k,v)
torch.cuda.synchronize(); print('memcheck ok')" 2>&1 | tail -3
timeout 300 compute-sanitizer --tool synccheck python -c "
import torch, paper_2312_11918_b200 as fm
q,k,v=(torch.randn(1,512,2,256,device='cuda').half() for _ in range(3)); o=fm.fmha_fwd(q,k,v)
torch.cuda.synchronize(); print('synccheck ok')" 2>&1 | tail -3
for i in 1 2; do timeout 300 python bench.py --config c4 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4_pair.json 2>/dev/null; cut -c1-160 gpurun_out/bench_c4_pair.json; done
FMHA_TUNE_PAIR=0 timeout 300 python bench.py --config c4 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | cut -c1-160
timeout 300 ./paper_2312_11918_b200/fmha-b200 sweep --iterations 20 2>&1 | tail -12
