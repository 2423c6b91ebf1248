for pair in 1 0; do echo "== pair=$pair"; FMHA_TUNE_PAIR=$pair timeout 300 compute-sanitizer --tool synccheck python -c "
import torch, paper_2312_11918_b200 as fm
q,k,v=(torch.randn(1,512,2,256,device='cuda').half() for _ in range(3)); o=fm.fmha_fwd(q,k,v)
torch.cuda.synchronize(); print('synccheck ok')" 2>&1 | grep -v "^=========     " | head -30; done
