# re-check of the two-CTAs-per-SM single-tile rules for d=128 after the ping-pong kernel's padded-step split
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/shapes.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2312_11918_b200 as fm
tag = sys.argv[1]
for (L, h, N) in [(2, 16, 4096), (8, 16, 1536), (4, 16, 3072), (1, 18, 2048), (2, 36, 1024), (4, 8, 2048), (1, 40, 1536)]:
    q, k, v = (torch.randn(L, N, h, 128, device="cuda", dtype=torch.float16) for _ in range(3))
    for _ in range(5): fm.fmha_fwd(q, k, v)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    best = 1e9
    for rep in range(5):
        s.record()
        for _ in range(20): fm.fmha_fwd(q, k, v)
        e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e) / 20)
    print(f"{tag:8s} L={L} h={h} N={N} {best:.4f} ms {4*L*h*N*N*128/best/1e9:7.1f} TF  {fm.kernel_for(L, N, h, 128, 'f16').split(' ')[0]}", flush=True)
PY
{
for rep in 1 2; do
  timeout 300 python /tmp/shapes.py default
  FMHA_TUNE_TINY2=0 timeout 300 python /tmp/shapes.py tiny2off
done
} > gpurun_out/tiny2_recheck.txt 2>&1
