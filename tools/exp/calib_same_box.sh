# same-box calibration (library kernels are NOT the product): cuDNN SDPA vs this repo, back to back, same shapes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/cudnn_only.py <<'PY'
import torch, torch.nn.functional as F
from torch.nn.attention import sdpa_kernel, SDPBackend
def bench(fn, iters=30):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    best = 1e9
    for rep in range(3):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters): fn()
        e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e) / iters)
    return best
for (L, h, N, d, dt) in [(16, 12, 512, 64, torch.float16), (4, 32, 4096, 64, torch.float16), (4, 16, 4096, 128, torch.float16),
                         (8, 32, 16384, 128, torch.bfloat16), (4, 16, 4096, 128, torch.bfloat16)]:
    fl = 4 * L * h * N * N * d
    q, k, v = (torch.randn(L, h, N, d, device="cuda", dtype=dt) for _ in range(3))
    with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
        ms = bench(lambda: F.scaled_dot_product_attention(q, k, v), 3 if N >= 16384 else 30)
    print(f"cudnn      L={L:2d} h={h:2d} N={N:5d} d={d:3d} {str(dt)[6:]:8s} {ms:.4f} ms {fl/ms/1e9:7.1f} TF", flush=True)
PY
{
for rep in 1 2; do
  timeout 600 python /tmp/cudnn_only.py
  timeout 600 python tools/exp/ab.py ours 0,1,2,3,6
done
} > gpurun_out/calib_same_box.txt 2>&1
