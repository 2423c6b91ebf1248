import torch
import torch.nn.functional as F
from torch.nn.attention import sdpa_kernel, SDPBackend
L, h, N, d = 4, 16, 4096, 128
q, k, v = (torch.randn(L, h, N, d, device="cuda", dtype=torch.float16) for _ in range(3))
with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
    for _ in range(5):
        F.scaled_dot_product_attention(q, k, v)
torch.cuda.synchronize()
