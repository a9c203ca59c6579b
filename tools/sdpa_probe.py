"""Dense causal 32K through torch SDPA (cuDNN) -- dev probe for ncu (launch config / pipes)."""
import torch
dev = torch.device("cuda:0")
n, hq, hkv = 32768, 16, 2
q = torch.randn(1, hq, n, 128, device=dev, dtype=torch.bfloat16)
k = torch.randn(1, hkv, n, 128, device=dev, dtype=torch.bfloat16).repeat_interleave(hq // hkv, 1)
v = torch.randn(1, hkv, n, 128, device=dev, dtype=torch.bfloat16).repeat_interleave(hq // hkv, 1)
from torch.nn.attention import sdpa_kernel, SDPBackend
with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
    for _ in range(3):
        torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
torch.cuda.synchronize()
