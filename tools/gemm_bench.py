"""Dev: tcgen05 GEMM (gemm.cu) vs torch.matmul (cuBLAS) on the decoder layer's shapes."""
import sys, torch
sys.path.insert(0, '.')
from paper_2601_21444_b200 import spava
dev = torch.device('cuda:0')
def t(fn, reps=10):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
M = 32768
for name, N, K in (("qkv", 2560, 2048), ("wo", 2048, 2048), ("w1", 11008, 2048), ("w2", 2048, 11008), ("sq8k", 8192, 8192)):
    m = 8192 if name == "sq8k" else M
    a = torch.randn(m, K, device=dev).to(torch.bfloat16)
    b = torch.randn(K, N, device=dev).to(torch.bfloat16)
    out = torch.empty(m, N, device=dev, dtype=torch.bfloat16)
    ms = t(lambda: spava.gemm(a, b, out))
    ms2 = t(lambda: torch.matmul(a, b, out=out))
    fl = 2.0 * m * N * K
    print(f"{name:5s} M={m} N={N} K={K}: ours {ms:.3f} ms {fl/ms/1e9:.0f} TF/s | cuBLAS {ms2:.3f} ms {fl/ms2/1e9:.0f} TF/s")
