"""Per-CTA fixed cost of the attention kernel: time launches whose CTAs each see T key tiles
(non-causal, one segment) and fit t(T) = waves * (a + b*T) -- dev tool."""
import sys, torch
sys.path.insert(0, '.')
from paper_2601_21444_b200 import spava
dev = torch.device('cuda:0')
hq, hkv, nq = 16, 2, 16064
q = torch.randn(nq, hq * 128, device=dev).to(torch.bfloat16)
k = torch.randn(4096, hkv * 128, device=dev).to(torch.bfloat16)
v = torch.randn(4096, hkv * 128, device=dev).to(torch.bfloat16)
ctas = ((nq + 255) // 256) * hq
waves = ctas / 148
for T in (1, 2, 4, 8, 16, 32):
    kk, vv = k[:128 * T], v[:128 * T]
    fn = lambda: spava.attention(q, [dict(k=kk, v=vv)], hq, hkv)
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    fl = 4.0 * nq * 128 * T * hq * 128
    print(f"T={T:3d} tiles/CTA: {ms*1e3:8.1f} us  per-CTA-wave {ms*1e3/waves:7.2f} us  {fl/ms/1e9:7.0f} TF/s")
