"""Time the exact and fast scorers at C1 shapes (one block) -- dev tool."""
import sys, torch
sys.path.insert(0, '.')
from paper_2601_21444_b200 import spava
dev = torch.device('cuda:0')
n_t, l_b, hq, hkv = 128, 16064, 16, 2
q = torch.randn(n_t, hq * 128, device=dev).to(torch.bfloat16)
k = torch.randn(l_b, hkv * 128, device=dev).to(torch.bfloat16)
for name, fn in (("exact softmax", lambda: spava.score_block(q, k, hq, hkv, 128, softmax=True)),
                 ("exact raw", lambda: spava.score_block(q, k, hq, hkv, 128, softmax=False)),
                 ("fast", lambda: spava.score_block_fast(q, k, hq, hkv, 128))):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record(); torch.cuda.synchronize()
    print(name, e0.elapsed_time(e1) / 10, 'ms per block')
