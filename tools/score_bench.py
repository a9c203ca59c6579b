"""Time the exact scorer at C1 shapes (softmax vs raw) -- dev tool."""
import sys, torch
sys.path.insert(0, '.')
from paper_2601_21444_b200 import spava
dev = torch.device('cuda:0')
n_t, l_b, hq, hkv = 128, 16064, 16, 2
q = torch.randn(n_t, hq * 128, device=dev).to(torch.bfloat16)
k = torch.randn(l_b, hkv * 128, device=dev).to(torch.bfloat16)
for sm in (True, False):
    for _ in range(3):
        spava.score_block(q, k, hq, hkv, 128, softmax=sm)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        spava.score_block(q, k, hq, hkv, 128, softmax=sm)
    e1.record(); torch.cuda.synchronize()
    print('softmax' if sm else 'raw', e0.elapsed_time(e1) / 10, 'ms per block')
