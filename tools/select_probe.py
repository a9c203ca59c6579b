"""Select + pack timing at C1 (l_b = 16064) and C1 H=8 (l_b = 2008) block sizes -- dev tool."""
import sys, torch
sys.path.insert(0, '.')
from paper_2601_21444_b200 import spava
dev = torch.device('cuda:0')
for l_b, l_p in ((16064, 256), (2008, 256), (128960, 2048)):
    s = torch.rand(l_b, device=dev)
    k = torch.randn(l_b, 256, device=dev).to(torch.bfloat16)
    for _ in range(3):
        spava.select_pack(s, l_p, 0, k, k)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        spava.select_pack(s, l_p, 0, k, k)
    e1.record(); torch.cuda.synchronize()
    print(f"l_b={l_b} l_p={l_p}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per select+pack")
