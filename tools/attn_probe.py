"""Dev probe: softmax body cycles with one Q tile per CTA (no ping-pong partner) vs two."""
import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_2601_21444_b200 import spava
dev = torch.device('cuda:0')
L = spava.lib()
buf = (C.c_uint64 * 16)()
names = ['mma_wait_k', 'mma_wait_v', 'mma_wait_p', 'mma_total', 'sm_wait_s', 'sm_body', 'sm_tiles', 'rescales']
for nq, hq, nk in ((128, 148, 16384), (256, 148, 16384)):
    q = torch.randn(nq, hq * 128, device=dev).to(torch.bfloat16)
    k = torch.randn(nk, hq * 128, device=dev).to(torch.bfloat16)
    v = torch.randn(nk, hq * 128, device=dev).to(torch.bfloat16)
    for _ in range(2):
        spava.attention(q, [dict(k=k, v=v)], hq, hq)
    torch.cuda.synchronize()
    L.spava_debug_attn_prof(buf)
    spava.attention(q, [dict(k=k, v=v)], hq, hq)
    torch.cuda.synchronize()
    L.spava_debug_attn_prof(buf)
    d = {n: buf[i] for i, n in enumerate(names)}
    t = d['sm_tiles']
    wg = 4 if nq == 128 else 8
    print(f"nq={nq}: softmax warp-tile wait_s {d['sm_wait_s']/t:.0f} body {d['sm_body']/t:.0f}; "
          f"mma per kv step {d['mma_total']/(t/wg):.0f} wait_p {d['mma_wait_p']/(t/wg):.0f}; "
          f"ld {buf[9]/t:.0f} ld+spec {buf[8]/t:.0f} tail {buf[12]/t:.0f}")
