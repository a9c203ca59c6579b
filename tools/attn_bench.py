"""Dev tool: time the attention kernel on C1 block-hi and dense-causal shapes."""
import os, sys, torch
sys.path.insert(0, '.')
from paper_2601_21444_b200 import spava
dev = torch.device('cuda:0')
hq, hkv = 16, 2
def t(fn, reps=10):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
lb, la, lp = 16064, 512, 256
q = torch.randn(lb, hq*128, device=dev).to(torch.bfloat16)
k = torch.randn(lb, hkv*128, device=dev).to(torch.bfloat16)
v = torch.randn(lb, hkv*128, device=dev).to(torch.bfloat16)
ka, va = k[:la], v[:la]
kp, vp = k[la:la+lp], v[la:la+lp]
segs = [dict(k=ka, v=va), dict(k=kp, v=vp), dict(k=k, v=v, causal=True)]
fl = (4*lb*(la+lp) + 2*lb*lb) * 128 * hq
ms = t(lambda: spava.attention(q, segs, hq, hkv))
n = 32768
qd = torch.randn(n, hq*128, device=dev).to(torch.bfloat16)
kd = torch.randn(n, hkv*128, device=dev).to(torch.bfloat16)
vd = torch.randn(n, hkv*128, device=dev).to(torch.bfloat16)
ms2 = t(lambda: spava.attention(qd, [dict(k=kd, v=vd, causal=True)], hq, hkv), 5)
fl2 = 2.0*n*n*hq*128
# fully visible (non-causal) 16K x 16K
ms3 = t(lambda: spava.attention(q, [dict(k=k, v=v)], hq, hkv), 5)
fl3 = 4.0*lb*lb*hq*128
print(f"variant {os.environ.get('SPAVA_ATTN_VARIANT','0')}: block {ms:.3f} ms {fl/ms/1e9:.0f} TF/s | dense causal {ms2:.3f} ms {fl2/ms2/1e9:.0f} TF/s | full {ms3:.3f} ms {fl3/ms3/1e9:.0f} TF/s")
if os.environ.get('SPAVA_ATTN_VARIANT') in ('1', '16'):
    import ctypes as C
    L = spava.lib()
    buf = (C.c_uint64 * 16)()
    L.spava_debug_attn_prof(buf)  # reset
    spava.attention(q, segs, hq, hkv); torch.cuda.synchronize()
    L.spava_debug_attn_prof(buf)
    names = ['mma_wait_k','mma_wait_v','mma_wait_p','mma_total','sm_wait_s','sm_body','sm_tiles','rescales']
    d = {n: buf[i] for i, n in enumerate(names)}
    tiles = d['sm_tiles']
    print({k: v for k, v in d.items()})
    print('per softmax warp-tile: wait_s %.0f  body %.0f cycles; mma per tile-pair total %.0f, wait_p %.0f wait_k %.0f wait_v %.0f' % (
        d['sm_wait_s']/tiles, d['sm_body']/tiles, d['mma_total']/(tiles/8), d['mma_wait_p']/(tiles/8), d['mma_wait_k']/(tiles/8), d['mma_wait_v']/(tiles/8)))
    print('softmax phases per warp-tile: ld %.0f  ld+mask+max %.0f  exp+pack+st %.0f (of which mid-tile wait_st/arrive %.0f)  tail wait_st/arrive %.0f' % (buf[9]/tiles, buf[8]/tiles, buf[10]/tiles, buf[11]/tiles, buf[12]/tiles))
