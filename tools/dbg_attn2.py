"""Dev: attention error vs the C oracle across pairing / segment-count configurations."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2601_21444_b200 import spava
from oracle import oracle as O
from tests.util import randn, max_abs
dev = torch.device('cuda:0')
td = lambda x: torch.from_numpy(x).to(dev).to(torch.bfloat16)
cases = [
    ("pair 1seg 700", 128, 8, 2, [(700, False)]),
    ("nopair(g1) 1seg 700", 128, 2, 2, [(700, False)]),
    ("256 rows 1seg 700", 256, 2, 1, [(700, False)]),
    ("pair 2seg 33+700", 128, 8, 2, [(33, False), (700, False)]),
    ("pair 1seg 64", 128, 8, 2, [(64, False)]),
    ("pair 1seg 128", 128, 8, 2, [(128, False)]),
    ("pair 1seg 192", 128, 8, 2, [(192, False)]),
    ("pair 1seg 256", 128, 8, 2, [(256, False)]),
    ("pair 1seg 320", 128, 8, 2, [(320, False)]),
    ("pair causal 128", 128, 8, 2, [(128, True)]),
    ("nopair 1seg 320", 128, 2, 2, [(320, False)]),
]
for name, nq, hq, hkv, segs in cases:
    rng = np.random.default_rng(1)
    q = randn(rng, nq, hq * 128)
    sn, sd = [], []
    for rows, causal in segs:
        k = randn(rng, rows, hkv * 128); v = randn(rng, rows, hkv * 128)
        sn.append(dict(k=k, v=v, causal=causal)); sd.append(dict(k=td(k), v=td(v), causal=causal))
    out, lse = spava.attention(td(q), sd, hq, hkv, out_f32=True, want_lse=True)
    torch.cuda.synchronize()
    ro, rl = O.mha_lse(q, sn, hq, hkv, 128, allow_invalid=True)
    o = out.cpu().numpy()
    err_h = [max_abs(o[:, h*128:(h+1)*128], ro[:, h*128:(h+1)*128]) for h in range(hq)]
    print(f"{name:24s} out maxabs per head {np.round(err_h, 3)} lse {max_abs(lse.cpu().numpy(), rl):.2e}", flush=True)
