import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2601_21444_b200 import spava
from oracle import oracle as O
from tests.util import randn, max_abs
dev = torch.device('cuda:0')
rng = np.random.default_rng(0)
nq, hq, hkv = 128, 1, 1
q = randn(rng, nq, 128); k = randn(rng, 128, 128); v = randn(rng, 128, 128)
td = lambda x: torch.from_numpy(x).to(dev).to(torch.bfloat16)
out, lse = spava.attention(td(q), [dict(k=td(k), v=td(v))], hq, hkv, out_f32=True, want_lse=True)
torch.cuda.synchronize()
ro, rl = O.mha_lse(q, [dict(k=k, v=v)], hq, hkv, 128)
print('visible 1 tile: maxabs', max_abs(out.cpu().numpy(), ro), 'lse', max_abs(lse.cpu().numpy(), rl), flush=True)
o = out.cpu().numpy()
print(o[0,:8], ro[0,:8])
out, lse = spava.attention(td(q), [dict(k=td(k), v=td(v), causal=True)], hq, hkv, out_f32=True, want_lse=True)
torch.cuda.synchronize()
ro, rl = O.mha_lse(q, [dict(k=k, v=v, causal=True)], hq, hkv, 128)
print('causal 1 tile: maxabs', max_abs(out.cpu().numpy(), ro), 'lse', max_abs(lse.cpu().numpy(), rl), flush=True)
nq=700; q = randn(rng, nq, 512); k = randn(rng, 900, 256); v = randn(rng, 900, 256)
out, lse = spava.attention(td(q), [dict(k=td(k), v=td(v)), dict(k=td(k[:700]), v=td(v[:700]), causal=True)], 4, 2, out_f32=True, want_lse=True)
torch.cuda.synchronize()
ro, rl = O.mha_lse(q, [dict(k=k, v=v), dict(k=k[:700], v=v[:700], causal=True)], 4, 2, 128)
print('multi: maxabs', max_abs(out.cpu().numpy(), ro), 'lse', max_abs(lse.cpu().numpy(), rl), flush=True)
