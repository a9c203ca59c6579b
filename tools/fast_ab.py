"""Dev A/B: fast-mode (score_mode=1) C1 layer with the scorer fused into the query launch (N1)
vs the standalone three-launch scorer; also the H=8 C1 simulated layer (per-host time)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2601_21444_b200 import spava
dev = torch.device('cuda:0')
L = spava.lib()
n, n_t, hq, hkv = 32768, 128, 16, 2
l_a, l_p = n // 64, n // 128
n_v = n - n_t
def layer_ms(fused, reps=20):
    spava._check(L.spava_debug_fused_score(fused))
    cfg = spava.LayerConfig.make(n_v, n_t, 1, l_a, l_p, hq, hkv, score_mode=1)
    fab = spava.Fabric(cfg, 0); H = fab.host(0)
    g = torch.Generator(device=dev).manual_seed(1)
    q, k, v = (torch.randn(H.rows, w * 128, device=dev, generator=g).to(torch.bfloat16) for w in (hq, hkv, hkv))
    out = torch.zeros(H.rows, hq * 128, dtype=torch.bfloat16, device=dev); sel = torch.zeros(2, l_p, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ts = []
    for i in range(reps + 3):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); H.layer(q, k, v, out, sel); e1.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(e0.elapsed_time(e1))
    s = sel.clone(); H.close(); fab.close()
    return sum(ts) / len(ts), s
def sim8_ms(fused):
    spava._check(L.spava_debug_fused_score(fused))
    hosts = 8
    cfg = spava.LayerConfig.make(n_v, n_t, hosts, l_a, l_p, hq, hkv, score_mode=1)
    fab = spava.Fabric(cfg, 0); hs = [fab.host(h) for h in range(hosts)]
    g = torch.Generator(device=dev).manual_seed(2)
    ins = [[torch.randn(H.rows, w * 128, device=dev, generator=g).to(torch.bfloat16) for w in (hq, hkv, hkv)] for H in hs]
    outs = [torch.zeros(H.rows, hq * 128, dtype=torch.bfloat16, device=dev) for H in hs]
    sels = [torch.zeros(2, l_p, dtype=torch.int32, device=dev) for H in hs]
    best = None
    for _ in range(5):
        ms = fab.sim_layer_timed(hs, [x[0] for x in ins], [x[1] for x in ins], [x[2] for x in ins], outs, sels)
        best = ms if best is None else [min(a, b) for a, b in zip(best, ms)]
    for H in hs: H.close()
    fab.close()
    return max(best)
for rep in range(2):
    for fused in (0, 1):
        ms, s = layer_ms(fused)
        print(f"C1 H=1 fast-mode layer, fused={fused}: {ms:.4f} ms  | C1 H=8 sim per-host max: {sim8_ms(fused):.4f} ms")
spava._check(L.spava_debug_fused_score(-1))
