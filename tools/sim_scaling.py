"""Per-host layer time of H Spava hosts simulated on ONE B200 (each host's phases run alone,
exchange through device memory): max over hosts = the per-GPU layer time an H-GPU run sees
before NCCL exchange cost.  Compares zigzag (load-balanced) vs naive pairing.

    python tools/sim_scaling.py [C3] [hosts ...]      -> JSON lines (projection, not a bench value)
"""
import json, sys, time, torch
sys.path.insert(0, '.')
import bench
from paper_2601_21444_b200 import spava

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "C3"
host_list = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
cfg = bench.CONFIGS[cfg_name]
dev = torch.device("cuda:0")
hq, hkv = cfg["hq"], cfg["hkv"]

# dense exact causal attention over the whole sequence on ONE GPU (our kernel), the
# comparator of BASELINE.json's configs
n = cfg["n"]
gen = torch.Generator(device=dev).manual_seed(3)
qd = torch.randn(n, hq * 128, device=dev, generator=gen).to(torch.bfloat16)
kd = torch.randn(n, hkv * 128, device=dev, generator=gen).to(torch.bfloat16)
vd = torch.randn(n, hkv * 128, device=dev, generator=gen).to(torch.bfloat16)
for _ in range(2):
    spava.attention(qd, [dict(k=kd, v=vd, causal=True)], hq, hkv)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    spava.attention(qd, [dict(k=kd, v=vd, causal=True)], hq, hkv)
e1.record()
torch.cuda.synchronize()
dense_ms = e0.elapsed_time(e1) / 3
dense_fl = 2.0 * n * n * hq * 128
print(json.dumps({"config": cfg_name, "n": n, "dense_exact_1gpu_ms": round(dense_ms, 3),
                  "dense_tflops": round(dense_fl / (dense_ms / 1e3) / 1e12, 1),
                  "dense_tokens_per_s": round(n / (dense_ms / 1e3))}), flush=True)
del qd, kd, vd
torch.cuda.empty_cache()
for H in host_list:
    for zz in ((True, False) if H > 1 else (True,)):
        g = bench.geometry(cfg, H, zz)
        lc = spava.LayerConfig.make(g["n_v"], g["n_t"], H, g["l_a"], g["l_p"], hq, hkv, 128, zigzag=zz)
        fab = spava.Fabric(lc, 0)
        hosts = [fab.host(h) for h in range(H)]
        gen = torch.Generator(device=dev).manual_seed(7)
        rows = hosts[0].rows
        qs = [torch.randn(rows, hq * 128, device=dev, generator=gen).to(torch.bfloat16) for _ in range(H)]
        ks = [torch.randn(rows, hkv * 128, device=dev, generator=gen).to(torch.bfloat16) for _ in range(H)]
        vs = [torch.randn(rows, hkv * 128, device=dev, generator=gen).to(torch.bfloat16) for _ in range(H)]
        outs = [torch.empty(rows, hq * 128, dtype=torch.bfloat16, device=dev) for _ in range(H)]
        for _ in range(2):
            fab.sim_layer_timed(hosts, qs, ks, vs, outs)
        # each host is timed early in some run (order rotated, 1 s idle before each run): a
        # sustained-load power cap (~70 ms at C4, SM clock 1965 -> 1590 MHz) would otherwise
        # bill the hosts that happen to run last (tools/sim_clocks.py)
        ms = [float("inf")] * H
        for rep in range(2):
            for rot in range(0, H, max(1, H // 4)):
                order = [(i + rot) % H for i in range(H)]
                torch.cuda.synchronize()
                time.sleep(1.0)
                r = fab.sim_layer_timed([hosts[i] for i in order], [qs[i] for i in order], [ks[i] for i in order],
                                        [vs[i] for i in order], [outs[i] for i in order])
                for pos, i in enumerate(order):
                    ms[i] = min(ms[i], r[pos])
        fl = [bench.attn_flops_host(g, hq, h, zz) for h in range(H)]
        mx = max(ms)
        print(json.dumps({"config": cfg_name, "n": g["n"], "hosts": H, "pairing": "zigzag" if zz else "naive",
                          "ms_per_host": [round(x, 3) for x in ms], "max_ms": round(mx, 3),
                          "max_over_min": round(mx / min(ms), 3),
                          "flops_max_over_min": round(max(fl) / min(fl), 3),
                          "projected_tokens_per_s_excl_comm": round(g["n"] / (mx / 1e3)),
                          "speedup_vs_dense_1gpu": round(dense_ms / mx, 2),
                          "attn_tflops_per_s_on_max_host": round(fl[ms.index(mx)] / (mx / 1e3) / 1e12, 1)}),
              flush=True)
        for h in hosts:
            h.close()
        fab.close()
        del qs, ks, vs, outs
        torch.cuda.empty_cache()
