"""Dump the layer runtime's schedule trace (reference Event JSONL + device t_us) for a
config: H = 1 through spava_host_layer, H > 1 through the simulated fabric.

    python tools/trace_dump.py C1 1 out.jsonl      (2 layers)
"""
import sys, torch
sys.path.insert(0, '.')
import bench
from paper_2601_21444_b200 import spava

cfg = bench.CONFIGS[sys.argv[1]]
H = int(sys.argv[2])
out_path = sys.argv[3]
g = bench.geometry(cfg, H)
hq, hkv = cfg["hq"], cfg["hkv"]
dev = torch.device("cuda:0")
lc = spava.LayerConfig.make(g["n_v"], g["n_t"], H, g["l_a"], g["l_p"], hq, hkv)
fab = spava.Fabric(lc, 0)
hs = [fab.host(h) for h in range(H)]
rows = hs[0].rows
gen = torch.Generator(device=dev).manual_seed(1)
ins = [[torch.randn(rows, w * 128, device=dev, generator=gen).to(torch.bfloat16) for w in (hq, hkv, hkv)]
       for _ in range(H)]
outs = [torch.empty(rows, hq * 128, dtype=torch.bfloat16, device=dev) for _ in range(H)]


def layer():
    if H == 1:
        hs[0].layer(*ins[0], outs[0])
    else:
        fab.sim_layer(hs, [x[0] for x in ins], [x[1] for x in ins], [x[2] for x in ins], outs)


layer()
torch.cuda.synchronize()
for h in hs:
    h.set_trace(True)
for _ in range(2):
    layer()
torch.cuda.synchronize()
ev = spava.trace_events([h.trace_records() for h in hs])
t0 = min(e["t_us"] for e in ev)
for e in ev:
    e["t_us"] = round(e["t_us"] - t0, 3)
open(out_path, "w").write(spava.trace_jsonl(ev))
print(f"{len(ev)} events -> {out_path}")
