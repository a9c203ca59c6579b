"""Step time of the C1 layer: direct launches vs CUDA-graph replay (dev)."""
import sys, torch
sys.path.insert(0, '.')
import bench
from paper_2601_21444_b200 import spava
cfg = bench.CONFIGS["C1"]
g = bench.geometry(cfg, 1)
hq, hkv = cfg["hq"], cfg["hkv"]
dev = torch.device("cuda:0")
lc = spava.LayerConfig.make(g["n_v"], g["n_t"], 1, g["l_a"], g["l_p"], hq, hkv)
fab = spava.Fabric(lc, 0)
host = fab.host(0)
rows = host.rows
q = torch.randn(rows, hq * 128, device=dev).to(torch.bfloat16)
k = torch.randn(rows, hkv * 128, device=dev).to(torch.bfloat16)
v = torch.randn(rows, hkv * 128, device=dev).to(torch.bfloat16)
out = torch.empty(rows, hq * 128, dtype=torch.bfloat16, device=dev)
sel = torch.empty(2, g["l_p"], dtype=torch.int32, device=dev)
s = torch.cuda.Stream()
host.capture_layer(q, k, v, out, sel, stream=s)
def t(fn, n=30):
    for _ in range(5): fn()
    s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(n): fn()
    e1.record(s)
    s.synchronize()
    return e0.elapsed_time(e1) / n
print("direct %.4f ms, graph %.4f ms (back-to-back steps, no L2 flush)" % (
    t(lambda: host.layer(q, k, v, out, sel, s)), t(lambda: host.replay_layer(s))))
