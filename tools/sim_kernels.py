"""Launch list of ONE simulated host's layer (C1, H hosts) for a per-kernel breakdown under
`ncu --metrics gpu__time_duration.sum` -- dev tool (runs sim_layer once, all hosts)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2601_21444_b200 import spava  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
H = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dev = torch.device("cuda:0")
hq, hkv = cfg["hq"], cfg["hkv"]
g = bench.geometry(cfg, H, True)
lc = spava.LayerConfig.make(g["n_v"], g["n_t"], H, g["l_a"], g["l_p"], hq, hkv, 128)
fab = spava.Fabric(lc, 0)
hosts = [fab.host(h) for h in range(H)]
rows = hosts[0].rows
mk = lambda w: [torch.randn(rows, w * 128, device=dev).to(torch.bfloat16) for _ in range(H)]
qs, ks, vs = mk(hq), mk(hkv), mk(hkv)
outs = [torch.empty(rows, hq * 128, dtype=torch.bfloat16, device=dev) for _ in range(H)]
fab.sim_layer(hosts, qs, ks, vs, outs)
torch.cuda.synchronize()
