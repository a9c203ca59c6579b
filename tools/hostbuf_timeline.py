"""Timeline of one C1 host-buffer layer (SPAVA_HOSTBUF_TIMELINE=1 prints it) -- dev tool."""
import os
import sys

os.environ["SPAVA_HOSTBUF_TIMELINE"] = "1"
sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2601_21444_b200 import spava  # noqa: E402

n, n_t, hq, hkv = 32768, 128, 16, 2
cfg = spava.LayerConfig.make(n - n_t, n_t, 1, n // 64, n // 128, hq, hkv)
fab = spava.Fabric(cfg, 0)
h = fab.host(0)
rows = h.rows
dev = torch.device("cuda:0")
ins = [torch.randn(rows, w * 128, device=dev).to(torch.bfloat16) for w in (hq, hkv, hkv)]
hins = [x.cpu().pin_memory() for x in ins]
out = torch.empty(rows, hq * 128, dtype=torch.bfloat16, device=dev)
oh = torch.empty(out.shape, dtype=out.dtype).pin_memory()
for it in range(3):
    if it == 2:
        print("---- step", it, file=sys.stderr, flush=True)
    h.layer_hostbuf(*hins, oh, *[torch.empty_like(x) for x in ins], out)
    torch.cuda.synchronize()
