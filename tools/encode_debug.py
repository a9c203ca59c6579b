"""Debug the peer encode gather: enqueue, then poll each rank stream (no blocking sync)."""
import os
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2601_21444_b200 import spava  # noqa: E402

world = int(sys.argv[1])
HQ, HKV = 8, 2
frames, tpf, width = 37, 96, 1024
n_v, n_t = frames * tpf, 24
l_a, l_p = n_v // 64, n_v // 128
cfg = spava.LayerConfig.make(n_v, n_t, world, l_a, l_p, HQ, HKV)
plan = spava.make_plan(n_v, n_t, world, l_a, l_p, True)
counts = spava.frame_partition(frames, world)
rows = [c * tpf for c in counts]
cap = max(rows) * width * 2
fabs = [spava.Fabric.create_peer(cfg, 0, world, r, encode_bytes=cap) for r in range(world)]
spava.Fabric.peer_attach(fabs)
hosts = [f.host(r) for r, f in enumerate(fabs)]
streams = [torch.cuda.Stream() for _ in range(world)]
ev = torch.randn(n_v, width, device="cuda:0").to(torch.bfloat16)
eq = torch.randn(n_t, width, device="cuda:0").to(torch.bfloat16)
outs = [torch.zeros((plan.l_a + 2 * plan.l_b + n_t, width), dtype=torch.bfloat16, device="cuda:0")
        for _ in range(world)]
torch.cuda.synchronize()
print("setup ok", flush=True)
off = 0
for r in range(world):
    t = fabs[r].encode_tensor(rows[r], width)
    print("encode tensor", r, t.shape, t.data_ptr(), flush=True)
    with torch.cuda.stream(streams[r]):
        t.copy_(ev[off:off + rows[r]])
    off += rows[r]
for r in range(world):
    print("poll after copy", r, streams[r].query(), flush=True)
for r in range(world):
    hosts[r].gather_context(rows, eq, outs[r], width * 2, stream=streams[r])
    print("enqueued", r, flush=True)
t0 = time.time()
while time.time() - t0 < 20:
    st = [s.query() for s in streams]
    if all(st):
        break
    time.sleep(0.5)
print("stream done:", [s.query() for s in streams], flush=True)
if all(s.query() for s in streams):
    glob = torch.cat([ev, eq])
    print("equal:", [torch.equal(outs[r], spava.split_rows(plan, r, glob)) for r in range(world)], flush=True)
os._exit(0)
