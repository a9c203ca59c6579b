"""GPU tests of the frame-parallel encode gather fused with split_context (
simhost.cpp:280-302, partition.cpp:30-85).

Each host holds only its frame_partition share of E_v; spava_gather_split_rows reads host
h's [anchor | lo | hi | query] rows straight from the owners' shares.  Bar: bit-identical
to split_context of the concatenated E_v (spava_split_rows, itself checked against the
reference's split_context in test_gpu_fullsize / the CPU oracle tests).
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("hosts,frames,tpf,zigzag", [(1, 5, 64, True), (2, 9, 100, True),
                                                     (4, 37, 96, False), (8, 64, 40, True),
                                                     (3, 7, 33, True)])
def test_gather_split_matches_split_context(cuda, hosts, frames, tpf, zigzag):
    import torch

    from paper_2601_21444_b200 import spava

    width, n_t = 768, 17
    n_v = frames * tpf
    l_a, l_p = max(n_v // 64, 1), n_v // 128
    plan = spava.make_plan(n_v, n_t, hosts, l_a, l_p, zigzag)
    counts = spava.frame_partition(frames, hosts)
    rows = [c * tpf for c in counts]
    g = torch.Generator(device=cuda).manual_seed(frames)
    ev = torch.randn(n_v, width, device=cuda, generator=g).to(torch.bfloat16)
    eq = torch.randn(n_t, width, device=cuda, generator=g).to(torch.bfloat16)
    parts, off = [], 0
    for r in rows:  # each host's share in its own allocation
        parts.append(ev[off:off + r].clone() if r else None)
        off += r
    glob = torch.cat([ev, eq])
    for h in range(hosts):
        got = spava.gather_split_rows(plan, h, parts, rows, eq)
        torch.cuda.synchronize()
        assert torch.equal(got, spava.split_rows(plan, h, glob)), h


def test_gather_split_rejects_bad_parts(cuda):
    import torch

    from paper_2601_21444_b200 import spava

    plan = spava.make_plan(1000, 8, 2, 16, 8)
    ev = torch.zeros(1000, 64, dtype=torch.bfloat16, device=cuda)
    eq = torch.zeros(8, 64, dtype=torch.bfloat16, device=cuda)
    with pytest.raises(spava.SpavaError):  # shares must sum to n_v
        spava.gather_split_rows(plan, 0, [ev[:500], ev[500:]], [500, 499], eq)


def test_peer_encode_gather_inprocess(cuda):
    # EAGER: one thread enqueues every rank, and a lazily loaded kernel's first launch
    # waits for the device, whose streams wait on flags of ranks not yet enqueued
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32", CUDA_MODULE_LOADING="EAGER",
               PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, "-m", "tests.peer_worker", "encode", "4", "3"], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0 and "PEER_OK encode 3" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
