"""The GPU layer runtime's schedule, emitted in the reference Event schema, passes the
reference's own happens-before checker (seqpar::validate_trace, simhost.cpp:567-657, run
from the reference sources via oracle/_ref/libseqpar_trace.so), and its device
timestamps show the overlap the schedule promises."""
import ctypes as C
import os

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TRACE_LIB = os.path.join(ROOT, "oracle", "_ref", "libseqpar_trace.so")


def ref_validate(jsonl):
    if not os.path.exists(TRACE_LIB):
        pytest.skip("oracle/_ref/libseqpar_trace.so not built (needs /root/reference at build time)")
    L = C.CDLL(TRACE_LIB)
    L.ref_validate_trace_jsonl.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
    buf = C.create_string_buffer(1 << 16)
    n = L.ref_validate_trace_jsonl(jsonl.encode(), buf, len(buf))
    return n, buf.value.decode()


def _inputs(torch, cuda, rows, hq, hkv, seed):
    g = torch.Generator(device=cuda).manual_seed(seed)
    return [torch.randn(rows, w * 128, device=cuda, generator=g).to(torch.bfloat16) for w in (hq, hkv, hkv)]


@pytest.mark.parametrize("hosts,zigzag", [(4, True), (4, False), (2, True)])
def test_sim_layer_trace_passes_reference_validator(cuda, hosts, zigzag):
    import torch

    from paper_2601_21444_b200 import spava

    n_v, n_t, l_a, l_p, hq, hkv = 4000, 64, 64, 128, 4, 2
    cfg = spava.LayerConfig.make(n_v, n_t, hosts, l_a, l_p, hq, hkv, zigzag=zigzag)
    fab = spava.Fabric(cfg, 0)
    hs = [fab.host(h) for h in range(hosts)]
    rows = hs[0].rows
    ins = [_inputs(torch, cuda, rows, hq, hkv, h) for h in range(hosts)]
    outs = [torch.empty(rows, hq * 128, dtype=torch.bfloat16, device=cuda) for _ in range(hosts)]
    for h in hs:
        h.set_trace(True)
    for _layer in range(2):
        fab.sim_layer(hs, [x[0] for x in ins], [x[1] for x in ins], [x[2] for x in ins], outs)
    torch.cuda.synchronize()
    events = spava.trace_events([h.trace_records() for h in hs])
    assert len(events) == hosts * 2 * 19  # per layer: score, 3 rounds x (issue, wait, done), 5 computes
    n, msg = ref_validate(spava.trace_jsonl(events))
    assert n == 0, msg
    # device time is monotone along each host's program order on the single sim stream
    for h in range(hosts):
        ts = [e["t_us"] for e in sorted((e for e in events if e["host"] == h), key=lambda e: e["seq"])]
        assert all(b >= a for a, b in zip(ts, ts[1:]))
    for h in hs:
        h.close()
    fab.close()


@pytest.mark.parametrize("nccl", [False, True])
def test_host_layer_trace_overlap(cuda, nccl):
    """H = 1 (local or NCCL world 1): the trace validates, and the scorer on the side stream
    overlaps the query attention (score ends after query attention begins)."""
    import torch

    from paper_2601_21444_b200 import spava

    n_v, n_t, l_a, l_p, hq, hkv = 16000, 128, 256, 256, 16, 2
    cfg = spava.LayerConfig.make(n_v, n_t, 1, l_a, l_p, hq, hkv)
    fab = (spava.Fabric(cfg, 0, unique_id=spava.nccl_unique_id(), world=1, rank=0) if nccl
           else spava.Fabric(cfg, 0))
    host = fab.host(0)
    q, k, v = _inputs(torch, cuda, host.rows, hq, hkv, 9)
    out = torch.empty(host.rows, hq * 128, dtype=torch.bfloat16, device=cuda)
    host.layer(q, k, v, out)  # warm-up outside the trace
    torch.cuda.synchronize()
    host.set_trace(True)
    for _ in range(3):
        host.layer(q, k, v, out)
    torch.cuda.synchronize()
    events = spava.trace_events([host.trace_records()])
    n, msg = ref_validate(spava.trace_jsonl(events))
    assert n == 0, msg
    for layer in range(3):
        t = {(e["kind"], e["label"]): e["t_us"] for e in events if e["layer"] == layer}
        assert t[("compute_end", "score")] > t[("compute_begin", "query_attn")], t
        assert t[("compute_begin", "stage2")] >= t[("compute_end", "score")]
        assert t[("compute_begin", "merge")] >= t[("compute_end", "stage2")]
    host.close()
    fab.close()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_fabric_trace_passes_reference_validator(cuda, world):
    """Peer fabric (ranks on one GPU, in one process): the per-rank program-order traces of
    two layers, joined by the exchange rounds' Lamport clocks, pass validate_trace."""
    import subprocess
    import sys

    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32", CUDA_MODULE_LOADING="EAGER",
               PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    r = subprocess.run([sys.executable, "-m", "tests.peer_worker", "trace", str(world), "2"], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    body = r.stdout.split("TRACE_JSONL_BEGIN\n", 1)[1].split("TRACE_JSONL_END", 1)[0]
    lines = [x for x in body.splitlines() if x.strip()]
    assert len(lines) == world * 2 * 19
    n, msg = ref_validate("\n".join(lines) + "\n")
    assert n == 0, msg
