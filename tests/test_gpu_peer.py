"""GPU tests of the peer fabric (NVLink P2P exchange without a collective library).

The pass rounds are stored by the select gather kernel and the qpartial round by the
query split-merge kernel straight into every peer's exchange slot; epoch flags (stream
memory operations) order them.  Parity bar: every rank's layer output and passing
indices bit-identical to the local fabric (the reference's in-process GatherFabric
order, simhost.cpp:61-166) over several consecutive layers, and the first layer's against
the C oracle of the whole layer on the same global inputs (indices exact, outputs within
the bf16 bar) -- every rank checked against the reference algorithm directly.

Only one GPU is available, so the ranks share cuda:0: either WORLD fabrics in one
process on WORLD streams, or WORLD real processes that map each other's exchange
buffers through CUDA IPC (the multi-GPU code path, minus NVLink itself).  Each runs in a
subprocess under a timeout.
"""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _env():
    env = dict(os.environ)
    env["CUDA_DEVICE_MAX_CONNECTIONS"] = "32"  # every rank stream its own hardware queue
    # one thread enqueues every rank: a lazily loaded kernel's first launch waits for the
    # device, whose streams may wait on flags of ranks not yet enqueued -> load eagerly
    env["CUDA_MODULE_LOADING"] = "EAGER"
    env["PYTHONPATH"] = ROOT + os.pathsep + env.get("PYTHONPATH", "")
    return env


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,zigzag,fused", [(2, True, "1"), (4, True, "1"), (3, False, "1"), (2, True, "0"),
                                                (4, True, "0")])
def test_peer_fabric_inprocess_matches_local(cuda, world, zigzag, fused):
    """fused=1 (default): the final query merge runs as trailing CTAs of the merged stage
    launch, waiting for the peers' qpartial flags in-kernel (receive-side merge); fused=0:
    separate merge launch after a stream wait.  Both bit-identical to the local fabric."""
    env = _env()
    env["PEER_ZIGZAG"] = "1" if zigzag else "0"
    env["SPAVA_FUSED_MERGE"] = fused
    r = subprocess.run([sys.executable, "-m", "tests.peer_worker", "inproc", str(world), "3"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0 and "PEER_OK all 3" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


def test_peer_fabric_two_processes_ipc_matches_local(cuda):
    world, port = 2, _free_port()
    procs = [subprocess.Popen([sys.executable, "-m", "tests.peer_worker", "rank", str(r), str(world),
                               "3", str(port)], cwd=ROOT, env=_env(), stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for r in range(world)]
    outs = []
    try:
        for p in procs:
            outs.append(p.communicate(timeout=300))
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for r, (p, (o, e)) in enumerate(zip(procs, outs)):
        assert p.returncode == 0 and f"PEER_OK {r} 3" in o, o[-2000:] + e[-4000:]
