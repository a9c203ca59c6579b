"""world_size-2 gloo tests of the multi-host (N>1) host logic on CPU.

The GPU runtime's exchange is an in-place allgather of per-host slots (pass1: lo
blocks, pass2: hi blocks, qpartial) and block v then reads the slot ranges
spava.passing_ranges(v).  Here two real processes run that protocol over gloo with
the C oracle's selections as payload and check, on every rank, that the assembled
passing set equals assemble_passing (approx.cpp:104-132) of the single-process
reference schedule, and that the query partials merge (host order) to the same
result as the oracle layer.  Also covers the NCCL unique-id broadcast used by bench.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from tests.util import randn

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, zigzag, errq):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        from paper_2601_21444_b200 import spava

        H = WORLD
        n_v, n_t, l_a, l_p, hq, hkv, dh = 230, 6, 10, 12, 2, 1, 16
        plan = spava.make_plan(n_v, n_t, H, l_a, l_p, zigzag)
        l_b = plan.l_b
        rng = np.random.default_rng(77)  # same global inputs on every rank
        n_pad = l_a + 2 * H * l_b + n_t
        Q, K, V = randn(rng, n_pad, hq * dh), randn(rng, n_pad, hkv * dh), randn(rng, n_pad, hkv * dh)
        ref = O.spava_layer(Q, K, V, n_v, n_t, H, l_a, l_p, hq, hkv, dh, zigzag=zigzag)
        qoff = spava.query_offset(plan)
        lo, hi = spava.virtual_pair(plan, rank)
        # this rank's selections (what its select+pack kernel would produce)
        mine = []
        for v in (lo, hi):
            o = spava.block_offset(plan, v)
            pad = spava.pad_mask(plan, v)
            s = O.score_block(Q[qoff:], K[o:o + l_b], hq, hkv, dh, pad)
            mine.append(O.select_essential(s, l_p, o))
        # in-place allgather of fixed-size slots, two rounds
        rounds = []
        for r in range(2):
            slot = torch.full((l_p,), -1, dtype=torch.int32)
            slot[:len(mine[r])] = torch.from_numpy(mine[r])
            out = torch.empty(WORLD * l_p, dtype=torch.int32)
            dist.all_gather_into_tensor(out, slot)
            rounds.append(out.view(WORLD, l_p).numpy())
        for v in (lo, hi):
            (a0, a1), (b0, b1) = spava.passing_ranges(plan, v)
            got = np.concatenate([rounds[0][a0:a1].ravel(), rounds[1][b0:b1].ravel()])
            want = np.concatenate([ref["sel"][s] for s in range(v)]) if v else np.zeros(0, np.int32)
            assert sorted(got.tolist()) == sorted(want.tolist()), (rank, v)
            # within each round the slots are contiguous and in source order of that round
            assert np.array_equal(got[:(a1 - a0) * l_p],
                                  np.concatenate([ref["sel"][spava.virtual_pair(plan, s)[0]]
                                                  for s in range(a0, a1)]) if a1 > a0 else np.zeros(0))
        # qpartial round + host-order merge on every rank
        po = torch.from_numpy(ref["qpart_out"][rank].copy())
        pl = torch.from_numpy(ref["qpart_lse"][rank].copy())
        go = [torch.empty_like(po) for _ in range(WORLD)]
        gl = [torch.empty_like(pl) for _ in range(WORLD)]
        dist.all_gather(go, po)
        dist.all_gather(gl, pl)
        merged = O.mha_merge([t.numpy() for t in go], [t.numpy() for t in gl], hq, dh)
        assert np.array_equal(merged, ref["query"])
        # bench.py's NCCL unique-id broadcast path (id content is opaque bytes)
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        assert obj[0] == bytes(range(128))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced through the queue
        import traceback

        errq.put(f"rank {rank}: {e}\n{traceback.format_exc()}")
        raise


@pytest.mark.parametrize("zigzag", [True, False])
def test_two_host_exchange_gloo(zigzag):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, zigzag, errq)) for r in range(WORLD)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
