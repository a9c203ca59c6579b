"""Peer-fabric (NVLink P2P) worker for tests/test_gpu_peer.py -- run as a subprocess so
CUDA_DEVICE_MAX_CONNECTIONS and the process layout are under the test's control.

  python -m tests.peer_worker inproc WORLD LAYERS   one process, WORLD peer fabrics on
                                                    cuda:0, each rank on its own stream
  python -m tests.peer_worker rank RANK WORLD LAYERS PORT
                                                    one rank of a WORLD-process job on
                                                    cuda:0 (IPC handles over gloo)

Every rank runs LAYERS consecutive layers (different inputs each, so the epoch flags and
the slot-release protocol are exercised) and checks its outputs and passing indices
bit-identical against the local fabric (spava_sim_layer) on the same inputs, and layer 0
against the C oracle (indices exact, outputs within the bf16 bar).
Prints one line "PEER_OK <rank|all> <layers>" on success.
"""
import os
import sys

import numpy as np
import torch

from oracle import oracle as O
from paper_2601_21444_b200 import spava
from tests.util import ATOL_BF16_OUT, RTOL_L2_BF16, host_local, max_abs, randn, rel_l2

N_V, N_T, L_A, L_P, HQ, HKV = 5000, 64, 64, 160, 8, 2
ZIGZAG = os.environ.get("PEER_ZIGZAG", "1") == "1"


def global_inputs(world, layer):
    """One layer's global padded Q/K/V (bf16-valued fp32, the same on every rank)."""
    plan = spava.make_plan(N_V, N_T, world, L_A, L_P, ZIGZAG)
    n_pad = L_A + 2 * world * plan.l_b + N_T
    rng = np.random.default_rng(1000 + layer)
    return plan, randn(rng, n_pad, HQ * 128), randn(rng, n_pad, HKV * 128), randn(rng, n_pad, HKV * 128)


def inputs(world, layer):
    """Per-host [anchor | lo | hi | query] rows of one consistent global sequence (the
    reference's split_context of the same Q/K/V), on cuda:0."""
    cfg = spava.LayerConfig.make(N_V, N_T, world, L_A, L_P, HQ, HKV, zigzag=ZIGZAG)
    plan, Q, K, V = global_inputs(world, layer)
    rows = L_A + 2 * plan.l_b + N_T
    qoff = spava.query_offset(plan)
    qs, ks, vs = [], [], []
    for h in range(world):
        lo, hi = spava.virtual_pair(plan, h)
        for X, lst in ((Q, qs), (K, ks), (V, vs)):
            lst.append(torch.from_numpy(host_local(X, L_A, plan.l_b, lo, hi, qoff, N_T)).to("cuda:0")
                       .to(torch.bfloat16))
    return cfg, rows, qs, ks, vs


def oracle_layer(world, layer):
    """C oracle (oracle/spava_oracle.c, the reference's run_host restated) of one layer:
    per host the passing indices of (lo, hi) and the expected [anchor | lo | hi | query]
    output rows.  Test infrastructure only (the checker)."""
    plan, Q, K, V = global_inputs(world, layer)
    want = O.spava_layer(Q, K, V, N_V, N_T, world, L_A, L_P, HQ, HKV, 128, zigzag=ZIGZAG)
    res = []
    for h in range(world):
        lo, hi = spava.virtual_pair(plan, h)
        out = np.concatenate([want["anchor"], want["blocks"][lo], want["blocks"][hi], want["query"]])
        res.append((np.stack([want["sel"][lo], want["sel"][hi]]), out))
    return res


def reference(world, layers):
    """Local fabric (the in-process GatherFabric) outputs, per layer and host; layer 0 of
    the local fabric is also checked against the C oracle (indices exact, outputs within
    the bf16 bar), so the peer ranks' bit-identity to it is parity with the reference."""
    res = []
    for layer in range(layers):
        cfg, rows, qs, ks, vs = inputs(world, layer)
        fab = spava.Fabric(cfg, 0)
        hs = [fab.host(h) for h in range(world)]
        outs = [torch.zeros(rows, HQ * 128, dtype=torch.bfloat16, device="cuda:0") for _ in hs]
        sels = [torch.zeros(2, L_P, dtype=torch.int32, device="cuda:0") for _ in hs]
        fab.sim_layer(hs, qs, ks, vs, outs, sels)
        torch.cuda.synchronize()
        assert all(h.status() == 0 for h in hs)
        res.append((outs, sels))
        for h in hs:
            h.close()
        fab.close()
    ORACLE.extend(oracle_layer(world, 0))
    return res


ORACLE = []  # layer 0 per host: (indices [2, l_p], output rows) from the C oracle


def check(ref, layer, rank, out, sel):
    want_out, want_sel = ref[layer][0][rank], ref[layer][1][rank]
    if not torch.equal(sel, want_sel):
        raise AssertionError(f"layer {layer} rank {rank}: passing indices differ")
    if not torch.equal(out, want_out):
        d = (out.float() - want_out.float()).abs().max().item()
        raise AssertionError(f"layer {layer} rank {rank}: output differs (max {d})")
    if layer == 0 and ORACLE:  # the peer rank against the reference algorithm directly
        o_sel, o_out = ORACLE[rank]
        if not np.array_equal(sel.cpu().numpy(), o_sel):
            raise AssertionError(f"rank {rank}: passing indices differ from the oracle")
        got = out.float().cpu().numpy()
        if max_abs(got, o_out) >= ATOL_BF16_OUT or rel_l2(got, o_out) >= RTOL_L2_BF16:
            raise AssertionError(f"rank {rank}: output vs oracle max {max_abs(got, o_out)} "
                                 f"rel-L2 {rel_l2(got, o_out)}")


def inproc(world, layers):
    ref = reference(world, layers)
    cfg, rows, _, _, _ = inputs(world, 0)
    fabs = [spava.Fabric.create_peer(cfg, 0, world, r) for r in range(world)]
    spava.Fabric.peer_attach(fabs)
    hosts = [f.host(r) for r, f in enumerate(fabs)]
    streams = [torch.cuda.Stream() for _ in range(world)]
    for layer in range(layers):
        _, _, qs, ks, vs = inputs(world, layer)
        torch.cuda.synchronize()
        outs = [torch.zeros(rows, HQ * 128, dtype=torch.bfloat16, device="cuda:0") for _ in hosts]
        sels = [torch.zeros(2, L_P, dtype=torch.int32, device="cuda:0") for _ in hosts]
        # enqueue every rank before any waits can be satisfied: the flag waits are in-stream
        hostbuf = layer == layers - 1  # last layer through the host-buffer entry point
        staged = []
        for r in range(world):
            if hostbuf:
                hb = [t.cpu().pin_memory() for t in (qs[r], ks[r], vs[r])]
                oh = torch.empty(outs[r].shape, dtype=outs[r].dtype).pin_memory()
                sh = torch.empty(sels[r].shape, dtype=sels[r].dtype).pin_memory()
                dq, dk, dv = (torch.empty_like(t) for t in (qs[r], ks[r], vs[r]))
                staged.append((oh, sh, dq, dk, dv, hb))
        torch.cuda.synchronize()
        for r in range(world):
            if hostbuf:
                oh, sh, dq, dk, dv, hb = staged[r]
                hosts[r].layer_hostbuf(hb[0], hb[1], hb[2], oh, dq, dk, dv, outs[r], sh,
                                       sels[r], stream=streams[r])
            else:
                hosts[r].layer(qs[r], ks[r], vs[r], outs[r], sels[r], stream=streams[r])
        torch.cuda.synchronize()
        for r in range(world):
            assert hosts[r].status() == 0
            check(ref, layer, r, outs[r], sels[r])
            if hostbuf:
                check(ref, layer, r, staged[r][0].to("cuda:0"), staged[r][1].to("cuda:0"))
    for h in hosts:
        h.close()
    for f in fabs:
        f.close()
    print(f"PEER_OK all {layers}", flush=True)


def trace_inproc(world, layers):
    """Peer-fabric layers with the event trace on; prints the trace JSONL (reference
    Event schema, Lamport clocks) between markers for the reference validator."""
    cfg, rows, _, _, _ = inputs(world, 0)
    fabs = [spava.Fabric.create_peer(cfg, 0, world, r) for r in range(world)]
    spava.Fabric.peer_attach(fabs)
    hosts = [f.host(r) for r, f in enumerate(fabs)]
    streams = [torch.cuda.Stream() for _ in range(world)]
    for h in hosts:
        h.set_trace(True)
    for layer in range(layers):
        _, _, qs, ks, vs = inputs(world, layer)
        outs = [torch.zeros(rows, HQ * 128, dtype=torch.bfloat16, device="cuda:0") for _ in hosts]
        torch.cuda.synchronize()
        for r in range(world):
            hosts[r].layer(qs[r], ks[r], vs[r], outs[r], stream=streams[r])
        torch.cuda.synchronize()
    events = spava.trace_events([h.trace_records() for h in hosts])
    print("TRACE_JSONL_BEGIN")
    print(spava.trace_jsonl(events))
    print("TRACE_JSONL_END", flush=True)
    for h in hosts:
        h.close()
    for f in fabs:
        f.close()


def encode_inproc(world, rounds):
    """Frame-parallel encode gather over the peer fabric: every rank's E_v share lives in
    its encode region; gather_context must equal split_context of the concatenation."""
    frames, tpf, width = 37, 96, 1024  # rows per frame, row width (bf16)
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
    for rnd in range(rounds):
        g = torch.Generator(device="cuda:0").manual_seed(500 + rnd)
        ev = torch.randn(n_v, width, device="cuda:0", generator=g).to(torch.bfloat16)
        eq = torch.randn(n_t, width, device="cuda:0", generator=g).to(torch.bfloat16)
        torch.cuda.synchronize()
        outs = [torch.full((plan.l_a + 2 * plan.l_b + n_t, width), 7.0, dtype=torch.bfloat16,
                           device="cuda:0") for _ in range(world)]
        off = 0
        for r in range(world):
            with torch.cuda.stream(streams[r]):
                fabs[r].encode_acquire(streams[r])  # peers have read the previous round
                fabs[r].encode_tensor(rows[r], width).copy_(ev[off:off + rows[r]])
            off += rows[r]
        for r in range(world):
            hosts[r].gather_context(rows, eq, outs[r], width * 2, stream=streams[r])
        torch.cuda.synchronize()
        glob = torch.cat([ev, eq])
        for r in range(world):
            want = spava.split_rows(plan, r, glob)
            if not torch.equal(outs[r], want):
                raise AssertionError(f"round {rnd} rank {r}: gathered rows differ")
    for h in hosts:
        h.close()
    for f in fabs:
        f.close()
    print(f"PEER_OK encode {rounds}", flush=True)


def one_rank(rank, world, layers, port):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ref = reference(world, layers)
    cfg, rows, _, _, _ = inputs(world, 0)
    fab = spava.Fabric.create_peer(cfg, 0, world, rank)
    handles = [None] * world
    dist.all_gather_object(handles, fab.peer_handle())
    fab.peer_open(handles)
    host = fab.host(rank)
    stream = torch.cuda.Stream()
    for layer in range(layers):
        _, _, qs, ks, vs = inputs(world, layer)
        torch.cuda.synchronize()
        out = torch.zeros(rows, HQ * 128, dtype=torch.bfloat16, device="cuda:0")
        sel = torch.zeros(2, L_P, dtype=torch.int32, device="cuda:0")
        host.layer(qs[rank], ks[rank], vs[rank], out, sel, stream=stream)
        stream.synchronize()
        assert host.status() == 0
        check(ref, layer, rank, out, sel)
    dist.barrier()  # peers store into this rank's buffer until their last layer is done
    host.close()
    fab.close()
    dist.barrier()
    dist.destroy_process_group()
    print(f"PEER_OK {rank} {layers}", flush=True)


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "inproc":
        inproc(int(sys.argv[2]), int(sys.argv[3]))
    elif mode == "trace":
        trace_inproc(int(sys.argv[2]), int(sys.argv[3]))
    elif mode == "encode":
        encode_inproc(int(sys.argv[2]), int(sys.argv[3]))
    else:
        one_rank(int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]))
