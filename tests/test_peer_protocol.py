"""CPU model check of the peer fabric's flag protocol (csrc/capi.cu layer_impl, peer
branch; csrc/peer.cu).

Each rank runs two in-order streams per layer, exactly the operation order layer_impl
enqueues (data stores into peers' slots, epoch flag raises, in-stream flag waits):

  side : fork (main stream finished layer e-1) | wait done[q] >= e-1 (all q)
         | store pass1 slot -> all peers, raise arrive[0]
         | store pass2 slot -> all peers, raise arrive[1]
  main : wait done[q] >= e-1 | store qpartial slot -> all peers, raise arrive[2]
         | wait arrive[0][q] >= e | read pass1 slots | wait arrive[1][q] >= e (+ own side
         stream's pass2 store) | read pass2 slots | wait arrive[2][q] >= e | read qpartial
         | raise done[me] = e in every peer

A random scheduler interleaves all streams of all ranks (any stream whose head operation
is enabled may step).  Checked over many seeds, ranks 2..8 and several layers: no
deadlock, and every read sees the slot of the SAME layer from every peer (a slot is never
overwritten before its reader is done, and never read before it is written).
"""
import random

import pytest


def run_model(world, layers, seed):
    rng = random.Random(seed)
    # slots[owner][round][writer] = layer tag of the data in owner's buffer
    slots = [[[0] * world for _ in range(3)] for _ in range(world)]
    arrive = [[[0] * world for _ in range(3)] for _ in range(world)]  # flags in owner's buffer
    done = [[0] * world for _ in range(world)]
    own_pass = [[0, 0] for _ in range(world)]  # side-stream progress seen by main (event)
    main_layer = [0] * world  # last layer the main stream finished (ev_fork for the side)

    def side_prog(r):
        for e in range(1, layers + 1):
            # the side stream forks from the main stream at the start of every layer
            yield ("wait", lambda r=r, e=e: main_layer[r] >= e - 1)
            yield ("wait", lambda r=r, e=e: all(done[r][q] >= e - 1 for q in range(world) if q != r))
            for rnd in (0, 1):
                def store(r=r, e=e, rnd=rnd):
                    for q in range(world):
                        slots[q][rnd][r] = e  # the gather kernel writes every copy (own too)
                yield ("do", store)

                def raise_(r=r, e=e, rnd=rnd):
                    for q in range(world):
                        if q != r:
                            arrive[q][rnd][r] = e
                    own_pass[r][rnd] = e  # cudaEventRecord(ev[rnd]) on the side stream
                yield ("do", raise_)

    def main_prog(r):
        for e in range(1, layers + 1):
            yield ("wait", lambda r=r, e=e: all(done[r][q] >= e - 1 for q in range(world) if q != r))

            def qstore(r=r, e=e):
                for q in range(world):
                    slots[q][2][r] = e
            yield ("do", qstore)

            def qraise(r=r, e=e):
                for q in range(world):
                    if q != r:
                        arrive[q][2][r] = e
            yield ("do", qraise)
            for rnd in (0, 1, 2):
                yield ("wait", lambda r=r, e=e, rnd=rnd: all(arrive[r][rnd][q] >= e for q in range(world)
                                                             if q != r)
                       and (rnd == 2 or own_pass[r][rnd] >= e))

                def read(r=r, e=e, rnd=rnd):
                    got = slots[r][rnd]
                    assert all(t == e for t in got), (r, e, rnd, got)
                yield ("do", read)

            def release(r=r, e=e):
                for q in range(world):
                    if q != r:
                        done[q][r] = e
                main_layer[r] = e
            yield ("do", release)

    progs = [side_prog(r) for r in range(world)] + [main_prog(r) for r in range(world)]
    heads = [next(p, None) for p in progs]
    steps = 0
    while any(h is not None for h in heads):
        ready = [i for i, h in enumerate(heads) if h is not None and (h[0] == "do" or h[1]())]
        if not ready:
            raise AssertionError(f"deadlock after {steps} steps")
        i = rng.choice(ready)
        if heads[i][0] == "do":
            heads[i][1]()
        heads[i] = next(progs[i], None)
        steps += 1
    return steps


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_peer_protocol_random_interleavings(world):
    for seed in range(60):
        run_model(world, layers=4, seed=seed * 31 + world)


def test_model_detects_missing_release_wait():
    """Sanity of the checker: without the done-wait a fast rank overwrites a slow rank's
    unread slot, which the model must catch for some interleaving."""
    import itertools

    world, layers = 2, 3
    caught = False
    for seed in itertools.islice(itertools.count(), 400):
        rng = random.Random(seed)
        slots = [[0] * world for _ in range(world)]
        arrive = [[0] * world for _ in range(world)]
        # rank program without done waits: store -> raise -> wait -> read, per layer
        progs, heads = [], []
        for r in range(world):
            def prog(r=r):
                for e in range(1, layers + 1):
                    def store(r=r, e=e):
                        for q in range(world):
                            slots[q][r] = e
                    yield ("do", store)

                    def raise_(r=r, e=e):
                        for q in range(world):
                            arrive[q][r] = e
                    yield ("do", raise_)
                    yield ("wait", lambda r=r, e=e: all(arrive[r][q] >= e for q in range(world)))
                    yield ("read", lambda r=r, e=e: all(t == e for t in slots[r]))
            progs.append(prog())
        heads = [next(p) for p in progs]
        while any(h is not None for h in heads):
            ready = [i for i, h in enumerate(heads) if h is not None and (h[0] != "wait" or h[1]())]
            i = rng.choice(ready)
            kind, fn = heads[i]
            if kind == "do":
                fn()
            elif kind == "read" and not fn():
                caught = True
            heads[i] = next(progs[i], None)
        if caught:
            break
    assert caught
