"""Generate tests/golden/*.npz from the UNMODIFIED reference operators.

Run in the build container (needs oracle/_ref/libseqpar_ref.so, i.e. /root/reference):
    make -C oracle && python tests/golden/make_golden.py

Every input is drawn from numpy's PCG64 with a fixed seed and rounded to bf16
(the GPU path's storage type), then fed to the reference as fp32; outputs are the
reference's own fp32 results.  The fixtures travel with the repo, so parity on
the GPU box never needs /root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 -> fp32 (numpy only)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def to_bits(x: np.ndarray) -> np.ndarray:
    """bf16-valued fp32 -> raw bf16 bits (uint16) for compact fixtures."""
    return (np.ascontiguousarray(x, np.float32).view(np.uint32) >> 16).astype(np.uint16)


def from_bits(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


def randn(rng, *shape):
    return bf16(rng.standard_normal(shape).astype(np.float32))


def layer_case(seed, n_v, n_t, hosts, l_a, l_p, hq, hkv, dh, zigzag=True, softmax=True):
    """One Spava layer composed from the reference operators in run_host order."""
    rng = np.random.default_rng(seed)
    g = O.split_geometry(n_v, n_t, hosts, l_a, l_p, impl="ref")
    lb, VH = g["l_b"], 2 * hosts
    n_pad = l_a + VH * lb + n_t
    Q, K, V = randn(rng, n_pad, hq * dh), randn(rng, n_pad, hkv * dh), randn(rng, n_pad, hkv * dh)
    for v in range(VH):  # pad rows are zero (projection of a zero row)
        for r in range(lb):
            if l_a + v * lb + r >= n_v:
                Q[l_a + v * lb + r] = 0
                K[l_a + v * lb + r] = 0
                V[l_a + v * lb + r] = 0
    qo = g["query_offset"]
    Qq, Kq, Vq = Q[qo:], K[qo:], V[qo:]
    pads = g["pad_masks"]
    sel, scores, pk, pv = [], [], [], []
    for v in range(VH):
        o = l_a + v * lb
        s = O.score_block(Qq, K[o:o + lb], hq, hkv, dh, pads[v], softmax, impl="ref")
        idx = O.select_essential(s, l_p, o, impl="ref")
        scores.append(s)
        sel.append(idx)
        pk.append(K[idx])
        pv.append(V[idx])
    outs, lses = [], []
    for h in range(hosts):
        lo, hi = O.virtual_pair(hosts, zigzag, h, impl="ref")
        a0, a1 = O.slice_anchor(l_a, hosts, h, impl="ref")
        olo, ohi = l_a + lo * lb, l_a + hi * lb
        o, l = O.query_attention(Qq, K[:l_a], V[:l_a], a0, a1, K[olo:olo + lb], V[olo:olo + lb],
                                 pads[lo], K[ohi:ohi + lb], V[ohi:ohi + lb], pads[hi], Kq, Vq,
                                 h == hosts - 1, hq, hkv, dh, impl="ref")
        outs.append(o)
        lses.append(l)
    query = O.mha_merge(outs, lses, hq, dh, impl="ref")
    anchor = O.anchor_attention(Q[:l_a], K[:l_a], V[:l_a], hq, hkv, dh, impl="ref")
    blocks = []
    for v in range(VH):
        o = l_a + v * lb
        kp = np.concatenate([pk[s] for s in range(v)]) if v else np.zeros((0, hkv * dh), np.float32)
        vp = np.concatenate([pv[s] for s in range(v)]) if v else np.zeros((0, hkv * dh), np.float32)
        blocks.append(O.block_attention(Q[o:o + lb], K[o:o + lb], V[o:o + lb], pads[v], K[:l_a],
                                        V[:l_a], kp, vp, hq, hkv, dh, impl="ref"))
    sel_arr = np.full((VH, max(l_p, 1)), -1, np.int32)
    for v in range(VH):
        sel_arr[v, :len(sel[v])] = sel[v]
    return dict(
        cfg=np.array([n_v, n_t, hosts, l_a, l_p, hq, hkv, dh, int(zigzag), int(softmax)], np.int32),
        Q=to_bits(Q), K=to_bits(K), V=to_bits(V), scores=np.stack(scores), sel=sel_arr,
        sel_count=np.array([len(s) for s in sel], np.int32),
        qpart_out=np.stack(outs), qpart_lse=np.stack(lses), query=query, anchor=anchor,
        blocks=np.stack(blocks))


def select_ties_case(seed=6, n_cases=300):
    """acceptance.cpp:271-294 style: tie-heavy score vectors and random l_p."""
    rng = np.random.default_rng(seed)
    ns = rng.integers(1, 200, n_cases)
    scores = np.full((n_cases, 200), -np.inf, np.float32)
    lps = np.zeros(n_cases, np.int32)
    sel = np.full((n_cases, 200), -1, np.int32)
    for c in range(n_cases):
        n = int(ns[c])
        s = (rng.integers(0, 4, n) / 3.0).astype(np.float32)
        if c % 5 == 0:
            s[rng.integers(0, n, max(1, n // 7))] = -np.inf
        lp = int(rng.integers(0, n + 1))
        scores[c, :n] = s
        lps[c] = lp
        idx = O.select_essential(s, lp, 0, impl="ref")
        sel[c, :len(idx)] = idx
    return dict(n=ns.astype(np.int32), scores=scores, l_p=lps, sel=sel)


def main():
    cases = {
        # C0 shape reduced in length (16 q / 2 kv heads, d=128) with a padded tail
        "layer_h2_gqa": layer_case(11, n_v=270, n_t=16, hosts=2, l_a=14, l_p=32, hq=16, hkv=2, dh=128),
        # H=4 zigzag with pad rows, small heads
        "layer_h4_pad": layer_case(12, n_v=517, n_t=8, hosts=4, l_a=8, l_p=16, hq=4, hkv=2, dh=128),
        # naive pairing (load balancing off)
        "layer_h2_naive": layer_case(13, n_v=300, n_t=8, hosts=2, l_a=12, l_p=24, hq=4, hkv=1, dh=128,
                                     zigzag=False),
        # no compression (l_p = l_b): exactness endpoint (acceptance criterion 8)
        "layer_h1_full": layer_case(14, n_v=264, n_t=8, hosts=1, l_a=8, l_p=128, hq=2, hkv=2, dh=128),
        # raw-logit aggregation (score_context softmax_aggregation=false)
        "layer_h2_raw": layer_case(15, n_v=300, n_t=8, hosts=2, l_a=12, l_p=24, hq=4, hkv=2, dh=128,
                                   softmax=False),
    }
    for name, d in cases.items():
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **d)
        print(name, {k: v.shape for k, v in d.items()})
    np.savez_compressed(os.path.join(OUT, "select_ties.npz"), **select_ties_case())
    print("select_ties")


if __name__ == "__main__":
    main()
