"""CPU tests of the parity checker itself.

1. The C restatement (oracle/liboracle.so) is bit-identical to the UNMODIFIED reference
   operators (oracle/_ref/libseqpar_ref.so) on random inputs -- when _ref is built.
2. It reproduces the committed golden fixtures (generated from the reference) exactly.
3. The reference's own unit-test pins (test_approx.cpp, test_tensor.cpp,
   acceptance.cpp criteria 2 and 6) hold for it.
"""
import numpy as np
import pytest

from oracle import oracle as O
from tests.util import bf16, load_golden, randn

HAVE_REF = O.available("ref")
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (needs /root/reference)")


def same_bits(a, b):
    a, b = np.asarray(a, np.float32), np.asarray(b, np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


# ------------------------------------------------------------- vs reference
@needs_ref
@pytest.mark.parametrize("seed", range(4))
def test_c_oracle_equals_reference_bitwise(seed):
    rng = np.random.default_rng(seed)
    hq, hkv, dh = [(4, 2, 16), (2, 2, 32), (6, 3, 8), (4, 1, 16)][seed]
    n_t, l_b, l_a = 5 + seed, 40 + 7 * seed, 6
    q = randn(rng, n_t, hq * dh)
    k, v = randn(rng, l_b, hkv * dh), randn(rng, l_b, hkv * dh)
    pad = (np.arange(l_b) >= l_b - seed).astype(np.uint8)
    for sm in (True, False):
        assert same_bits(O.score_block(q, k, hq, hkv, dh, pad, sm, "c"),
                         O.score_block(q, k, hq, hkv, dh, pad, sm, "ref"))
    s = O.score_block(q, k, hq, hkv, dh, pad, True, "c")
    for lp in (0, 3, l_b // 2, l_b):
        assert np.array_equal(O.select_essential(s, lp, 11, "c"), O.select_essential(s, lp, 11, "ref"))
    qb = randn(rng, l_b, hq * dh)
    ka, va = randn(rng, l_a, hkv * dh), randn(rng, l_a, hkv * dh)
    kp, vp = randn(rng, 9, hkv * dh), randn(rng, 9, hkv * dh)
    assert same_bits(O.block_attention(qb, k, v, pad, ka, va, kp, vp, hq, hkv, dh, "c"),
                     O.block_attention(qb, k, v, pad, ka, va, kp, vp, hq, hkv, dh, "ref"))
    kq, vq = randn(rng, n_t, hkv * dh), randn(rng, n_t, hkv * dh)
    for incl in (True, False):
        a = O.query_attention(q, ka, va, 1, 4, k, v, pad, k, v, None, kq, vq, incl, hq, hkv, dh, "c")
        b = O.query_attention(q, ka, va, 1, 4, k, v, pad, k, v, None, kq, vq, incl, hq, hkv, dh, "ref")
        assert same_bits(a[0], b[0]) and same_bits(a[1], b[1])
    assert same_bits(O.anchor_attention(qb[:l_a], ka, va, hq, hkv, dh, "c"),
                     O.anchor_attention(qb[:l_a], ka, va, hq, hkv, dh, "ref"))
    outs = [rng.standard_normal((n_t, hq * dh)).astype(np.float32) for _ in range(3)]
    lses = [rng.standard_normal((n_t, hq)).astype(np.float32) for _ in range(3)]
    lses[2][0, 0] = -np.inf
    assert same_bits(O.mha_merge(outs, lses, hq, dh, "c"), O.mha_merge(outs, lses, hq, dh, "ref"))


@needs_ref
def test_partition_equals_reference():
    for hosts in range(1, 9):
        for zz in (True, False):
            for h in range(hosts):
                assert O.virtual_pair(hosts, zz, h, "c") == O.virtual_pair(hosts, zz, h, "ref")
            for v in range(2 * hosts):
                assert O.physical_of(hosts, zz, v, "c") == O.physical_of(hosts, zz, v, "ref")
        for n_v in (20, 21, 517, 8128):
            for l_a in (0, 4, 16):
                a = O.split_geometry(n_v, 3, hosts, l_a, 0, "c")
                b = O.split_geometry(n_v, 3, hosts, l_a, 0, "ref")
                assert a["l_b"] == b["l_b"] and a["pad"] == b["pad"]
                assert np.array_equal(a["offsets"], b["offsets"])
                assert np.array_equal(a["pad_masks"], b["pad_masks"])
        for l_a in range(0, 21):
            for h in range(hosts):
                assert O.slice_anchor(l_a, hosts, h, "c") == O.slice_anchor(l_a, hosts, h, "ref")


# ------------------------------------------------------------- vs golden
@pytest.mark.parametrize("name", ["layer_h2_gqa", "layer_h4_pad", "layer_h2_naive",
                                  "layer_h1_full", "layer_h2_raw"])
def test_c_oracle_reproduces_golden_layer(name):
    g = load_golden(name)
    n_v, n_t, hosts, l_a, l_p, hq, hkv, dh, zz, sm = [int(x) for x in g["cfg"]]
    r = O.spava_layer(g["Q"], g["K"], g["V"], n_v, n_t, hosts, l_a, l_p, hq, hkv, dh,
                      zigzag=bool(zz), softmax_scores=bool(sm))
    for v in range(2 * hosts):
        c = int(g["sel_count"][v])
        assert int(r["sel_count"][v]) == c
        assert np.array_equal(r["sel"][v, :c], g["sel"][v, :c])
    assert same_bits(r["anchor"], g["anchor"])
    assert same_bits(r["blocks"], g["blocks"])
    assert same_bits(r["query"], g["query"])
    assert same_bits(r["qpart_out"], g["qpart_out"]) and same_bits(r["qpart_lse"], g["qpart_lse"])


def test_select_ties_golden():
    g = load_golden("select_ties")
    for c in range(len(g["n"])):
        n, lp = int(g["n"][c]), int(g["l_p"][c])
        want = g["sel"][c][g["sel"][c] >= 0]
        assert np.array_equal(O.select_essential(g["scores"][c, :n], lp, 0), want)


# ------------------------------------------------------ reference test pins
def test_score_context_closed_form():
    """test_approx.cpp:26-44"""
    k = np.array([[0.0], [np.log(np.float32(3.0))]], np.float32)
    s = O.score_context(np.ones((1, 1), np.float32), k, 1.0)
    assert abs(s[0] - 0.25) < 1e-6 and abs(s[1] - 0.75) < 1e-6
    s2 = O.score_context(np.ones((2, 1), np.float32), k, 1.0)
    assert abs(s2[0] - 0.5) < 1e-6 and abs(s2[1] - 1.5) < 1e-6


def test_score_context_vs_fp64_bruteforce():
    """test_approx.cpp:46-69"""
    rng = np.random.default_rng(21)
    q = rng.standard_normal((4, 6)).astype(np.float32)
    k = rng.standard_normal((16, 6)).astype(np.float32)
    scale = np.float32(1.0 / np.sqrt(6.0))
    s = O.score_context(q, k, scale)
    lg = (q.astype(np.float64) @ k.astype(np.float64).T) * scale
    p = np.exp(lg - lg.max(1, keepdims=True))
    p /= p.sum(1, keepdims=True)
    assert np.allclose(s, p.sum(0), rtol=1e-6)


def test_score_context_pad_and_raw():
    """test_approx.cpp:71-88"""
    rng = np.random.default_rng(22)
    q = rng.standard_normal((2, 4)).astype(np.float32)
    k = rng.standard_normal((5, 4)).astype(np.float32)
    pad = np.array([0, 0, 1, 0, 1], np.uint8)
    s = O.score_context(q, k, 0.5, pad)
    assert np.isinf(s[2]) and np.isinf(s[4]) and np.isfinite(s[0])
    raw = O.score_context(q, k, 0.5, pad, softmax=False)
    assert abs(raw[0] - 0.5 * float((q.astype(np.float64) @ k[0].astype(np.float64)).sum())) < 1e-5


def test_select_pins():
    """test_approx.cpp:90-105"""
    sv = np.array([0.1, 0.9, 0.5, 0.9], np.float32)
    assert O.select_essential(sv, 2, 0).tolist() == [1, 3]
    assert O.select_essential(np.full(4, 0.5, np.float32), 2, 0).tolist() == [0, 1]
    assert O.select_essential(sv, 4, 10).tolist() == [10, 11, 12, 13]


def test_select_vs_stable_sort_1000():
    """acceptance.cpp:271-294 (criterion 6)"""
    rng = np.random.default_rng(6)
    for _ in range(1000):
        n = int(rng.integers(1, 25))
        lp = int(rng.integers(0, n + 1))
        s = (rng.integers(0, 4, n) / 3.0).astype(np.float32)
        order = sorted(range(n), key=lambda j: -s[j])  # Python sort is stable
        assert O.select_essential(s, lp, 0).tolist() == sorted(order[:lp])


def test_attention_single_key_and_invalid_rows():
    """test_tensor.cpp:116-128, 163-174"""
    rng = np.random.default_rng(9)
    q, k, v = (rng.standard_normal((1, 4)).astype(np.float32) for _ in range(3))
    out, lse = O.attention_lse(q, [dict(k=k, v=v)], 0.5)
    assert np.allclose(out, v, atol=1e-6)
    assert abs(lse[0] - float(np.float32((q * k).sum()) * np.float32(0.5))) < 1e-5
    q2 = rng.standard_normal((2, 4)).astype(np.float32)
    k3 = rng.standard_normal((3, 4)).astype(np.float32)
    pad = np.ones(3, np.uint8)
    with pytest.raises(O.OracleError):
        O.attention_lse(q2, [dict(k=k3, v=k3, pad=pad)], 1.0)
    out, lse = O.attention_lse(q2, [dict(k=k3, v=k3, pad=pad)], 1.0, allow_invalid=True)
    assert not np.isfinite(lse[0]) and out[0, 0] == 0.0


def test_causal_vs_bruteforce():
    """test_tensor.cpp:148-161"""
    rng = np.random.default_rng(11)
    q, k, v = (rng.standard_normal((4, 6)).astype(np.float32) for _ in range(3))
    scale = np.float32(1.0 / np.sqrt(6.0))
    out, _ = O.attention_lse(q, [dict(k=k, v=v, causal=True)], scale)
    lg = (q.astype(np.float64) @ k.astype(np.float64).T) * scale
    lg[np.triu_indices(4, 1)] = -np.inf
    p = np.exp(lg - lg.max(1, keepdims=True))
    p /= p.sum(1, keepdims=True)
    assert np.abs(out - p @ v).max() <= 1e-6


def test_merge_over_random_partitions():
    """acceptance.cpp:91-127 (criterion 2): merge over disjoint partitions == dense."""
    for seed in range(100):
        rng = np.random.default_rng(seed)
        n_k, n_q, d = int(rng.integers(2, 33)), int(rng.integers(1, 7)), int(rng.integers(2, 13))
        q, k, v = (rng.standard_normal((r, d)).astype(np.float32) for r in (n_q, n_k, n_k))
        scale = np.float32(1.0 / np.sqrt(d))
        segs = int(rng.integers(1, min(8, n_k) + 1))
        assign = np.concatenate([np.arange(segs), rng.integers(0, segs, n_k - segs)])
        rng.shuffle(assign)
        outs, lses = [], []
        for s in range(segs):
            m = np.where(assign == s)[0]
            o, l = O.attention_lse(q, [dict(k=k[m], v=v[m])], scale)
            outs.append(o)
            lses.append(l)
        merged = O.merge_partials(outs, lses)
        lg = (q.astype(np.float64) @ k.astype(np.float64).T) * scale
        p = np.exp(lg - lg.max(1, keepdims=True))
        p /= p.sum(1, keepdims=True)
        assert np.abs(merged - p @ v).max() <= 1e-6


def test_determinism():
    """test_tensor.cpp:254-264"""
    rng = np.random.default_rng(15)
    q, k, v = rng.standard_normal((5, 8)), rng.standard_normal((7, 8)), rng.standard_normal((7, 8))
    a = O.attention_lse(q, [dict(k=k, v=v)], 0.3)
    b = O.attention_lse(q, [dict(k=k, v=v)], 0.3)
    assert same_bits(a[0], b[0]) and same_bits(a[1], b[1])


def test_no_compression_exactness_vs_dense():
    """acceptance.cpp:60-88 / criterion 8: with l_p = l_b every block sees all earlier
    keys, so the Spava layer equals dense causal attention over [anchor|blocks|query]."""
    rng = np.random.default_rng(3)
    hq, hkv, dh = 2, 1, 16
    n_v, n_t, hosts, l_a = 130, 6, 2, 10
    g = O.split_geometry(n_v, n_t, hosts, l_a, 0)
    l_b = g["l_b"]
    n_pad = l_a + 2 * hosts * l_b + n_t
    Q, K, V = randn(rng, n_pad, hq * dh), randn(rng, n_pad, hkv * dh), randn(rng, n_pad, hkv * dh)
    r = O.spava_layer(Q, K, V, n_v, n_t, hosts, l_a, l_b, hq, hkv, dh)
    dense, _ = O.mha_lse(Q, [dict(k=K, v=V, causal=True)], hq, hkv, dh)
    assert np.abs(r["anchor"] - dense[:l_a]).max() <= 1e-5
    for v in range(2 * hosts):
        o = l_a + v * l_b
        assert np.abs(r["blocks"][v] - dense[o:o + l_b]).max() <= 1e-5
    assert np.abs(r["query"] - dense[-n_t:]).max() <= 1e-5
    _ = bf16
