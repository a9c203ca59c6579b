"""Parity at BASELINE.json's full C1 size (32K tokens, Qwen2.5-VL-3B heads):
* passing-block selection bit-exact against the C oracle on a full 16064-key block;
* the no-compression endpoint (l_p = l_b, acceptance.cpp:60-127 "C1") of the whole layer
  equals dense causal attention over the 32K sequence (torch SDPA as the independent
  reference), i.e. the layer's segment bookkeeping is exact at full size."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.util import max_abs, rel_l2

pytestmark = pytest.mark.gpu


def test_c1_block_selection_bit_exact(cuda):
    import torch

    from paper_2601_21444_b200 import spava

    n_t, l_b, hq, hkv, l_p = 128, 16064, 16, 2, 256
    g = torch.Generator(device=cuda).manual_seed(21)
    q = torch.randn(n_t, hq * 128, device=cuda, generator=g).to(torch.bfloat16)
    k = torch.randn(l_b, hkv * 128, device=cuda, generator=g).to(torch.bfloat16)
    got = spava.score_block(q, k, hq, hkv, 128)
    idx, _, _ = spava.select_essential(got, l_p, 512)
    ref = O.score_block(q.float().cpu().numpy(), k.float().cpu().numpy(), hq, hkv, 128, None, True)
    want = O.select_essential(ref, l_p, 512)
    assert np.array_equal(idx.cpu().numpy(), want)
    fin = np.isfinite(ref)
    assert float(np.mean(got.cpu().numpy()[fin] == ref[fin])) > 0.95


def test_c1_no_compression_equals_dense_causal(cuda):
    import torch
    import torch.nn.functional as F

    from paper_2601_21444_b200 import spava

    n, n_t, hq, hkv = 32768, 128, 16, 2
    l_a = n // 64
    n_v = n - n_t
    l_b = (n_v - l_a) // 2
    cfg = spava.LayerConfig.make(n_v, n_t, 1, l_a, l_b, hq, hkv)  # l_p = l_b: no compression
    fab = spava.Fabric(cfg, 0)
    host = fab.host(0)
    assert host.rows == n  # H = 1 zigzag pair (0, 1), no pad: host rows == sequence order
    g = torch.Generator(device=cuda).manual_seed(5)
    q = torch.randn(n, hq * 128, device=cuda, generator=g).to(torch.bfloat16)
    k = torch.randn(n, hkv * 128, device=cuda, generator=g).to(torch.bfloat16)
    v = torch.randn(n, hkv * 128, device=cuda, generator=g).to(torch.bfloat16)
    out = torch.empty(n, hq * 128, dtype=torch.bfloat16, device=cuda)
    sel = torch.empty(2, l_b, dtype=torch.int32, device=cuda)
    host.layer(q, k, v, out, sel)
    torch.cuda.synchronize()
    assert host.status() == 0
    # every block keeps all of its keys, in order (select_essential with l_p = l_b)
    assert torch.equal(sel[0].cpu(), torch.arange(l_a, l_a + l_b, dtype=torch.int32))
    qh = q.view(n, hq, 128).transpose(0, 1).unsqueeze(0)
    kh = k.view(n, hkv, 128).transpose(0, 1).unsqueeze(0)
    vh = v.view(n, hkv, 128).transpose(0, 1).unsqueeze(0)
    dense = F.scaled_dot_product_attention(qh, kh, vh, is_causal=True, enable_gqa=True)
    dense = dense.squeeze(0).transpose(0, 1).reshape(n, hq * 128)
    a, b = out.float(), dense.float()
    err = (a - b).abs().max().item()
    rl2 = ((a - b).norm() / b.norm()).item()
    assert err < 5e-2 and rl2 < 1e-2, (err, rl2)
    host.close()
    fab.close()


def test_split_rows_matches_split_context(cuda):
    """spava_split_rows == split_context's host-local rows (tests/util.host_local, the C
    oracle's layout) bit for bit, pads zero; merge_rows inverts it on the non-pad rows."""
    import torch

    from paper_2601_21444_b200 import spava
    from tests.util import host_local

    for n_v, n_t, hosts, l_a, zz in ((1021, 32, 2, 16, True), (4000, 64, 4, 64, False), (700, 8, 1, 5, True)):
        plan = spava.make_plan(n_v, n_t, hosts, l_a, 64, zz)
        X = torch.arange((n_v + n_t) * 64, dtype=torch.float32, device=cuda).view(n_v + n_t, 64)
        Xp = torch.zeros(plan.l_a + 2 * hosts * plan.l_b + n_t, 64, device=cuda)  # padded global
        Xp[:n_v] = X[:n_v]
        Xp[spava.query_offset(plan):] = X[n_v:]
        back = torch.full_like(X, -1.0)
        for h in range(hosts):
            lo, hi = spava.virtual_pair(plan, h)
            got = spava.split_rows(plan, h, X)
            want = host_local(Xp.cpu().numpy(), plan.l_a, plan.l_b, lo, hi, spava.query_offset(plan), n_t)
            assert np.array_equal(got.cpu().numpy(), want)
            spava.merge_rows(plan, h, got, back, write_shared=(h == 0))
        assert torch.equal(back, X)


@pytest.mark.parametrize("zigzag", [True, False])
def test_c3_eight_hosts_no_compression_equals_dense(cuda, zigzag):
    """C3 (131072 tokens) on 8 simulated hosts with l_p = l_b: device split_context ->
    sim layer (every exchange round, passing range and zigzag/naive placement at full size)
    -> merge back == dense causal attention over the whole sequence (torch SDPA)."""
    import torch
    import torch.nn.functional as F

    from paper_2601_21444_b200 import spava

    n, n_t, hq, hkv, H = 131072, 128, 16, 2, 8
    n_v, l_a = n - n_t, n // 64
    plan = spava.make_plan(n_v, n_t, H, l_a, 1, zigzag)
    l_b = plan.l_b
    assert plan.pad == 0
    cfg = spava.LayerConfig.make(n_v, n_t, H, l_a, l_b, hq, hkv, zigzag=zigzag)
    fab = spava.Fabric(cfg, 0)
    hs = [fab.host(h) for h in range(H)]
    g = torch.Generator(device=cuda).manual_seed(13)
    Q = torch.randn(n, hq * 128, device=cuda, generator=g).to(torch.bfloat16)
    K = torch.randn(n, hkv * 128, device=cuda, generator=g).to(torch.bfloat16)
    V = torch.randn(n, hkv * 128, device=cuda, generator=g).to(torch.bfloat16)
    qs = [spava.split_rows(plan, h, Q) for h in range(H)]
    ks = [spava.split_rows(plan, h, K) for h in range(H)]
    vs = [spava.split_rows(plan, h, V) for h in range(H)]
    outs = [torch.empty_like(x) for x in qs]
    fab.sim_layer(hs, qs, ks, vs, outs)
    out = torch.empty_like(Q)
    for h in range(H):
        spava.merge_rows(plan, h, outs[h], out, write_shared=(h == 0))
    torch.cuda.synchronize()
    del qs, ks, vs, outs
    qh = Q.view(n, hq, 128).transpose(0, 1).unsqueeze(0)
    kh = K.view(n, hkv, 128).transpose(0, 1).unsqueeze(0)
    vh = V.view(n, hkv, 128).transpose(0, 1).unsqueeze(0)
    dense = F.scaled_dot_product_attention(qh, kh, vh, is_causal=True, enable_gqa=True)
    dense = dense.squeeze(0).transpose(0, 1).reshape(n, hq * 128)
    a, b = out.float(), dense.float()
    err = (a - b).abs().max().item()
    rl2 = ((a - b).norm() / b.norm()).item()
    assert err < 5e-2 and rl2 < 1e-2, (err, rl2)
    for h in hs:
        h.close()
    fab.close()
