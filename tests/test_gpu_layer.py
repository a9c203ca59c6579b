"""GPU parity of a whole Spava layer (run_host order, simhost.cpp:321-426) through the
C ABI's layer runtime, against the reference's golden fixtures and the C oracle.

Checked per layer: passing-block indices of every virtual block bit-exact; anchor,
block (non-pad rows) and merged query outputs within the bf16 tolerances.
"""
import numpy as np
import pytest

from oracle import oracle as O
from tests.util import (ATOL_BF16_OUT, RTOL_L2_BF16, host_local, load_golden, max_abs, randn,
                        rel_l2)

pytestmark = pytest.mark.gpu


def run_layer(cuda, Q, K, V, n_v, n_t, hosts, l_a, l_p, hq, hkv, zigzag=True, softmax=True,
              query_splits=0, timed_order=None):
    """Drive the local fabric (H simulated hosts on one GPU) over the global padded inputs
    (timed_order: through sim_layer_timed with the hosts in that order)."""
    import torch

    from paper_2601_21444_b200 import spava

    cfg = spava.LayerConfig.make(n_v, n_t, hosts, l_a, l_p, hq, hkv, 128, zigzag=zigzag,
                                 softmax_scores=softmax, query_splits=query_splits)
    fab = spava.Fabric(cfg, 0)
    plan = spava.make_plan(n_v, n_t, hosts, l_a, l_p, zigzag)
    l_b, qoff = plan.l_b, spava.query_offset(plan)
    hs, qs, ks, vs, outs, sels = [], [], [], [], [], []
    for h in range(hosts):
        lo, hi = spava.virtual_pair(plan, h)
        H = fab.host(h)
        hs.append(H)
        for X, lst in ((Q, qs), (K, ks), (V, vs)):
            lst.append(torch.from_numpy(host_local(X, l_a, l_b, lo, hi, qoff, n_t)).to(cuda)
                       .to(torch.bfloat16).contiguous())
        outs.append(torch.zeros((H.rows, hq * 128), dtype=torch.bfloat16, device=cuda))
        sels.append(torch.full((2, max(l_p, 1)), -1, dtype=torch.int32, device=cuda))
    if timed_order is None:
        fab.sim_layer(hs, qs, ks, vs, outs, sels)
    else:
        ms = fab.sim_layer_timed(*[[x[i] for i in timed_order] for x in (hs, qs, ks, vs, outs, sels)])
        assert len(ms) == hosts and all(t > 0 for t in ms)
    torch.cuda.synchronize()
    status = [H.status() for H in hs]
    res = dict(plan=plan, status=status, out=[o.float().cpu().numpy() for o in outs],
               sel=[s.cpu().numpy() for s in sels])
    for H in hs:
        H.close()
    fab.close()
    return res


def check_layer(res, want, n_t, hosts, l_a, zigzag=True):
    from paper_2601_21444_b200 import spava

    plan = res["plan"]
    l_b, l_p = plan.l_b, plan.l_p
    assert res["status"] == [0] * hosts
    for h in range(hosts):
        lo, hi = spava.virtual_pair(plan, h)
        out = res["out"][h]
        for r, v in enumerate((lo, hi)):
            cnt = int(want["sel_count"][v])
            # the contract: passing-block indices bit-exact (ties -> lowest index)
            assert np.array_equal(res["sel"][h][r, :cnt], want["sel"][v, :cnt]), (h, v)
            nv = spava.block_valid_rows(plan, v)
            got = out[l_a + r * l_b: l_a + r * l_b + nv]
            ref = want["blocks"][v][:nv]
            assert max_abs(got, ref) <= ATOL_BF16_OUT, (h, v, max_abs(got, ref))
            assert rel_l2(got, ref) <= RTOL_L2_BF16, (h, v, rel_l2(got, ref))
        if l_a:
            assert max_abs(out[:l_a], want["anchor"]) <= ATOL_BF16_OUT
            assert rel_l2(out[:l_a], want["anchor"]) <= RTOL_L2_BF16
        q = out[l_a + 2 * l_b: l_a + 2 * l_b + n_t]
        assert max_abs(q, want["query"]) <= ATOL_BF16_OUT, max_abs(q, want["query"])
        assert rel_l2(q, want["query"]) <= RTOL_L2_BF16


@pytest.mark.parametrize("name", ["layer_h2_gqa", "layer_h4_pad", "layer_h2_naive",
                                  "layer_h1_full", "layer_h2_raw"])
def test_layer_golden(cuda, name):
    """Golden fixtures generated from the UNMODIFIED reference operators."""
    g = load_golden(name)
    n_v, n_t, hosts, l_a, l_p, hq, hkv, dh, zz, sm = [int(x) for x in g["cfg"]]
    assert dh == 128
    res = run_layer(cuda, g["Q"], g["K"], g["V"], n_v, n_t, hosts, l_a, l_p, hq, hkv, bool(zz),
                    bool(sm))
    check_layer(res, g, n_t, hosts, l_a, bool(zz))


@pytest.mark.parametrize("hosts,zigzag,splits", [(4, True, 0), (2, False, 3)])
def test_layer_c0_shape(cuda, hosts, zigzag, splits):
    """C0 geometry (8K tokens, 16 q / 2 kv heads, d=128) against the C oracle layer."""
    from paper_2601_21444_b200 import spava

    n, n_t, hq, hkv = 8192, 64, 16, 2
    n_v = n - n_t
    l_a, l_p = n // 64, n // 128
    plan = spava.make_plan(n_v, n_t, hosts, l_a, l_p, zigzag)
    n_pad = l_a + 2 * hosts * plan.l_b + n_t
    rng = np.random.default_rng(100 + hosts)
    Q, K, V = randn(rng, n_pad, hq * 128), randn(rng, n_pad, hkv * 128), randn(rng, n_pad, hkv * 128)
    want = O.spava_layer(Q, K, V, n_v, n_t, hosts, l_a, l_p, hq, hkv, 128, zigzag=zigzag)
    res = run_layer(cuda, Q, K, V, n_v, n_t, hosts, l_a, l_p, hq, hkv, zigzag, True, splits)
    check_layer(res, want, n_t, hosts, l_a, zigzag)


def test_sim_layer_timed_any_host_order(cuda):
    """sim_layer_timed accepts the fabric's hosts in any order (tools/sim_scaling.py rotates
    it so every host is timed before a power cap sets in): outputs and passing indices are
    bit-identical to sim_layer's; a host listed twice is rejected."""
    import torch

    from paper_2601_21444_b200 import spava

    n, n_t, hq, hkv, hosts = 8192, 64, 16, 2, 4
    n_v, l_a, l_p = n - n_t, n // 64, n // 128
    plan = spava.make_plan(n_v, n_t, hosts, l_a, l_p, True)
    n_pad = l_a + 2 * hosts * plan.l_b + n_t
    rng = np.random.default_rng(31)
    Q, K, V = randn(rng, n_pad, hq * 128), randn(rng, n_pad, hkv * 128), randn(rng, n_pad, hkv * 128)
    base = run_layer(cuda, Q, K, V, n_v, n_t, hosts, l_a, l_p, hq, hkv)
    for order in ([2, 3, 0, 1], [3, 1, 2, 0]):
        got = run_layer(cuda, Q, K, V, n_v, n_t, hosts, l_a, l_p, hq, hkv, timed_order=order)
        assert got["status"] == [0] * hosts
        for h in range(hosts):
            assert np.array_equal(got["sel"][h], base["sel"][h]), (order, h)
            assert np.array_equal(got["out"][h], base["out"][h]), (order, h)
    cfg = spava.LayerConfig.make(n_v, n_t, hosts, l_a, l_p, hq, hkv, 128)
    fab = spava.Fabric(cfg, 0)
    hs = [fab.host(h) for h in range(hosts)]
    bufs = [[torch.zeros((hs[0].rows, w * 128), dtype=torch.bfloat16, device=cuda) for _ in range(hosts)]
            for w in (hq, hkv, hkv, hq)]
    with pytest.raises(RuntimeError, match="each once"):
        fab.sim_layer_timed([hs[0], hs[0], hs[2], hs[3]], *bufs)
    for H in hs:
        H.close()
    fab.close()


def test_nccl_fabric_world1_matches_local(cuda):
    """The NCCL fabric (in-place allgathers on the comm stream, event-ordered) at world
    size 1 gives the same layer as the local fabric (H=1)."""
    import torch

    from paper_2601_21444_b200 import spava

    n_v, n_t, l_a, l_p, hq, hkv = 1300, 32, 20, 96, 4, 2
    cfg = spava.LayerConfig.make(n_v, n_t, 1, l_a, l_p, hq, hkv)
    loc = spava.Fabric(cfg, 0)
    nc = spava.Fabric(cfg, 0, unique_id=spava.nccl_unique_id(), world=1, rank=0)
    h_loc, h_nc = loc.host(0), nc.host(0)
    rows = h_loc.rows
    g = torch.Generator(device=cuda).manual_seed(5)
    q = torch.randn(rows, hq * 128, device=cuda, generator=g).to(torch.bfloat16)
    k = torch.randn(rows, hkv * 128, device=cuda, generator=g).to(torch.bfloat16)
    v = torch.randn(rows, hkv * 128, device=cuda, generator=g).to(torch.bfloat16)
    outs, sels = [], []
    for host in (h_loc, h_nc):
        o = torch.zeros(rows, hq * 128, dtype=torch.bfloat16, device=cuda)
        s = torch.zeros(2, l_p, dtype=torch.int32, device=cuda)
        host.layer(q, k, v, o, s)
        torch.cuda.synchronize()
        assert host.status() == 0
        outs.append(o)
        sels.append(s)
    assert torch.equal(sels[0], sels[1])
    assert torch.equal(outs[0], outs[1])
    for x in (h_loc, h_nc):
        x.close()
    loc.close()
    nc.close()


@pytest.mark.parametrize("nccl", [False, True])
def test_host_buffer_layer_matches_device_layer(cuda, nccl):
    """spava_host_layer_hostbuf (pinned host in/out, copies pipelined with the phases) gives
    bit-identical outputs and indices to spava_host_layer on device buffers, and runs
    back to back without the copies of one step racing the kernels of the next."""
    import torch

    from paper_2601_21444_b200 import spava

    n_v, n_t, l_a, l_p, hq, hkv = 2100, 64, 32, 128, 4, 2
    cfg = spava.LayerConfig.make(n_v, n_t, 1, l_a, l_p, hq, hkv)
    fab = (spava.Fabric(cfg, 0, unique_id=spava.nccl_unique_id(), world=1, rank=0) if nccl
           else spava.Fabric(cfg, 0))
    host = fab.host(0)
    rows = host.rows
    g = torch.Generator(device=cuda).manual_seed(11)
    ins = [torch.randn(rows, w * 128, device=cuda, generator=g).to(torch.bfloat16) for w in (hq, hkv, hkv)]
    o_ref = torch.zeros(rows, hq * 128, dtype=torch.bfloat16, device=cuda)
    s_ref = torch.zeros(2, l_p, dtype=torch.int32, device=cuda)
    host.layer(*ins, o_ref, s_ref)
    torch.cuda.synchronize()
    hins = [x.cpu().pin_memory() for x in ins]
    dev_bufs = [torch.empty_like(x) for x in ins]
    o_d = torch.empty_like(o_ref)
    s_d = torch.empty_like(s_ref)
    for it in range(3):
        o_h = torch.zeros(o_ref.shape, dtype=o_ref.dtype).pin_memory()
        s_h = torch.zeros(s_ref.shape, dtype=s_ref.dtype).pin_memory()
        host.layer_hostbuf(*hins, o_h, *dev_bufs, o_d, s_h, s_d)
        torch.cuda.synchronize()
        assert host.status() == 0
        assert torch.equal(s_h, s_ref.cpu()), it
        assert torch.equal(o_h, o_ref.cpu()), it
    host.close()
    fab.close()


@pytest.mark.parametrize("hosts,n_t", [(2, 37), (8, 128)])
def test_layer_7b_heads(cuda, hosts, n_t):
    """Qwen2.5-VL-7B head shape (28 q / 4 kv heads, GQA group 7 -> no head pairing) with a
    ragged query block and, at 8 hosts, a padded tail, against the C oracle layer."""
    from paper_2601_21444_b200 import spava

    n_v, hq, hkv = 3001, 28, 4
    l_a, l_p = 40, 96
    plan = spava.make_plan(n_v, n_t, hosts, l_a, l_p, True)
    n_pad = l_a + 2 * hosts * plan.l_b + n_t
    rng = np.random.default_rng(700 + hosts)
    Q, K, V = randn(rng, n_pad, hq * 128), randn(rng, n_pad, hkv * 128), randn(rng, n_pad, hkv * 128)
    want = O.spava_layer(Q, K, V, n_v, n_t, hosts, l_a, l_p, hq, hkv, 128)
    res = run_layer(cuda, Q, K, V, n_v, n_t, hosts, l_a, l_p, hq, hkv)
    check_layer(res, want, n_t, hosts, l_a, True)


@pytest.mark.parametrize("nccl", [False, True])
def test_graph_replay_matches_layer(cuda, nccl):
    """A layer captured as a CUDA graph (side / comm streams and NCCL rounds included)
    replays bit-identically to spava_host_layer, also after the inputs are refilled."""
    import torch

    from paper_2601_21444_b200 import spava

    n_v, n_t, l_a, l_p, hq, hkv = 3000, 64, 32, 128, 4, 2
    cfg = spava.LayerConfig.make(n_v, n_t, 1, l_a, l_p, hq, hkv)
    fab = (spava.Fabric(cfg, 0, unique_id=spava.nccl_unique_id(), world=1, rank=0) if nccl
           else spava.Fabric(cfg, 0))
    host = fab.host(0)
    rows = host.rows
    g = torch.Generator(device=cuda).manual_seed(23)
    q, k, v = [torch.randn(rows, w * 128, device=cuda, generator=g).to(torch.bfloat16) for w in (hq, hkv, hkv)]
    out = torch.zeros(rows, hq * 128, dtype=torch.bfloat16, device=cuda)
    sel = torch.zeros(2, l_p, dtype=torch.int32, device=cuda)
    s = torch.cuda.Stream()
    host.capture_layer(q, k, v, out, sel, stream=s)
    for it in range(2):
        if it:
            for x in (q, k, v):
                x.copy_(torch.randn(x.shape, device=cuda, generator=g).to(torch.bfloat16))
        o_ref = torch.zeros_like(out)
        s_ref = torch.zeros_like(sel)
        host.layer(q, k, v, o_ref, s_ref)
        torch.cuda.synchronize()
        host.replay_layer(s)
        s.synchronize()
        assert torch.equal(sel, s_ref), it
        assert torch.equal(out, o_ref), it
    host.close()
    fab.close()


@pytest.mark.parametrize("nccl", [False, True])
def test_schedule_and_delay_independence(cuda, nccl):
    """acceptance.cpp:221-268 (criterion 5) on the GPU runtime: the overlapped schedule, the
    serialized one (scorer on the caller's stream) and runs with a delay injected before
    each phase's stream position give bit-identical outputs and indices."""
    import torch

    from paper_2601_21444_b200 import spava

    n_v, n_t, l_a, l_p, hq, hkv = 5000, 64, 64, 128, 4, 2
    cfg = spava.LayerConfig.make(n_v, n_t, 1, l_a, l_p, hq, hkv)
    fab = (spava.Fabric(cfg, 0, unique_id=spava.nccl_unique_id(), world=1, rank=0) if nccl
           else spava.Fabric(cfg, 0))
    host = fab.host(0)
    rows = host.rows
    g = torch.Generator(device=cuda).manual_seed(31)
    q, k, v = [torch.randn(rows, w * 128, device=cuda, generator=g).to(torch.bfloat16) for w in (hq, hkv, hkv)]

    def run():
        o = torch.zeros(rows, hq * 128, dtype=torch.bfloat16, device=cuda)
        s = torch.zeros(2, l_p, dtype=torch.int32, device=cuda)
        host.layer(q, k, v, o, s)
        torch.cuda.synchronize()
        assert host.status() == 0
        return o, s

    o_ref, s_ref = run()
    host.set_timing(2)  # serialized: scorer on the caller's stream
    o, s = run()
    host.set_timing(False)
    assert torch.equal(o, o_ref) and torch.equal(s, s_ref)
    for which in range(4):
        host.set_delay(which, 2_000_000)  # 2 ms
        o, s = run()
        host.set_delay(which, 0)
        assert torch.equal(o, o_ref) and torch.equal(s, s_ref), which
    host.close()
    fab.close()


def test_instrumented_flops_match_formula(cuda):
    """acceptance.cpp:130-182 (criterion 3) on the GPU runtime: the attention FLOPs the
    runtime counts at launch (reference convention, attention.cpp:33-36) equal bench.py's
    per-host formula exactly; minus the block->anchor and query terms they equal the
    reference's attn_flops_per_host (metrics.cpp:11-15); zigzag balances them, naive does
    not."""
    import random

    import torch

    import bench
    from paper_2601_21444_b200 import spava

    rnd = random.Random(3)
    for _ in range(6):
        hosts = rnd.randint(1, 4)
        l_b, l_a, n_t = rnd.randint(2, 5) * 64, rnd.choice([0, 64, 128]), rnd.choice([16, 64])
        l_p = rnd.randint(0, l_b // 64) * 32
        n_v = l_a + 2 * hosts * l_b  # no pad rows
        hq, hkv = 4, 2
        subsets = {}
        for zz in (True, False):
            cfg = spava.LayerConfig.make(n_v, n_t, hosts, l_a, l_p, hq, hkv, zigzag=zz)
            fab = spava.Fabric(cfg, 0)
            hs = [fab.host(h) for h in range(hosts)]
            rows = hs[0].rows
            ins = [[torch.randn(rows, w * 128, device=cuda).to(torch.bfloat16) for w in (hq, hkv, hkv)]
                   for _ in range(hosts)]
            outs = [torch.empty(rows, hq * 128, dtype=torch.bfloat16, device=cuda) for _ in range(hosts)]
            for h in hs:
                h.set_timing(True)
            fab.sim_layer(hs, [x[0] for x in ins], [x[1] for x in ins], [x[2] for x in ins], outs)
            torch.cuda.synchronize()
            g = dict(hosts=hosts, l_a=l_a, l_b=l_b, l_p=l_p, n_t=n_t)
            d = hq * 128
            sub = []
            for h, X in enumerate(hs):
                got = X.timing()["attention_flops"]
                assert got == bench.attn_flops_host(g, hq, h, zz), (hosts, zz, h)
                a0, a1 = spava.slice_anchor(l_a, hosts, h)
                extra = (8 * l_a * l_b + 4 * n_t * ((a1 - a0) + 2 * l_b) +
                         (2 * n_t * n_t if h == hosts - 1 else 0)) * d
                sub.append(got - extra)
                X.set_timing(False)
            if zz:
                b2 = 2 * l_a * l_a * d + 4 * l_b * l_b * d + 4 * (2 * hosts - 1) * l_p * l_b * d
                assert all(x == b2 for x in sub), (sub, b2)
            subsets[zz] = sub
            for X in hs:
                X.close()
            fab.close()
        if hosts >= 2 and l_p >= 1:
            assert max(subsets[False]) / min(subsets[False]) > 1.0


@pytest.mark.parametrize("norm", [True, False])
def test_decoder_layer_matches_reference_math(cuda, norm):
    """f2: the decoder layer around the path (simhost.cpp:196-207, 431-436) against an fp32
    restatement of the same math whose attention is the C oracle's Spava layer on the
    same (bf16-rounded) q, k, v."""
    import torch

    from paper_2601_21444_b200 import spava

    n_v, n_t, l_a, l_p, hq, hkv, D, ffn = 1500, 32, 32, 96, 4, 2, 512, 1024
    plan = spava.make_plan(n_v, n_t, 1, l_a, l_p)
    cfg = spava.LayerConfig.make(n_v, n_t, 1, l_a, l_p, hq, hkv)
    fab = spava.Fabric(cfg, 0)
    host = fab.host(0)
    rows = host.rows
    g = torch.Generator(device=cuda).manual_seed(41)
    bf = lambda *s, sc=1.0: (torch.randn(*s, device=cuda, generator=g) * sc).to(torch.bfloat16)
    x = bf(rows, D)
    w_qkv = bf(D, (hq + 2 * hkv) * 128, sc=D ** -0.5)
    w_o = bf(hq * 128, D, sc=(hq * 128) ** -0.5)
    w_1 = bf(D, ffn, sc=D ** -0.5)
    w_2 = bf(ffn, D, sc=ffn ** -0.5)
    g_1 = (1 + 0.1 * torch.randn(D, device=cuda, generator=g)) if norm else None
    g_2 = (1 + 0.1 * torch.randn(D, device=cuda, generator=g)) if norm else None
    x0 = x.float().clone()
    host.decoder_layer(x, w_qkv, w_o, w_1, w_2, g_1, g_2)
    torch.cuda.synchronize()
    assert host.status() == 0

    def ln(t, gain):
        if gain is None:
            return t
        return torch.nn.functional.layer_norm(t, (D,), eps=1e-5) * gain

    xn = ln(x0, g_1).to(torch.bfloat16).float()
    qkv = (xn @ w_qkv.float()).to(torch.bfloat16).float()
    q, k, v = qkv[:, :hq * 128], qkv[:, hq * 128:(hq + hkv) * 128], qkv[:, (hq + hkv) * 128:]
    want = O.spava_layer(q.cpu().numpy(), k.cpu().numpy(), v.cpu().numpy(), n_v, n_t, 1, l_a, l_p, hq, hkv, 128)
    att = np.concatenate([want["anchor"], want["blocks"][0], want["blocks"][1], want["query"]])
    a = torch.from_numpy(att).to(cuda).to(torch.bfloat16).float()
    xr = x0 + a @ w_o.float()
    f = ln(xr, g_2).to(torch.bfloat16).float()
    h = torch.relu(f @ w_1.float()).to(torch.bfloat16).float()
    xr = xr + h @ w_2.float()
    got = x.float()
    rl2 = ((got - xr).norm() / xr.norm()).item()
    assert rl2 < 1.5e-2, rl2
    host.close()
    fab.close()


def test_fused_query_merge_matches_separate_launch(cuda):
    """f1: the final query merge rides in the stage-2 launch (trailing CTAs) -- outputs and
    indices bit-identical to the separate merge launch, with one launch fewer per layer."""
    import torch

    from paper_2601_21444_b200 import spava

    n_v, n_t, l_a, l_p, hq, hkv = 3000, 96, 40, 128, 16, 2
    cfg = spava.LayerConfig.make(n_v, n_t, 1, l_a, l_p, hq, hkv)
    fab = spava.Fabric(cfg, 0)
    H = fab.host(0)
    g = torch.Generator(device=cuda).manual_seed(7)
    q = torch.randn(H.rows, hq * 128, device=cuda, generator=g).to(torch.bfloat16)
    k = torch.randn(H.rows, hkv * 128, device=cuda, generator=g).to(torch.bfloat16)
    v = torch.randn(H.rows, hkv * 128, device=cuda, generator=g).to(torch.bfloat16)
    res = {}
    try:
        for fused in (0, 1):
            spava._check(spava.lib().spava_debug_fused_merge(fused))
            out = torch.zeros(H.rows, hq * 128, dtype=torch.bfloat16, device=cuda)
            sel = torch.zeros(2, l_p, dtype=torch.int32, device=cuda)
            H.layer(q, k, v, out, sel)  # warm (lazy module loads)
            torch.cuda.synchronize()
            n0 = spava.kernel_launches()
            H.layer(q, k, v, out, sel)
            torch.cuda.synchronize()
            res[fused] = (out.clone(), sel.clone(), spava.kernel_launches() - n0)
    finally:
        spava._check(spava.lib().spava_debug_fused_merge(-1))
    assert torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1])
    assert res[1][2] == res[0][2] - 1, (res[0][2], res[1][2])
