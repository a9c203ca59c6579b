"""bench.py's geometry and FLOP convention on the CPU: geometry == the C ABI's
split_context plan for every BASELINE config and host count; the per-host attention
FLOPs are balanced under zigzag pairing and not under naive pairing (metrics.cpp:11-15,
acceptance.cpp:130-182), and their B.2 subset equals the reference's attn_flops_per_host
(including its test pin 7680, test_metrics.cpp:47-51)."""
import pytest

import bench
from paper_2601_21444_b200 import spava


@pytest.mark.parametrize("name", sorted(bench.CONFIGS))
@pytest.mark.parametrize("hosts", [1, 2, 4, 8])
def test_geometry_matches_plan(name, hosts):
    g = bench.geometry(bench.CONFIGS[name], hosts)
    p = spava.make_plan(g["n_v"], g["n_t"], hosts, g["l_a"], g["l_p"])
    assert (p.l_b, p.pad, p.l_p, p.l_a) == (g["l_b"], g["pad"], g["l_p"], g["l_a"])


def ref_attn_flops_per_host(l_a, l_b, l_p, hosts, d):
    """metrics.cpp:11-15 restated."""
    return 2 * l_a * l_a * d + 4 * l_b * l_b * d + 4 * (2 * hosts - 1) * l_p * l_b * d


def test_reference_formula_pin():
    assert ref_attn_flops_per_host(4, 8, 2, 2, 16) == 7680  # test_metrics.cpp:48


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
@pytest.mark.parametrize("hosts", [2, 4, 8])
def test_zigzag_balanced_naive_not(name, hosts):
    cfg = bench.CONFIGS[name]
    hq = cfg["hq"]
    g = bench.geometry(cfg, hosts)
    d = hq * bench.DH
    zz = [bench.attn_flops_host(g, hq, h, True) for h in range(hosts)]
    nv = [bench.attn_flops_host(g, hq, h, False) for h in range(hosts)]
    # the B.2 subset (everything but block->anchor and the query terms) is identical per host
    for h in range(hosts):
        a0, a1 = spava.slice_anchor(g["l_a"], hosts, h)
        extra = (8 * g["l_a"] * g["l_b"] + 4 * g["n_t"] * ((a1 - a0) + 2 * g["l_b"]) +
                 (2 * g["n_t"] ** 2 if h == hosts - 1 else 0)) * d
        assert zz[h] - extra == ref_attn_flops_per_host(g["l_a"], g["l_b"], g["l_p"], hosts, d)
    assert max(nv) / min(nv) > 1.05 and max(zz) / min(zz) < 1.01


@pytest.mark.parametrize("n,want", [(1, "C1"), (2, "C1"), (4, "C2"), (8, "C3")])
def test_default_workload_per_gpu_count(n, want):
    """bench.py's default job at N GPUs is the BASELINE config quoted at that count
    (configs[1] C1 at 1 / 2, configs[2] C2 at 4, configs[3] C3 at 8), split over N hosts."""
    import argparse

    args = argparse.Namespace(config=None, gpus=n)
    name, cfg, g = bench.job_config(args, n)
    assert name == want and cfg is bench.CONFIGS[want] and g["hosts"] == n
    assert bench.job_config(argparse.Namespace(config="C4", gpus=n), n)[0] == "C4"
