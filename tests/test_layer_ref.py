"""oracle/layer_ref.py (the full-size checker and the reference arm's work items) on the CPU:
the row-slice x head decomposition of a whole layer through the UNMODIFIED reference
operators is bit-identical to the C oracle's whole-layer run (orc_spava_layer, run_host
order) -- selections, every block row, the anchor and the merged query -- so the
decomposition is an exact restatement, not an approximation.  Also: bench.py's
reference arm runs one whole (small) layer split over its steps."""
import numpy as np
import pytest

import bench
from oracle import layer_ref as LR
from oracle import oracle as O


@pytest.mark.parametrize("hosts,zigzag", [(2, True), (3, True), (2, False)])
def test_row_slices_equal_whole_layer(hosts, zigzag):
    n_v, n_t, l_a, l_p, hq, hkv, dh = 1021, 32, 16, 24, 4, 2, 128
    g = LR.geometry(n_v, n_t, hosts, l_a, l_p, zigzag)
    Q, K, V = LR.layer_inputs(g, hq, hkv, dh, seed=3)
    want = O.spava_layer(Q, K, V, n_v, n_t, hosts, l_a, l_p, hq, hkv, dh, zigzag=zigzag)
    ref = LR.LayerRef(Q, K, V, g, hq, hkv, dh)
    LR.run_items(ref.run_item, ref.score_items(), 4)
    ref.finish_scores()
    for v in range(2 * hosts):
        assert np.array_equal(ref.sel[v], want["sel"][v][:want["sel_count"][v]]), v
    rows_b = {v: range(LR.valid_rows(g, v)) for v in range(2 * hosts)}
    LR.run_items(ref.run_item, ref.attention_items(range(l_a), rows_b, range(n_t), m=5), 4)
    a, _ = ref.rows("anchor", 0, range(l_a))
    assert np.array_equal(a, want["anchor"])
    for v in range(2 * hosts):
        nv = LR.valid_rows(g, v)
        b, _ = ref.rows("block", v, range(nv))
        assert np.array_equal(b, want["blocks"][v][:nv]), v
    assert np.array_equal(ref.query_rows(range(n_t)), want["query"])


def test_reference_arm_runs_whole_layer_over_steps():
    g = LR.geometry(1021, 32, 2, 16, 24)
    g["n"] = g["n_v"] + g["n_t"]
    r = bench.reference_job(g, 4, 2, steps=5, warmup=1, threads=2, max_s=1e9, m=32)
    assert r["frac"] == pytest.approx(1.0)
    assert len(r["step_s"]) == 5 and r["value"] > 0
    r2 = bench.reference_job(g, 4, 2, steps=3, warmup=0, threads=2, max_s=1e-4, m=8)
    assert r2["frac"] < 1.0 and "extrapolated" in r2["sample"]
