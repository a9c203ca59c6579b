"""CPU tests of the C-ABI host logic (plan / topology / exchange-slot mapping) in
libspava_b200.so against the reference's test_partition.cpp pins and the oracle.
These entry points are pure host code: no GPU is needed."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2601_21444_b200 import spava


def test_zigzag_pairs():
    """test_partition.cpp:42-52"""
    p = spava.make_plan(100, 0, 4, 4, 0)
    assert [spava.virtual_pair(p, h) for h in range(4)] == [(0, 7), (1, 6), (2, 5), (3, 4)]
    assert spava.virtual_pair(spava.make_plan(100, 0, 1, 4, 0), 0) == (0, 1)
    p2 = spava.make_plan(100, 0, 2, 4, 0)
    assert spava.virtual_pair(p2, 0) == (0, 3) and spava.virtual_pair(p2, 1) == (1, 2)
    with pytest.raises(spava.SpavaError):
        spava.virtual_pair(p, 4)


@pytest.mark.parametrize("hosts", range(1, 10))
def test_pairing_bijection(hosts):
    """test_partition.cpp:54-69"""
    for zz in (True, False):
        p = spava.make_plan(1000, 0, hosts, 4, 0, zz)
        seen = np.zeros(2 * hosts, int)
        for h in range(hosts):
            lo, hi = spava.virtual_pair(p, h)
            seen[lo] += 1
            seen[hi] += 1
            assert spava.physical_of(p, lo) == h and spava.physical_of(p, hi) == h
            assert (lo, hi) == O.virtual_pair(hosts, zz, h)
            if zz:
                assert lo + hi == 2 * hosts - 1
        assert (seen == 1).all()


def test_split_geometry():
    """test_partition.cpp:71-87"""
    p = spava.make_plan(20, 3, 2, 4, 0)
    assert p.pad == 0 and p.l_b == 4
    assert [spava.block_offset(p, v) for v in range(4)] == [4, 8, 12, 16]
    p = spava.make_plan(21, 3, 2, 4, 0)
    assert p.pad == 3 and p.l_b == 5
    assert spava.pad_mask(p, 3).tolist() == [0, 0, 1, 1, 1]
    assert spava.query_offset(p) == 24
    with pytest.raises(spava.SpavaError):
        spava.make_plan(4, 3, 2, 4, 0)  # l_a >= n_v
    with pytest.raises(spava.SpavaError):
        spava.make_plan(20, 3, 2, 4, 9)  # l_p > l_b


def test_split_sweep_vs_oracle():
    """test_partition.cpp:89-120 round-trip geometry, against the oracle."""
    rng = np.random.default_rng(3)
    for _ in range(60):
        n_v, hosts = int(rng.integers(8, 121)), int(rng.integers(1, 5))
        l_a = int(rng.integers(0, n_v))
        p = spava.make_plan(n_v, 2, hosts, l_a, 0)
        g = O.split_geometry(n_v, 2, hosts, l_a, 0)
        assert p.l_b == g["l_b"] and p.pad == g["pad"]
        assert p.l_a + p.virtual_hosts * p.l_b == p.n_v + p.pad and p.pad < p.virtual_hosts
        for v in range(2 * hosts):
            assert spava.block_offset(p, v) == g["offsets"][v]
            assert np.array_equal(spava.pad_mask(p, v), g["pad_masks"][v])
            assert spava.block_valid_rows(p, v) == int((g["pad_masks"][v] == 0).sum())


def test_frame_partition():
    """test_partition.cpp:23-28 pins; sums and balance (acceptance.cpp:186-195, Eq. 6)"""
    assert spava.frame_partition(64, 8) == [8] * 8
    assert spava.frame_partition(10, 3) == [4, 3, 3]
    assert spava.frame_partition(7, 8) == [1, 1, 1, 1, 1, 1, 1, 0]
    with pytest.raises(spava.SpavaError):
        spava.frame_partition(4, 0)
    for f in range(0, 40):
        for h in range(1, 9):
            c = spava.frame_partition(f, h)
            assert sum(c) == f and max(c) - min(c) <= 1 and c == sorted(c, reverse=True)


def test_slice_anchor():
    """test_partition.cpp:122-144"""
    assert spava.slice_anchor(8, 4, 0) == (0, 2) and spava.slice_anchor(8, 4, 3) == (6, 8)
    assert spava.slice_anchor(5, 2, 0) == (0, 3) and spava.slice_anchor(5, 2, 1) == (3, 5)
    assert spava.slice_anchor(10, 1, 0) == (0, 10)
    with pytest.raises(spava.SpavaError):
        spava.slice_anchor(8, 4, 4)
    for l_a in range(21):
        for hosts in range(1, 7):
            e = 0
            for h in range(hosts):
                b, en = spava.slice_anchor(l_a, hosts, h)
                assert b == e and (b, en) == O.slice_anchor(l_a, hosts, h)
                e = en
            assert e == l_a


def test_default_plan():
    """test_partition.cpp:146-159"""
    p = spava.default_plan(8192, 4)
    assert p.l_a == 128 and p.l_p == 64
    p = spava.default_plan(128, 2)
    assert p.l_a == 2 and p.l_p == 1
    with pytest.raises(spava.SpavaError):
        spava.default_plan(64, 2)
    p = spava.default_plan(1024, 32)
    assert p.l_p == min(1024 // 128, p.l_b)
    assert O.default_plan(8192, 4)["l_b"] == spava.default_plan(8192, 4).l_b


@pytest.mark.parametrize("hosts", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("zigzag", [True, False])
def test_passing_ranges_are_assemble_passing(hosts, zigzag):
    """assemble_passing (approx.cpp:104-132): block v sees exactly the sources < v.
    Round 0 slot s carries host s's lo block, round 1 slot s its hi block."""
    p = spava.make_plan(10 * hosts + 5, 2, hosts, 5, 1, zigzag)
    for v in range(2 * hosts):
        (a0, a1), (b0, b1) = spava.passing_ranges(p, v)
        srcs = [spava.virtual_pair(p, s)[0] for s in range(a0, a1)] + \
               [spava.virtual_pair(p, s)[1] for s in range(b0, b1)]
        assert sorted(srcs) == list(range(v)), (v, srcs)
    # per physical host the passing budget is (2H-1) * l_p under zigzag (test_approx.cpp:148-154)
    if zigzag:
        for h in range(hosts):
            lo, hi = spava.virtual_pair(p, h)
            n = sum(e - b for rng in (spava.passing_ranges(p, lo), spava.passing_ranges(p, hi))
                    for b, e in rng)
            assert n == 2 * hosts - 1
