"""Shared helpers for the parity tests (host-side only)."""
from __future__ import annotations

import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def bf16(x):
    """fp32 -> nearest-even bf16 -> fp32 (numpy)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def from_bits(b):
    return (np.asarray(b).astype(np.uint32) << 16).view(np.float32)


def randn(rng, *shape, scale=1.0):
    return bf16(rng.standard_normal(shape).astype(np.float32) * scale)


def load_golden(name):
    d = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    for k in ("Q", "K", "V"):
        if k in d and d[k].dtype == np.uint16:
            d[k] = from_bits(d[k])
    return d


def host_local(X, l_a, l_b, lo, hi, qoff, n_t):
    """Global padded rows -> host-local [anchor | block lo | block hi | query]."""
    return np.concatenate([X[:l_a], X[l_a + lo * l_b:l_a + (lo + 1) * l_b],
                           X[l_a + hi * l_b:l_a + (hi + 1) * l_b], X[qoff:qoff + n_t]])


def max_abs(a, b):
    return float(np.max(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)))) if np.size(a) else 0.0


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / d) if d > 0 else float(np.linalg.norm(a - b))


def ulp_diff(a, b):
    """Max distance in float32 ulps between finite arrays (inf == inf counts 0)."""
    a = np.asarray(a, np.float32)
    b = np.asarray(b, np.float32)
    same = (a == b)
    ia = a.view(np.int32).astype(np.int64)
    ib = b.view(np.int32).astype(np.int64)
    ia = np.where(ia < 0, -(ia & 0x7FFFFFFF), ia)
    ib = np.where(ib < 0, -(ib & 0x7FFFFFFF), ib)
    d = np.where(same, 0, np.abs(ia - ib))
    return int(d.max()) if d.size else 0


# Tolerances of the bf16 attention path against the fp32 oracle (stated in DESIGN.md):
# P is rounded to bf16 before P.V and outputs are bf16 -> ~2^-9 relative per element.
ATOL_BF16_OUT = 2.5e-2   # max-abs on bf16 outputs
RTOL_L2_BF16 = 6e-3      # relative L2 on bf16 outputs
ATOL_F32_OUT = 1.5e-2    # max-abs on f32 partial outputs (bf16 P)
RTOL_L2_F32 = 5e-3
ATOL_LSE = 2e-3          # lse (natural log) abs error
