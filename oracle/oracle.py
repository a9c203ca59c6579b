"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY.

numpy/ctypes front end for the two CPU checkers of the Spava hot path:

* ``impl="c"``   -- oracle/liboracle.so, the plain-C restatement
                    (oracle/spava_oracle.c, each routine cites its reference line).
* ``impl="ref"`` -- oracle/_ref/libseqpar_ref.so, the UNMODIFIED reference
                    operators (/root/reference/proj/core/src/*.cpp) behind
                    oracle/ref_shim.cpp.  The reference has no GQA, so K/V heads
                    are repeated before the call (exact: SURVEY.md s0).

Nothing in paper_2601_21444_b200/ imports this module; only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline leg do.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_F = C.POINTER(C.c_float)
_I = C.POINTER(C.c_int)
_U8 = C.POINTER(C.c_uint8)


class OracleError(RuntimeError):
    pass


class _Seg(C.Structure):  # orc_mseg / ref_seg share this layout
    _fields_ = [("k", _F), ("v", _F), ("rows", C.c_int), ("causal", C.c_int), ("pad", _U8)]


class _LayerCfg(C.Structure):
    _fields_ = [(n, C.c_int) for n in (
        "n_v", "n_t", "hosts", "l_a", "l_p", "zigzag", "designated", "hq", "hkv", "dh",
        "softmax_scores", "query_self_all")]


_libs: dict = {}


def lib(impl: str = "c"):
    if impl not in _libs:
        path = (os.path.join(HERE, "liboracle.so") if impl == "c"
                else os.path.join(HERE, "_ref", "libseqpar_ref.so"))
        if not os.path.exists(path):
            raise OracleError(f"oracle library {path} not built (run `make -C oracle`)")
        L = C.CDLL(path)
        pre = "orc_" if impl == "c" else "ref_"
        L.last_error = getattr(L, pre + "last_error")
        L.last_error.restype = C.c_char_p
        _libs[impl] = L
    return _libs[impl]


def available(impl: str) -> bool:
    try:
        lib(impl)
        return True
    except OracleError:
        return False


def _f(a):
    return a.ctypes.data_as(_F) if a is not None else None


def _i(a):
    return a.ctypes.data_as(_I) if a is not None else None


def _u8(a):
    return a.ctypes.data_as(_U8) if a is not None else None


def _c32(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float32)


def _cu8(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.uint8)


def _check(rc, L, what):
    if rc != 0:
        raise OracleError(f"{what}: rc={rc}: {L.last_error().decode()}")


def expand_kv(x: np.ndarray, hq: int, hkv: int, dh: int) -> np.ndarray:
    """[rows, hkv*dh] -> [rows, hq*dh] repeating each kv head hq/hkv times."""
    if hq == hkv:
        return np.ascontiguousarray(x, dtype=np.float32)
    g = hq // hkv
    r = x.reshape(x.shape[0], hkv, 1, dh)
    return np.ascontiguousarray(np.broadcast_to(r, (x.shape[0], hkv, g, dh)).reshape(x.shape[0], hq * dh),
                                dtype=np.float32)


# ------------------------------------------------------------------ partition
def virtual_pair(hosts, zigzag, h, impl="c"):
    L = lib(impl)
    lo, hi = C.c_int(), C.c_int()
    fn = L.orc_virtual_pair if impl == "c" else L.ref_virtual_pair
    _check(fn(hosts, int(zigzag), h, C.byref(lo), C.byref(hi)), L, "virtual_pair")
    return lo.value, hi.value


def physical_of(hosts, zigzag, v, impl="c"):
    L = lib(impl)
    h = C.c_int()
    fn = L.orc_physical_of if impl == "c" else L.ref_physical_of
    _check(fn(hosts, int(zigzag), v, C.byref(h)), L, "physical_of")
    return h.value


def split_geometry(n_v, n_t, hosts, l_a, l_p, impl="c"):
    L = lib(impl)
    lb, pad, qoff = C.c_int(), C.c_int(), C.c_int()
    fn = L.orc_split_geometry if impl == "c" else L.ref_split_geometry
    _check(fn(n_v, n_t, hosts, l_a, l_p, C.byref(lb), C.byref(pad), None, None, C.byref(qoff)), L,
           "split_geometry")
    offs = np.zeros(2 * hosts, np.int32)
    masks = np.zeros((2 * hosts, max(lb.value, 1)), np.uint8)
    fn(n_v, n_t, hosts, l_a, l_p, C.byref(lb), C.byref(pad), _i(offs), _u8(masks), C.byref(qoff))
    return dict(l_b=lb.value, pad=pad.value, offsets=offs, pad_masks=masks[:, :lb.value],
                query_offset=qoff.value)


def slice_anchor(l_a, hosts, h, impl="c"):
    L = lib(impl)
    b, e = C.c_int(), C.c_int()
    fn = L.orc_slice_anchor if impl == "c" else L.ref_slice_anchor
    _check(fn(l_a, hosts, h, C.byref(b), C.byref(e)), L, "slice_anchor")
    return b.value, e.value


def default_plan(n, hosts, impl="c"):
    L = lib(impl)
    la, lb, lp, pad = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    fn = L.orc_default_plan if impl == "c" else L.ref_default_plan
    _check(fn(n, hosts, C.byref(la), C.byref(lb), C.byref(lp), C.byref(pad)), L, "default_plan")
    return dict(l_a=la.value, l_b=lb.value, l_p=lp.value, pad=pad.value)


# -------------------------------------------------------------------- scoring
def score_context(q, k, scale, pad=None, softmax=True, impl="c"):
    q, k, pad = _c32(q), _c32(k), _cu8(pad)
    L = lib(impl)
    out = np.zeros(k.shape[0], np.float32)
    fn = L.orc_score_context if impl == "c" else L.ref_score_context
    fn.argtypes = [_F, C.c_int, _F, C.c_int, C.c_int, C.c_float, _U8, C.c_int, _F]
    _check(fn(_f(q), q.shape[0], _f(k), k.shape[0], q.shape[1], scale, _u8(pad), int(softmax),
              _f(out)), L, "score_context")
    return out


def score_block(q, k, hq, hkv, dh, pad=None, softmax=True, impl="c"):
    """score_block (simhost.cpp:209-224). q: [n_t, hq*dh], k: [l_b, hkv*dh]."""
    q, k, pad = _c32(q), _c32(k), _cu8(pad)
    L = lib(impl)
    out = np.zeros(k.shape[0], np.float32)
    if impl == "c":
        _check(L.orc_score_block(_f(q), q.shape[0], _f(k), k.shape[0], hq, hkv, dh, _u8(pad),
                                 int(softmax), _f(out)), L, "score_block")
    else:
        ke = expand_kv(k, hq, hkv, dh)
        _check(L.ref_score_block(_f(q), q.shape[0], _f(ke), k.shape[0], hq, dh, _u8(pad),
                                 int(softmax), _f(out)), L, "score_block")
    return out


def select_essential(scores, l_p, global_offset=0, impl="c"):
    """select_essential (approx.cpp:71-102) -> int32 global indices, ascending."""
    s = _c32(scores)
    L = lib(impl)
    idx = np.zeros(max(len(s), 1), np.int32)
    cnt = C.c_int()
    if impl == "c":
        _check(L.orc_select_essential(_f(s), len(s), l_p, global_offset, _i(idx), C.byref(cnt)), L,
               "select_essential")
    else:
        _check(L.ref_select_essential(None, None, len(s), 1, _f(s), l_p, global_offset, _i(idx),
                                      None, None, C.byref(cnt)), L, "select_essential")
    return idx[:cnt.value].copy()


# ------------------------------------------------------------------ attention
def _segs(segs, hq, hkv, dh, impl, keep):
    arr = (_Seg * max(len(segs), 1))()
    for n, s in enumerate(segs):
        k, v = _c32(s["k"]), _c32(s["v"])
        if impl == "ref":
            k, v = expand_kv(k, hq, hkv, dh), expand_kv(v, hq, hkv, dh)
        pad = _cu8(s.get("pad"))
        keep += [k, v, pad]
        arr[n].k, arr[n].v = _f(k), _f(v)
        arr[n].rows = k.shape[0]
        arr[n].causal = int(s.get("causal", False))
        arr[n].pad = _u8(pad)
    return arr


def mha_lse(q, segs, hq, hkv, dh, allow_invalid=False, impl="c"):
    """mha_lse (attention.cpp:158-178). segs: list of dict(k, v, causal, pad)."""
    q = _c32(q)
    L = lib(impl)
    keep = []
    arr = _segs(segs, hq, hkv, dh, impl, keep)
    out = np.zeros((q.shape[0], hq * dh), np.float32)
    lse = np.zeros((q.shape[0], hq), np.float32)
    if impl == "c":
        rc = L.orc_mha_lse(_f(q), q.shape[0], hq, hkv, dh, arr, len(segs), int(allow_invalid),
                           _f(out), _f(lse))
    else:
        rc = L.ref_mha_lse(_f(q), q.shape[0], hq * dh, hq, arr, len(segs), int(allow_invalid),
                           _f(out), _f(lse))
    _check(rc, L, "mha_lse")
    return out, lse


def attention_lse(q, segs, scale, allow_invalid=False, impl="c"):
    """attention_lse (attention.cpp:18-86), single head, explicit scale."""
    q = _c32(q)
    L = lib(impl)
    keep = []
    d = q.shape[1]
    arr = _segs(segs, 1, 1, d, "c", keep)
    out = np.zeros((q.shape[0], d), np.float32)
    lse = np.zeros(q.shape[0], np.float32)
    fn = L.orc_attention_lse if impl == "c" else L.ref_attention_lse
    fn.argtypes = [_F, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_float, C.c_int, _F, _F]
    _check(fn(_f(q), q.shape[0], d, C.cast(arr, C.c_void_p), len(segs), scale, int(allow_invalid),
              _f(out), _f(lse)), L, "attention_lse")
    return out, lse


def mha_merge(outs, lses, hq, dh, impl="c"):
    """mha_merge (attention.cpp:180-197) over parts in host order."""
    outs = [_c32(o) for o in outs]
    lses = [_c32(l) for l in lses]
    L = lib(impl)
    n = len(outs)
    po = (_F * n)(*[_f(o) for o in outs])
    pl = (_F * n)(*[_f(l) for l in lses])
    rows = outs[0].shape[0]
    out = np.zeros((rows, hq * dh), np.float32)
    if impl == "c":
        rc = L.orc_mha_merge(n, po, pl, rows, hq, dh, _f(out))
    else:
        rc = L.ref_mha_merge(n, po, pl, rows, hq * dh, hq, _f(out))
    _check(rc, L, "mha_merge")
    return out


def merge_partials(outs, lses, impl="c"):
    outs = [_c32(o) for o in outs]
    lses = [_c32(l) for l in lses]
    L = lib(impl)
    n = len(outs)
    po = (_F * n)(*[_f(o) for o in outs])
    pl = (_F * n)(*[_f(l) for l in lses])
    rows, d = outs[0].shape
    out = np.zeros((rows, d), np.float32)
    fn = L.orc_merge_partials if impl == "c" else L.ref_merge_partials
    _check(fn(n, po, pl, rows, d, _f(out)), L, "merge_partials")
    return out


def block_attention(q, k, v, pad, k_a, v_a, k_p, v_p, hq, hkv, dh, impl="c"):
    """block_attention (approx.cpp:140-154) with the passing set pre-assembled."""
    segs = []
    if k_a is not None and len(k_a):
        segs.append(dict(k=k_a, v=v_a))
    if k_p is not None and len(k_p):
        segs.append(dict(k=k_p, v=v_p))
    segs.append(dict(k=k, v=v, causal=True, pad=pad))
    return mha_lse(q, segs, hq, hkv, dh, allow_invalid=True, impl=impl)[0]


def anchor_attention(q, k, v, hq, hkv, dh, impl="c"):
    return mha_lse(q, [dict(k=k, v=v, causal=True)], hq, hkv, dh, impl=impl)[0]


def query_attention(q, k_a, v_a, a0, a1, k_lo, v_lo, pad_lo, k_hi, v_hi, pad_hi, k_q, v_q,
                    include_self, hq, hkv, dh, impl="c"):
    """query_attention (approx.cpp:156-188) -> (out, lse)."""
    segs = []
    if a1 > a0:
        segs.append(dict(k=k_a[a0:a1], v=v_a[a0:a1]))
    segs.append(dict(k=k_lo, v=v_lo, pad=pad_lo))
    segs.append(dict(k=k_hi, v=v_hi, pad=pad_hi))
    if include_self:
        segs.append(dict(k=k_q, v=v_q, causal=True))
    return mha_lse(q, segs, hq, hkv, dh, allow_invalid=True, impl=impl)


def spava_layer(Q, K, V, n_v, n_t, hosts, l_a, l_p, hq, hkv, dh, zigzag=True, designated=-1,
                softmax_scores=True, query_self_all=False):
    """Whole Spava layer for all hosts (C oracle; run_host order simhost.cpp:321-426)."""
    L = lib("c")
    g = split_geometry(n_v, n_t, hosts, l_a, l_p)
    lb, VH = g["l_b"], 2 * hosts
    cfg = _LayerCfg(n_v, n_t, hosts, l_a, l_p, int(zigzag), designated, hq, hkv, dh,
                    int(softmax_scores), int(query_self_all))
    Q, K, V = _c32(Q), _c32(K), _c32(V)
    sel = np.zeros((VH, max(l_p, 1)), np.int32)
    cnt = np.zeros(VH, np.int32)
    anchor = np.zeros((l_a, hq * dh), np.float32)
    blocks = np.zeros((VH, lb, hq * dh), np.float32)
    query = np.zeros((n_t, hq * dh), np.float32)
    qpo = np.zeros((hosts, n_t, hq * dh), np.float32)
    qpl = np.zeros((hosts, n_t, hq), np.float32)
    _check(L.orc_spava_layer(C.byref(cfg), _f(Q), _f(K), _f(V), _i(sel), _i(cnt), _f(anchor),
                             _f(blocks), _f(query), _f(qpo), _f(qpl)), L, "spava_layer")
    return dict(sel=sel[:, :l_p], sel_count=cnt, anchor=anchor, blocks=blocks, query=query,
                qpart_out=qpo, qpart_lse=qpl, geometry=g)
