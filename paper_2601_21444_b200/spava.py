"""ctypes binding of include/spava_b200.h + a Python mirror of the reference API.

Names and argument meanings follow the reference ``seqpar`` operators
(/root/reference/proj/core/include/seqpar/{partition,approx,attention}.hpp) so the
parity tests read like the reference's own doctest suites.  Tensors are torch CUDA
tensors: Q/K/V bf16 token-major [rows, heads*dh]; scores/partials f32.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# SPAVA_LIB: dev-only override (A/B timing of two builds of the same C ABI)
LIB_PATH = os.environ.get("SPAVA_LIB") or os.path.join(HERE, "libspava_b200.so")

__all__ = [
    "SpavaError", "lib", "Plan", "LayerConfig", "Fabric", "Host", "make_plan", "default_plan",
    "virtual_pair", "physical_of", "slice_anchor", "block_offset", "query_offset", "pad_mask",
    "block_valid_rows", "passing_ranges", "score_block", "select_pack", "select_essential", "attention",
    "mha_merge", "anchor_attention", "block_attention", "query_attention", "nccl_unique_id",
    "kernel_launches", "device_ok", "EXPORTED_SYMBOLS", "gemm",
]

EINVAL, ERANGE, ERUNTIME, ECUDA, ENCCL = 1, 2, 3, 4, 5

EXPORTED_SYMBOLS = [
    "spava_last_error", "spava_version", "spava_device_ok", "spava_make_plan",
    "spava_default_plan", "spava_virtual_pair", "spava_physical_of", "spava_slice_anchor",
    "spava_block_offset", "spava_query_offset", "spava_pad_mask", "spava_block_valid_rows",
    "spava_passing_ranges", "spava_split_rows", "spava_merge_rows",
    "spava_score_workspace", "spava_score_block", "spava_score_block_ex", "spava_score_fast_workspace",
    "spava_score_block_fast", "spava_select_pack",
    "spava_attention_workspace", "spava_attention", "spava_attention_ex", "spava_mha_merge",
    "spava_fabric_create_local", "spava_nccl_unique_id", "spava_fabric_create_nccl",
    "spava_fabric_create_peer", "spava_fabric_peer_handle", "spava_fabric_peer_open",
    "spava_fabric_peer_attach", "spava_frame_partition", "spava_gather_split_rows",
    "spava_fabric_encode_region", "spava_fabric_encode_acquire", "spava_host_gather_context",
    "spava_fabric_destroy", "spava_host_create", "spava_host_destroy", "spava_host_plan",
    "spava_host_rows", "spava_host_layer", "spava_host_layer_hostbuf", "spava_sim_layer",
    "spava_sim_layer_timed", "spava_host_set_trace", "spava_host_trace_read",
    "spava_host_capture_layer", "spava_host_replay_layer", "spava_host_set_delay",
    "spava_decoder_workspace", "spava_host_decoder_layer", "spava_gemm",
    "spava_host_status",
    "spava_host_set_timing", "spava_host_timing", "spava_kernel_launches",
    "spava_debug_attn_prof", "spava_debug_attn_variant", "spava_debug_fused_merge", "spava_debug_fused_score",
]


class SpavaError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[spava status {code}] {msg}")
        self.code = code


class Plan(C.Structure):
    _fields_ = [(n, C.c_int) for n in (
        "n_v", "n_t", "hosts", "l_a", "l_b", "l_p", "pad", "virtual_hosts", "zigzag")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class _Segment(C.Structure):
    _fields_ = [("k", C.c_void_p), ("v", C.c_void_p), ("ld", C.c_int64), ("rows", C.c_int),
                ("causal", C.c_int)]


class TraceEvent(C.Structure):
    _fields_ = [("kind", C.c_int), ("layer", C.c_int), ("label", C.c_char * 16), ("tag", C.c_char * 24),
                ("t_us", C.c_double)]


# seqpar::EventKind names as written to JSONL (simhost.cpp:19-37)
EVENT_KINDS = ("comm_issued", "comm_wait_start", "comm_completed", "compute_begin", "compute_end")


def trace_events(records_per_host):
    """Reference EventTrace (simhost.hpp:28-40) from per-host program-order records:
    per-host seq, Lamport clocks as HostRecorder::record (simhost.cpp:168-179) with a
    completion merging the max issuing clock of all contributors (GatherFabric::wait),
    global order by (clock, host, seq) (simhost.cpp:549-560).  Each event keeps the device
    timestamp as an extra 't_us' field (ignored by the reference reader)."""
    issue_clock = {}
    per_host = []
    for h, recs in enumerate(records_per_host):
        clock, evs = 0, []
        for seq, (kind, label, layer, tag, t_us) in enumerate(recs):
            evs.append(dict(host=h, seq=seq, kind=EVENT_KINDS[kind], label=label, layer=layer,
                            tag=tag, t_us=round(t_us, 3)))
        per_host.append(evs)
    # a completion's clock depends on the other hosts' issue clocks, which (across layers)
    # depend on earlier completions: iterate the per-host sweeps to the fixpoint
    while True:
        changed = False
        for evs in per_host:
            clock = 0
            for e in evs:
                merge = issue_clock.get(e["tag"], 0) if e["kind"] == "comm_completed" else 0
                clock = max(clock, merge) + 1
                e["clock"] = clock
                if e["kind"] == "comm_issued" and issue_clock.get(e["tag"], 0) < clock:
                    issue_clock[e["tag"]] = clock
                    changed = True
        if not changed:
            break
    events = sorted((e for evs in per_host for e in evs), key=lambda e: (e["clock"], e["host"], e["seq"]))
    for i, e in enumerate(events):
        e["global_index"] = i
    return events


def trace_jsonl(events):
    import json

    keys = ("global_index", "host", "seq", "kind", "label", "layer", "tag", "clock", "t_us")
    return "".join(json.dumps({k: e[k] for k in keys}) + "\n" for e in events)


class DecoderWeights(C.Structure):
    """spava_decoder_weights: device pointers of the decoder layer around the path."""
    _fields_ = [("w_qkv", C.c_void_p), ("w_o", C.c_void_p), ("w_1", C.c_void_p), ("w_2", C.c_void_p),
                ("g_1", C.c_void_p), ("g_2", C.c_void_p), ("d_model", C.c_int), ("ffn", C.c_int),
                ("norm", C.c_int)]


class LayerConfig(C.Structure):
    _fields_ = [(n, C.c_int) for n in (
        "n_v", "n_t", "hosts", "l_a", "l_p", "zigzag", "designated", "query_self_all",
        "softmax_scores", "hq", "hkv", "dh", "query_splits", "score_mode")]

    @classmethod
    def make(cls, n_v, n_t, hosts, l_a, l_p, hq, hkv, dh=128, zigzag=True, designated=-1,
             query_self_all=False, softmax_scores=True, query_splits=0, score_mode=0):
        """score_mode 0 = exact (bit-faithful scorer), 1 = fast (tensor-core scorer)."""
        return cls(n_v, n_t, hosts, l_a, l_p, int(zigzag), designated, int(query_self_all),
                   int(softmax_scores), hq, hkv, dh, query_splits, int(score_mode))


_lib = None


def lib():
    """Load libspava_b200.so; raises (no fallback) if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SpavaError(ECUDA, f"{LIB_PATH} missing: build it with __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        L.spava_last_error.restype = C.c_char_p
        L.spava_version.restype = C.c_char_p
        L.spava_score_workspace.restype = C.c_size_t
        L.spava_score_workspace.argtypes = [C.c_int, C.c_int, C.c_int]
        L.spava_score_fast_workspace.restype = C.c_size_t
        L.spava_score_fast_workspace.argtypes = [C.c_int, C.c_int, C.c_int]
        L.spava_score_block_fast.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_int64,
                                             C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                             C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
        L.spava_attention_workspace.restype = C.c_size_t
        L.spava_attention_workspace.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int]
        L.spava_gemm.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                 C.c_void_p, C.c_int64, C.c_float, C.c_int, C.c_void_p]
        L.spava_kernel_launches.restype = C.c_uint64
        L.spava_score_block.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_int64,
                                        C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
        L.spava_select_pack.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                        C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.spava_attention.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_int,
                                      C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_int,
                                      C.c_void_p, C.c_int, C.c_void_p, C.c_size_t, C.c_void_p]
        L.spava_mha_merge.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int64,
                                      C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_int,
                                      C.c_void_p, C.c_void_p, C.c_void_p]
        L.spava_host_layer.argtypes = [C.c_void_p] * 7
        L.spava_host_layer_hostbuf.argtypes = [C.c_void_p] * 12
        L.spava_sim_layer.argtypes = [C.c_void_p] * 8
        L.spava_sim_layer_timed.argtypes = [C.c_void_p] * 9
        L.spava_host_set_trace.argtypes = [C.c_void_p, C.c_int]
        L.spava_host_capture_layer.argtypes = [C.c_void_p] * 7
        L.spava_host_replay_layer.argtypes = [C.c_void_p, C.c_void_p]
        L.spava_host_set_delay.argtypes = [C.c_void_p, C.c_int, C.c_uint64]
        L.spava_decoder_workspace.restype = C.c_size_t
        L.spava_decoder_workspace.argtypes = [C.c_void_p, C.c_void_p]
        L.spava_host_decoder_layer.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                               C.c_size_t, C.c_void_p]
        L.spava_debug_attn_variant.argtypes = [C.c_int]
        L.spava_debug_fused_merge.argtypes = [C.c_int]
        L.spava_debug_fused_score.argtypes = [C.c_int]
        L.spava_split_rows.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                       C.c_int, C.c_void_p]
        L.spava_merge_rows.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                       C.c_int, C.c_int, C.c_void_p]
        L.spava_fabric_create_peer.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_void_p]
        L.spava_frame_partition.argtypes = [C.c_int, C.c_int, C.c_void_p]
        L.spava_gather_split_rows.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int64,
                                              C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int,
                                              C.c_void_p]
        L.spava_fabric_encode_region.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.spava_fabric_encode_acquire.argtypes = [C.c_void_p, C.c_void_p]
        L.spava_host_gather_context.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                                C.c_void_p, C.c_int64, C.c_int, C.c_void_p]
        L.spava_host_trace_read.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
        L.spava_host_create.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.spava_host_destroy.argtypes = [C.c_void_p]
        L.spava_host_rows.argtypes = [C.c_void_p]
        L.spava_host_plan.argtypes = [C.c_void_p, C.c_void_p]
        L.spava_host_status.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.spava_host_set_timing.argtypes = [C.c_void_p, C.c_int]
        L.spava_host_timing.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.spava_fabric_destroy.argtypes = [C.c_void_p]
        L.spava_fabric_create_local.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.spava_fabric_create_nccl.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int,
                                               C.c_void_p]
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise SpavaError(rc, lib().spava_last_error().decode())


def device_ok() -> bool:
    return bool(lib().spava_device_ok())


def kernel_launches() -> int:
    return int(lib().spava_kernel_launches())


def _stream(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _require(t, dtype, name):
    import torch

    if t.device.type != "cuda":
        raise SpavaError(EINVAL, f"{name}: expected a CUDA tensor (there is no CPU path)")
    if t.dtype != dtype:
        raise SpavaError(EINVAL, f"{name}: expected {dtype}, got {t.dtype}")
    if t.dim() != 2 or t.stride(1) != 1:
        raise SpavaError(EINVAL, f"{name}: expected a row-major 2-D tensor")
    _ = torch


# ------------------------------------------------------------------ partition
def make_plan(n_v, n_t, hosts, l_a, l_p, zigzag=True) -> Plan:
    """split_context geometry (partition.cpp:40-85)."""
    p = Plan()
    _check(lib().spava_make_plan(n_v, n_t, hosts, l_a, l_p, int(zigzag), C.byref(p)))
    return p


def default_plan(n, hosts) -> Plan:
    """default_plan (partition.cpp:96-113)."""
    p = Plan()
    _check(lib().spava_default_plan(n, hosts, C.byref(p)))
    return p


def virtual_pair(plan: Plan, h):
    lo, hi = C.c_int(), C.c_int()
    _check(lib().spava_virtual_pair(C.byref(plan), h, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def physical_of(plan: Plan, v):
    h = C.c_int()
    _check(lib().spava_physical_of(C.byref(plan), v, C.byref(h)))
    return h.value


def slice_anchor(l_a, hosts, h):
    b, e = C.c_int(), C.c_int()
    _check(lib().spava_slice_anchor(l_a, hosts, h, C.byref(b), C.byref(e)))
    return b.value, e.value


def block_offset(plan: Plan, v):
    return lib().spava_block_offset(C.byref(plan), v)


def query_offset(plan: Plan):
    return lib().spava_query_offset(C.byref(plan))


def block_valid_rows(plan: Plan, v):
    return lib().spava_block_valid_rows(C.byref(plan), v)


def passing_ranges(plan: Plan, v):
    """Exchange slots holding the sources < v: ((r0_begin, r0_end), (r1_begin, r1_end))."""
    a, b, c, d = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    _check(lib().spava_passing_ranges(C.byref(plan), v, C.byref(a), C.byref(b), C.byref(c),
                                      C.byref(d)))
    return (a.value, b.value), (c.value, d.value)


def pad_mask(plan: Plan, v):
    m = np.zeros(max(plan.l_b, 1), np.uint8)
    _check(lib().spava_pad_mask(C.byref(plan), v, m.ctypes.data_as(C.c_void_p)))
    return m[:plan.l_b]


# -------------------------------------------------------------------- device ops
def score_block(q, k, hq, hkv, dh=128, pad=None, n_valid=None, softmax=True, stream=None):
    """score_block (simhost.cpp:209-224): per-key importance, pads -> -inf."""
    import torch

    _require(q, torch.bfloat16, "q")
    _require(k, torch.bfloat16, "k")
    n_t, l_b = q.shape[0], k.shape[0]
    ws_bytes = lib().spava_score_workspace(n_t, l_b, hq)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=q.device)
    out = torch.empty(l_b, dtype=torch.float32, device=q.device)
    padt = None
    if pad is not None:
        padt = torch.as_tensor(np.asarray(pad, np.uint8)).to(q.device)
    _check(lib().spava_score_block(_ptr(q), q.stride(0), n_t, _ptr(k), k.stride(0), l_b, _ptr(padt),
                                   l_b if n_valid is None else n_valid, hq, hkv, dh, int(softmax),
                                   _ptr(out), _ptr(ws), ws_bytes, _stream(stream)))
    return out


def split_rows(plan, h, src, dst=None, stream=None):
    """split_context for host h on the device: global [n_v + n_t, w] -> host-local rows."""
    import torch

    rows = plan.l_a + 2 * plan.l_b + plan.n_t
    if dst is None:
        dst = torch.empty((rows, src.shape[1]), dtype=src.dtype, device=src.device)
    es = src.element_size()
    _check(lib().spava_split_rows(C.byref(plan), h, _ptr(src), src.stride(0) * es, _ptr(dst),
                                  dst.stride(0) * es, src.shape[1] * es, _stream(stream)))
    return dst


def frame_partition(frames, hosts):
    """frame_partition (partition.cpp:30-37): frames per host, the first frames % hosts get +1."""
    out = (C.c_int * max(hosts, 1))()
    _check(lib().spava_frame_partition(frames, hosts, out))
    return list(out)[:hosts]


def gather_split_rows(plan, h, parts, part_rows, e_q, dst=None, stream=None):
    """Encode gather fused with split_context: host h's rows [anchor | lo | hi | query] read
    from the hosts' E_v parts (tensors [part_rows[q], w], frame order) and e_q [n_t, w]."""
    import torch

    rows = plan.l_a + 2 * plan.l_b + plan.n_t
    ref = next(t for t in parts if t is not None)
    if dst is None:
        dst = torch.empty((rows, ref.shape[1]), dtype=ref.dtype, device=ref.device)
    es = ref.element_size()
    n = len(parts)
    ptrs = (C.c_void_p * n)(*[t.data_ptr() if t is not None and t.numel() else None for t in parts])
    prow = (C.c_int64 * n)(*part_rows)
    _check(lib().spava_gather_split_rows(C.byref(plan), h, ptrs, prow, ref.stride(0) * es, _ptr(e_q),
                                         e_q.stride(0) * es, _ptr(dst), dst.stride(0) * es,
                                         ref.shape[1] * es, _stream(stream)))
    return dst


class _CudaArray:
    """__cuda_array_interface__ view of raw device memory (torch.as_tensor aliases it)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": tuple(shape),
                                         "typestr": typestr, "version": 3, "strides": None}


def merge_rows(plan, h, src, dst, write_shared, stream=None):
    """Host h's output rows back to the global sequence positions (inverse of split_rows)."""
    es = src.element_size()
    _check(lib().spava_merge_rows(C.byref(plan), h, _ptr(src), src.stride(0) * es, _ptr(dst),
                                  dst.stride(0) * es, src.shape[1] * es, int(write_shared), _stream(stream)))
    return dst


def score_block_fast(q, k, hq, hkv, dh=128, pad=None, n_valid=None, stream=None):
    """score_block on the tensor cores (spava_score_block_fast): same definition, not
    bit-faithful -- indices agree with the exact scorer except near-ties."""
    import torch

    _require(q, torch.bfloat16, "q")
    _require(k, torch.bfloat16, "k")
    n_t, l_b = q.shape[0], k.shape[0]
    ws_bytes = lib().spava_score_fast_workspace(n_t, l_b, hq)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=q.device)
    out = torch.empty(l_b, dtype=torch.float32, device=q.device)
    padt = None
    if pad is not None:
        padt = torch.as_tensor(np.asarray(pad, np.uint8)).to(q.device)
    _check(lib().spava_score_block_fast(_ptr(q), q.stride(0), n_t, _ptr(k), k.stride(0), l_b, _ptr(padt),
                                        l_b if n_valid is None else n_valid, hq, hkv, dh,
                                        _ptr(out), _ptr(ws), ws_bytes, _stream(stream)))
    return out


def select_pack(scores, l_p, global_offset=0, k=None, v=None, stream=None):
    """select_essential (approx.cpp:71-102) on device; returns device tensors
    (idx[l_p], count[1], k_c, v_c, status[1]); rows >= count are zero."""
    import torch

    dev = scores.device
    l_b = scores.shape[0]
    idx = torch.full((max(l_p, 1),), -1, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    kc = vc = None
    width, ld = 8, 8
    if k is not None:
        width, ld = k.shape[1], k.stride(0)
        kc = torch.zeros((max(l_p, 1), width), dtype=k.dtype, device=dev)
        vc = torch.zeros((max(l_p, 1), width), dtype=k.dtype, device=dev)
    _check(lib().spava_select_pack(_ptr(scores), l_b, l_p, global_offset, _ptr(k), _ptr(v), ld,
                                   width, _ptr(idx), _ptr(kc), _ptr(vc), width, _ptr(cnt), _ptr(st),
                                   _stream(stream)))
    return idx, cnt, kc, vc, st


def select_essential(scores, l_p, global_offset=0, k=None, v=None):
    """Host-facing select_essential: trims to the selected count (synchronises)."""
    idx, cnt, kc, vc, st = select_pack(scores, l_p, global_offset, k, v)
    if int(st.item()):
        raise SpavaError(EINVAL, "select_essential: NaN score")
    n = int(cnt.item())
    return idx[:n], (kc[:n] if kc is not None else None), (vc[:n] if vc is not None else None)


def gemm(a, b, out=None, beta=0.0, relu=False, stream=None):
    """out = a @ b (+ beta * out) (ReLU), bf16 row-major, fp32 accumulation (tcgen05 kernel)."""
    import torch

    _require(a, torch.bfloat16, "a")
    _require(b, torch.bfloat16, "b")
    M, K = a.shape
    K2, N = b.shape
    if K2 != K:
        raise SpavaError(EINVAL, "gemm: inner dimensions differ")
    if out is None:
        out = torch.empty((M, N), dtype=torch.bfloat16, device=a.device)
    _require(out, torch.bfloat16, "out")
    _check(lib().spava_gemm(M, N, K, _ptr(a), a.stride(0), _ptr(b), b.stride(0), _ptr(out), out.stride(0),
                            float(beta), int(bool(relu)), _stream(stream)))
    return out


def attention(q, segments, hq, hkv, dh=128, out_f32=False, want_lse=False, splits=1, stream=None):
    """mha_lse (attention.cpp:158-178) over a segment table.

    segments: list of dict(k=, v=, rows=None, causal=False); rows < k.shape[0] masks
    the tail (pads).  Returns (out [nq, hq*dh], lse [nq, hq] or None)."""
    import torch

    _require(q, torch.bfloat16, "q")
    nq = q.shape[0]
    arr = (_Segment * max(len(segments), 1))()
    for i, s in enumerate(segments):
        _require(s["k"], torch.bfloat16, "k")
        _require(s["v"], torch.bfloat16, "v")
        if s["k"].stride(0) != s["v"].stride(0):
            raise SpavaError(EINVAL, "segment k/v must share a row stride")
        arr[i].k = s["k"].data_ptr()
        arr[i].v = s["v"].data_ptr()
        arr[i].ld = s["k"].stride(0)
        arr[i].rows = s["k"].shape[0] if s.get("rows") is None else int(s["rows"])
        arr[i].causal = int(bool(s.get("causal", False)))
    out = torch.empty((nq, hq * dh), dtype=torch.float32 if out_f32 else torch.bfloat16,
                      device=q.device)
    lse = torch.empty((nq, hq), dtype=torch.float32, device=q.device) if want_lse else None
    ws_bytes = lib().spava_attention_workspace(nq, hq, dh, splits)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=q.device)
    _check(lib().spava_attention(_ptr(q), q.stride(0), nq, arr, len(segments), hq, hkv, dh,
                                 _ptr(out), out.stride(0), int(out_f32), _ptr(lse), splits,
                                 _ptr(ws), ws_bytes, _stream(stream)))
    return out, lse


def mha_merge(outs, lses, hq, dh=128, out_f32=True, want_lse=False, stream=None):
    """mha_merge (attention.cpp:180-197) in part order."""
    import torch

    n = len(outs)
    rows = outs[0].shape[0]
    po = (C.c_void_p * n)(*[o.data_ptr() for o in outs])
    pl = (C.c_void_p * n)(*[l.data_ptr() for l in lses])
    dst = torch.empty((rows, hq * dh), dtype=torch.float32 if out_f32 else torch.bfloat16,
                      device=outs[0].device)
    dl = torch.empty((rows, hq), dtype=torch.float32, device=outs[0].device) if want_lse else None
    st = torch.zeros(1, dtype=torch.int32, device=outs[0].device)
    _check(lib().spava_mha_merge(n, po, pl, rows, outs[0].stride(0), hq, dh, _ptr(dst),
                                 dst.stride(0), int(out_f32), _ptr(dl), _ptr(st), _stream(stream)))
    return dst, dl, st


def anchor_attention(q_a, k_a, v_a, hq, hkv, dh=128, out_f32=False):
    """anchor_attention (approx.cpp:134-138)."""
    return attention(q_a, [dict(k=k_a, v=v_a, causal=True)], hq, hkv, dh, out_f32)[0]


def block_attention(q, k, v, n_valid, k_a, v_a, k_p, v_p, hq, hkv, dh=128, out_f32=False):
    """block_attention (approx.cpp:140-154): [anchor | passing | own causal+pad]."""
    segs = []
    if k_a is not None and k_a.shape[0] > 0:
        segs.append(dict(k=k_a, v=v_a))
    if k_p is not None and k_p.shape[0] > 0:
        segs.append(dict(k=k_p, v=v_p))
    segs.append(dict(k=k, v=v, rows=n_valid, causal=True))
    return attention(q, segs, hq, hkv, dh, out_f32)[0]


def query_attention(q, k_a, v_a, a0, a1, k_lo, v_lo, nv_lo, k_hi, v_hi, nv_hi, k_q, v_q,
                    include_self, hq, hkv, dh=128, splits=1):
    """query_attention (approx.cpp:156-188) -> (out f32, lse)."""
    segs = []
    if a1 > a0:
        segs.append(dict(k=k_a[a0:a1], v=v_a[a0:a1]))
    if nv_lo > 0:
        segs.append(dict(k=k_lo, v=v_lo, rows=nv_lo))
    if nv_hi > 0:
        segs.append(dict(k=k_hi, v=v_hi, rows=nv_hi))
    if include_self:
        segs.append(dict(k=k_q, v=v_q, causal=True))
    return attention(q, segs, hq, hkv, dh, out_f32=True, want_lse=True, splits=splits)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().spava_nccl_unique_id(buf))
    return buf.raw


# ------------------------------------------------------------------ layer runtime
class Host:
    def __init__(self, fabric, h):
        self.fabric = fabric
        self.h = h
        self._p = C.c_void_p()
        _check(lib().spava_host_create(fabric._p, h, C.byref(self._p)))
        self.rows = lib().spava_host_rows(self._p)
        self.plan = Plan()
        lib().spava_host_plan(self._p, C.byref(self.plan))

    def check_buffers(self, q, k, v, out, sel=None):
        """The C ABI takes raw device pointers sized from the plan (rows = l_a + 2 l_b + n_t,
        widths hq*dh / hkv*dh bf16, sel >= 2*l_p int32): reject anything else here so a
        wrong-shaped, fp32 or strided tensor cannot read or write out of bounds."""
        import torch

        c = self.fabric.cfg
        dev = torch.device("cuda", self.fabric.device)
        for t, w, name in ((q, c.hq * c.dh, "q"), (k, c.hkv * c.dh, "k"), (v, c.hkv * c.dh, "v"),
                           (out, c.hq * c.dh, "out")):
            _require(t, torch.bfloat16, name)
            if tuple(t.shape) != (self.rows, w) or not t.is_contiguous():
                raise SpavaError(EINVAL, f"{name}: expected a contiguous [{self.rows}, {w}] tensor, "
                                         f"got {tuple(t.shape)} strides {t.stride()}")
            if t.device != dev:
                raise SpavaError(EINVAL, f"{name}: on {t.device}, the fabric is on {dev}")
        if sel is not None:
            if sel.device != dev or sel.dtype != torch.int32 or not sel.is_contiguous() \
                    or sel.numel() < 2 * max(self.plan.l_p, 1):
                raise SpavaError(EINVAL, f"sel: expected a contiguous int32 tensor of >= "
                                         f"{2 * max(self.plan.l_p, 1)} entries on {dev}")

    def layer(self, q, k, v, out, sel=None, stream=None):
        """One layer of this host (NCCL fabric, or a local fabric with H == 1)."""
        self.check_buffers(q, k, v, out, sel)
        _check(lib().spava_host_layer(self._p, _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(sel),
                                      _stream(stream)))

    def gather_context(self, part_rows, e_q, dst, ld_part_bytes, stream=None):
        """Peer fabric: announce this rank's encode region, wait for the peers', and gather
        this host's [anchor | lo | hi | query] rows over NVLink (spava_host_gather_context)."""
        es = dst.element_size()
        prow = (C.c_int64 * len(part_rows))(*part_rows)
        _check(lib().spava_host_gather_context(self._p, prow, ld_part_bytes, _ptr(e_q), e_q.stride(0) * es,
                                               _ptr(dst), dst.stride(0) * es, dst.shape[1] * es,
                                               _stream(stream)))

    def layer_hostbuf(self, q_h, k_h, v_h, out_h, q_d, k_d, v_d, out_d, sel_h=None, sel_d=None,
                      stream=None):
        """One layer from HOST buffers (pinned CPU tensors) through caller-owned device
        staging buffers; copies are pipelined with the phases (spava_host_layer_hostbuf)."""
        for t in (q_h, k_h, v_h, out_h):
            if t.is_cuda or not t.is_contiguous():
                raise ValueError("layer_hostbuf: host tensors must be contiguous CPU tensors")
        self.check_buffers(q_d, k_d, v_d, out_d, sel_d)
        for th, td in ((q_h, q_d), (k_h, k_d), (v_h, v_d), (out_h, out_d)):
            if th.shape != td.shape or th.dtype != td.dtype:
                raise ValueError("layer_hostbuf: host and device buffers differ in shape or dtype")
        if sel_h is not None and (sel_h.dtype != sel_d.dtype or sel_h.numel() < sel_d.numel()):
            raise ValueError("layer_hostbuf: sel_h must match sel_d")
        _check(lib().spava_host_layer_hostbuf(
            self._p, C.c_void_p(q_h.data_ptr()), C.c_void_p(k_h.data_ptr()), C.c_void_p(v_h.data_ptr()),
            C.c_void_p(out_h.data_ptr()), C.c_void_p(sel_h.data_ptr()) if sel_h is not None else None,
            _ptr(q_d), _ptr(k_d), _ptr(v_d), _ptr(out_d), _ptr(sel_d), _stream(stream)))

    def decoder_layer(self, x, w_qkv, w_o, w_1, w_2, g_1=None, g_2=None, stream=None, ws=None):
        """x += Spava-attention decoder layer (in place); weights are torch CUDA tensors
        (bf16 row-major, gains fp32).  Returns the workspace for reuse."""
        import torch

        dw = DecoderWeights(w_qkv.data_ptr(), w_o.data_ptr(), w_1.data_ptr(), w_2.data_ptr(),
                            g_1.data_ptr() if g_1 is not None else None,
                            g_2.data_ptr() if g_2 is not None else None,
                            x.shape[1], w_1.shape[1], int(g_1 is not None))
        need = lib().spava_decoder_workspace(self._p, C.byref(dw))
        if ws is None or ws.numel() < need:
            ws = torch.empty(need, dtype=torch.uint8, device=x.device)
        _check(lib().spava_host_decoder_layer(self._p, C.byref(dw), _ptr(x), x.stride(0), _ptr(ws),
                                              ws.numel(), _stream(stream)))
        return ws

    def set_delay(self, which, ns):
        """Spin `ns` ns before phase `which` (0 score, 1 exchange, 2 query, 3 stage 1)."""
        _check(lib().spava_host_set_delay(self._p, int(which), int(ns)))

    def capture_layer(self, q, k, v, out, sel=None, stream=None):
        """Capture one layer on these buffers as a CUDA graph (replay_layer launches it)."""
        self.check_buffers(q, k, v, out, sel)
        _check(lib().spava_host_capture_layer(self._p, _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(sel),
                                              _stream(stream)))

    def replay_layer(self, stream=None):
        _check(lib().spava_host_replay_layer(self._p, _stream(stream)))

    def set_trace(self, enable=True):
        """Record run_host's schedule events (reference Event schema) on every layer call."""
        _check(lib().spava_host_set_trace(self._p, int(enable)))

    def trace_records(self):
        """Program-order records: [(kind, label, layer, tag, t_us)] (kind per EVENT_KINDS)."""
        n = C.c_int()
        _check(lib().spava_host_trace_read(self._p, None, 0, C.byref(n)))
        buf = (TraceEvent * max(n.value, 1))()
        _check(lib().spava_host_trace_read(self._p, buf, n.value, C.byref(n)))
        return [(e.kind, e.label.decode(), e.layer, e.tag.decode(), e.t_us) for e in buf[:n.value]]

    def set_timing(self, enable=True):
        _check(lib().spava_host_set_timing(self._p, int(enable)))

    def timing(self):
        """{'attention','score','select','merge'} ms summed over recorded launches,
        plus algorithmic attention FLOPs and the attention launch count."""
        ms = (C.c_double * 4)()
        fl = C.c_double()
        n = C.c_uint64()
        _check(lib().spava_host_timing(self._p, ms, C.byref(fl), C.byref(n)))
        return dict(attention_ms=ms[0], score_ms=ms[1], select_ms=ms[2], merge_ms=ms[3],
                    attention_flops=fl.value, attention_launches=n.value)

    def status(self, stream=None):
        s = C.c_int32()
        _check(lib().spava_host_status(self._p, _stream(stream), C.byref(s)))
        return s.value

    def close(self):
        if self._p:
            lib().spava_host_destroy(self._p)
            self._p = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


PEER_HANDLE_BYTES = 64


class Fabric:
    """GatherFabric (simhost.cpp:61-166) equivalent: local (one device), NCCL, or peer
    (NVLink P2P stores from the producing kernels + epoch flags; `Fabric.peer`)."""

    def __init__(self, cfg: LayerConfig, device=0, unique_id=None, world=1, rank=0,
                 peer=False, encode_bytes=0):
        self.cfg = cfg
        self.device = device
        self._p = C.c_void_p()
        self.nccl = self.peer = False
        if peer:
            _check(lib().spava_fabric_create_peer(C.byref(cfg), device, world, rank, encode_bytes,
                                                  C.byref(self._p)))
            self.peer = True
        elif unique_id is None:
            _check(lib().spava_fabric_create_local(C.byref(cfg), device, C.byref(self._p)))
        else:
            buf = C.create_string_buffer(unique_id, 128)
            _check(lib().spava_fabric_create_nccl(C.byref(cfg), device, buf, world, rank,
                                                  C.byref(self._p)))
            self.nccl = True

    @classmethod
    def create_peer(cls, cfg: LayerConfig, device, world, rank, encode_bytes=0):
        return cls(cfg, device, world=world, rank=rank, peer=True, encode_bytes=encode_bytes)

    def encode_tensor(self, rows, cols):
        """bf16 [rows, cols] torch view of this rank's encode region (its E_v share)."""
        import torch

        ptr, nbytes = C.c_void_p(), C.c_int64()
        _check(lib().spava_fabric_encode_region(self._p, C.byref(ptr), C.byref(nbytes)))
        if rows * cols * 2 > nbytes.value:
            raise ValueError("encode_tensor: larger than the encode region")
        arr = _CudaArray(ptr.value, (rows, cols), "<i2")
        return torch.as_tensor(arr, device=f"cuda:{self.device}").view(torch.bfloat16)

    def encode_acquire(self, stream=None):
        """Enqueue: wait until every peer has read the previous encode round."""
        _check(lib().spava_fabric_encode_acquire(self._p, _stream(stream)))

    def peer_handle(self) -> bytes:
        """64-byte IPC handle of this rank's exchange buffer (send it to every rank)."""
        buf = C.create_string_buffer(PEER_HANDLE_BYTES)
        _check(lib().spava_fabric_peer_handle(self._p, buf))
        return buf.raw

    def peer_open(self, handles):
        """Map every other rank's exchange buffer; `handles` = the ranks' handles in order."""
        blob = b"".join(handles)
        _check(lib().spava_fabric_peer_open(self._p, C.create_string_buffer(blob, len(blob))))

    @staticmethod
    def peer_attach(fabrics):
        """In-process peer fabrics (one device): fabrics[r] is rank r."""
        n = len(fabrics)
        _check(lib().spava_fabric_peer_attach((C.c_void_p * n)(*[f._p.value for f in fabrics]), n))

    def host(self, h) -> Host:
        return Host(self, h)

    def sim_layer(self, hosts, qs, ks, vs, outs, sels=None, stream=None):
        n = len(hosts)
        for i, h in enumerate(hosts):
            h.check_buffers(qs[i], ks[i], vs[i], outs[i], sels[i] if sels is not None else None)
        arr = lambda ts: (C.c_void_p * n)(*[t.data_ptr() if t is not None else None for t in ts])
        _check(lib().spava_sim_layer(self._p, (C.c_void_p * n)(*[h._p.value for h in hosts]),
                                     arr(qs), arr(ks), arr(vs), arr(outs),
                                     arr(sels) if sels is not None else None, _stream(stream)))

    def sim_layer_timed(self, hosts, qs, ks, vs, outs, sels=None, stream=None):
        """sim_layer with each host's phases timed alone on the GPU: list of ms per host."""
        n = len(hosts)
        for i, h in enumerate(hosts):
            h.check_buffers(qs[i], ks[i], vs[i], outs[i], sels[i] if sels is not None else None)
        arr = lambda ts: (C.c_void_p * n)(*[t.data_ptr() if t is not None else None for t in ts])
        ms = (C.c_float * n)()
        _check(lib().spava_sim_layer_timed(self._p, (C.c_void_p * n)(*[h._p.value for h in hosts]),
                                           arr(qs), arr(ks), arr(vs), arr(outs),
                                           arr(sels) if sels is not None else None, _stream(stream), ms))
        return list(ms)

    def close(self):
        if self._p:
            lib().spava_fabric_destroy(self._p)
            self._p = C.c_void_p()


@dataclass
class HostLayout:
    """Row ranges of the host-local buffers [anchor | lo | hi | query]."""
    l_a: int
    l_b: int
    n_t: int

    @property
    def lo(self):
        return slice(self.l_a, self.l_a + self.l_b)

    @property
    def hi(self):
        return slice(self.l_a + self.l_b, self.l_a + 2 * self.l_b)

    @property
    def query(self):
        return slice(self.l_a + 2 * self.l_b, self.l_a + 2 * self.l_b + self.n_t)

    @property
    def anchor(self):
        return slice(0, self.l_a)
