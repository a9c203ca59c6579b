#!/usr/bin/env python
"""bench.py -- Spava sequence-parallel prefill attention on B200 (one layer per step).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C1] [--impl spava|reference]

N>1 is launched by the driver under torch.distributed.run (one rank per GPU).
Rank h is physical host h of the reference's partition (zigzag virtual pair (h, 2H-1-h));
the three exchange rounds (pass1, pass2, qpartial) run inside the C-ABI layer call: by
default as NVLink stores from the select-gather / query-merge kernels into the peers'
IPC-mapped exchange buffers with epoch flags (`--fabric peer`), or as in-place
ncclAllGathers on a comm stream (`--fabric nccl`).  A "step" is one Spava attention layer of the whole job:
score -> select+pack -> exchange -> query / anchor / block attention -> lse merge
(run_host's per-layer body, simhost.cpp:321-426, minus projections/FFN).

Workload (BASELINE.json configs[1] = C1): Qwen2.5-VL-3B-shaped attention (16 q / 2 kv
heads, d=128), n = 32768 tokens (n_t = 128 query rows), l_a = n/64, l_p = n/128, one
layer, synthetic bf16 N(0,1) activations resident in HBM.  L2 is flushed (256 MiB
write) between timed steps, outside the timed events.

JSON line: value = tokens/s of the whole job (n per step / max-over-ranks device
time); e2e = the same through the public C-ABI call with pinned HOST buffers (H2D of
this rank's Q/K/V and D2H of its attention outputs inside the timed region);
roofline = the attention kernel (attn_fwd_kernel, all launches of the step) against
the measured bf16 tensor peak; cpu_baseline = the reference's own operators
(oracle/_ref, the unmodified C++ sources) on a bounded sample of the same layer.
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "C1": dict(desc="single Spava attention layer, Qwen2.5-VL-3B shape (16q/2kv, d=128), 32K tokens",
               n=32768, n_t=128, hq=16, hkv=2, layers=1, model="Qwen2.5-VL-3B-shaped attention"),
    "C2": dict(desc="Qwen2.5-VL-3B shape, 64K tokens, one of 36 layers",
               n=65536, n_t=128, hq=16, hkv=2, layers=1, model="Qwen2.5-VL-3B-shaped attention"),
    "C3": dict(desc="long video ~128K tokens, Qwen2.5-VL-3B shape, one of 36 layers",
               n=131072, n_t=128, hq=16, hkv=2, layers=1, model="Qwen2.5-VL-3B-shaped attention"),
    "C4": dict(desc="Qwen2.5-VL-7B shape (28q/4kv), 256K tokens, one of 28 layers",
               n=262144, n_t=128, hq=28, hkv=4, layers=1, model="Qwen2.5-VL-7B-shaped attention"),
}
DH = 128
METRIC = "Spava prefill-attn tokens/s"


def geometry(cfg, hosts, zigzag=True):
    n, n_t = cfg["n"], cfg["n_t"]
    n_v = n - n_t
    l_a = n // 64  # resolve_lengths ratios over n = n_v + n_t (config.cpp:34-56)
    vh = 2 * hosts
    rem = n_v - l_a
    pad = (vh - rem % vh) % vh
    l_b = (rem + pad) // vh
    l_p = min(n // 128, l_b)
    return dict(n=n, n_v=n_v, n_t=n_t, l_a=l_a, l_b=l_b, l_p=l_p, pad=pad, hosts=hosts,
                zigzag=zigzag)


def attn_flops_host(g, hq, h, zigzag=True):
    """Reference FLOP convention (attention.cpp:33-36) for physical host h, one layer."""
    H, l_a, l_b, l_p, n_t = g["hosts"], g["l_a"], g["l_b"], g["l_p"], g["n_t"]
    lo, hi = (h, 2 * H - 1 - h) if zigzag else (2 * h, 2 * h + 1)
    base = l_a // H
    a = base + (1 if h < l_a % H else 0)
    f = 2 * l_a * l_a  # anchor self (causal)
    for v in (lo, hi):
        f += 4 * l_b * l_a + 4 * l_b * (v * l_p) + 2 * l_b * l_b
    f += 4 * n_t * (a + 2 * l_b) + (2 * n_t * n_t if h == H - 1 else 0)
    return f * DH * hq


def score_flops_host(g, hq):
    return 2 * (2 * g["n_t"] * g["l_b"] * DH * hq)


# ------------------------------------------------------------- measured peaks
def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return dict(bf16_burst=float(d["bf16_tflops"]), bf16_sustained=float(d["bf16_tflops_sustained"]),
                    hbm=float(d["hbm_gbs"]), src="measured")
    except Exception:
        return dict(bf16_burst=1590.0, bf16_sustained=1400.0, hbm=6650.0, src="fallback")


# ------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index):
        self.samples, self.reasons, self.stop_evt = [], 0, threading.Event()
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self.stop_evt.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop_evt.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1],
                "samples": len(self.samples)}


# -------------------------------------------------------- reference CPU baseline
def reference_job(g, hq, hkv, steps, warmup, threads, max_s=100.0, seed=1234, m=128):
    """The reference's own operators (oracle/_ref: the unmodified seqpar C++ sources; the C
    restatement if _ref is absent) over ONE Spava layer of the whole job on the host cores,
    on the same synthetic inputs as the GPU arm (oracle/layer_ref.layer_inputs, same seed):
    every block's score_block + select_essential, then anchor / block / query attention as
    row-slice x head work items (exact sub-problems of the full calls, run_host order
    simhost.cpp:328-426).  The layer's work items are split over the `steps` timed steps
    (scoring first), so the steps together execute the layer once; when the estimated
    layer time exceeds `max_s` a uniform, FLOP-stratified fraction of the attention items
    runs instead and the rate is extrapolated (said in `sample`).  Returns a dict."""
    from oracle import layer_ref as LR

    Q, K, V = LR.layer_inputs(g, hq, hkv, seed=seed)
    ref = LR.LayerRef(Q, K, V, g, hq, hkv)
    H = g["hosts"]
    score = ref.score_items()
    attn = ref.attention_items(range(g["l_a"]), {v: range(LR.valid_rows(g, v)) for v in range(2 * H)},
                               range(g["n_t"]), m=m)
    # the anchor is computed by every host (redundantly, simhost.cpp:308-311): count it H times
    total = sum(it[5] for it in score) + sum(it[5] * (H if it[0] == "anchor" else 1) for it in attn)
    est_rate = 2.0e9 * threads  # ~2 GFLOP/s per core (scalar fp32 reference)
    frac = min(1.0, max_s * est_rate / total)
    if frac < 1.0:  # stratified: every k-th item in FLOP order
        attn = sorted(attn, key=lambda it: it[5])
        k = int(round(1.0 / frac))
        attn = attn[::k]
    done_total = sum(it[5] for it in score) + sum(it[5] * (H if it[0] == "anchor" else 1) for it in attn)
    frac = done_total / total
    seq = score + [None] + attn  # None: score_block totals + select_essential of every block
    per = sum(it[5] for it in seq if it) / max(1, steps)
    groups, cur, acc = [], [], 0.0
    for it in seq:
        cur.append(it)
        acc += it[5] if it else 0.0
        if acc >= per * (len(groups) + 1) and len(groups) < steps - 1:
            groups.append(cur)
            cur = []
    groups.append(cur)
    while len(groups) < steps:
        groups.append([])
    for _ in range(warmup):  # untimed: a few scoring items (their results are overwritten)
        LR.run_items(ref.run_item, score[:threads], threads)
    step_s = []
    for grp in groups:
        t0 = time.perf_counter()
        if None in grp:
            i = grp.index(None)
            LR.run_items(ref.run_item, grp[:i], threads)
            ref.finish_scores()
            LR.run_items(ref.run_item, grp[i + 1:], threads)
        elif grp:
            LR.run_items(ref.run_item, grp, threads)
        step_s.append(time.perf_counter() - t0)
    layer_s = sum(step_s) / frac
    kind = "reference" if ref.impl == "ref" else "port"
    sample = (f"one whole layer of the job ({H} host(s): scores + select of {2 * H} blocks, "
              f"anchor/block/query attention as {m}-row x head work items) split over {steps} steps, "
              f"{sum(step_s):.1f} s on {threads} threads"
              if frac >= 0.999 else
              f"{frac:.1%} of one layer's FLOPs (all scoring + every {int(round(1 / max(frac, 1e-9)))}-th "
              f"attention work item in FLOP order) split over {steps} steps, {sum(step_s):.1f} s on "
              f"{threads} threads; layer time extrapolated as measured time / FLOP fraction")
    return dict(value=g["n"] / layer_s, layer_s=layer_s, step_s=step_s, frac=frac, kind=kind,
                sample=sample, gflops_per_s=done_total / sum(step_s) / 1e9, impl=ref.impl)


# --------------------------------------------------------------------- arms
def dist_env():
    local = int(os.environ.get("LOCAL_RANK", 0))
    if os.environ.get("SPAVA_BENCH_ONE_GPU") == "1":  # test aid: every rank on cuda:0 (gloo)
        local = 0
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), local


def job_config(args, world):
    """(config name, cfg, geometry) of the job, unless --config says otherwise: the BASELINE
    config quoted at that GPU count -- C1 at N = 1 and 2 (configs[1]: "32K tokens, 1 B200 vs
    2 GPUs"), C2 at N = 3..4 (configs[2]: 64K tokens, "4 and 8 B200"), the 128K-token C3 at
    N > 4 (configs[3], north_star's 1 -> 8 scaling target)."""
    n = max(world, args.gpus)
    name = args.config or ("C1" if n <= 2 else "C2" if n <= 4 else "C3")
    cfg = CONFIGS[name]
    return name, cfg, geometry(cfg, max(world, args.gpus))


def config_dict(name, cfg, g, H, fabric=None, fabric_note=None):
    """The `config` object both arms print (identical keys and values for the same job)."""
    return {"workload": f"{name}: {cfg['desc']}", "n": g["n"], "n_t": g["n_t"], "l_a": g["l_a"],
            "l_b": g["l_b"], "l_p": g["l_p"], "hosts": H, "heads": f"{cfg['hq']}q/{cfg['hkv']}kv",
            "dh": DH, "layers_per_step": 1,
            "parallelism": f"sp{H} (Spava zigzag virtual hosts, one per GPU)",
            "inputs": "oracle/layer_ref.layer_inputs(seed=1234): N(0,1) rounded to bf16, same bits in both arms",
            "scoring": "exact (score_block arithmetic order, selection bit-exact vs the reference)"}


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    name, cfg, g = job_config(args, world)
    H = g["hosts"]
    threads = os.cpu_count() or 1
    r = reference_job(g, cfg["hq"], cfg["hkv"], args.steps, args.warmup, threads, max_s=args.ref_max_s)
    ms = [x * 1e3 for x in r["step_s"]]
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": "tokens/s",
        "n_gpus": max(world, args.gpus), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sum(ms) / len(ms), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic N(0,1) bf16-valued activations",
        "config": config_dict(name, cfg, g, H),
        "cpu_baseline": {"value": r["value"], "unit": "tokens/s", "cores": threads, "kind": r["kind"],
                         "sample": r["sample"], "layer_s": round(r["layer_s"], 2),
                         "gflops_per_s": round(r["gflops_per_s"], 2), "fraction_of_layer": round(r["frac"], 4)},
        "e2e": {"value": r["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step_ms": [round(x, 1) for x in ms],
    }
    print(json.dumps(line), flush=True)


def bind_gpu_numa(dev_index):
    """Pin this process to the CPUs local to the GPU's PCIe root (sysfs local_cpulist), so
    the pinned host buffers of the e2e leg are allocated on the GPU's NUMA node; returns
    the cpulist used (None if unavailable)."""
    import torch

    try:
        pr = torch.cuda.get_device_properties(dev_index)
        bdf = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        path = f"/sys/bus/pci/devices/{bdf}/local_cpulist"
        with open(path) as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
            return spec
    except (OSError, ValueError, AttributeError):
        pass
    return None


def make_fabric(spava, dist, lc, local, world, rank, fabric):
    """This rank's fabric: local (N=1), peer (NVLink stores + epoch flags) or NCCL."""
    note, peer_err = None, ""
    if world == 1:
        return spava.Fabric(lc, local), "local", note, peer_err
    fab = None
    if fabric == "peer":
        fab = spava.Fabric.create_peer(lc, local, world, rank)
        handles = [None] * world
        dist.all_gather_object(handles, fab.peer_handle())
        try:
            fab.peer_open(handles)
        except spava.SpavaError as e:  # e.g. peers not visible to this process
            peer_err = str(e)[:160]
        errs = [None] * world
        dist.all_gather_object(errs, peer_err)
        if any(errs):  # every rank switches together
            note = "peer open failed (" + next(x for x in errs if x) + "); nccl used"
            fab.close()
            fab = None
            fabric = "nccl"
    if fab is None:
        obj = [spava.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        fab = spava.Fabric(lc, local, unique_id=obj[0], world=world, rank=rank)
    return fab, fabric, note, peer_err


def hbm_rooflines(g, hq, hkv, tim, steps, hbm_peak):
    """Achieved HBM GB/s of the scorer and of select + pack (north_star: against ~8 TB/s),
    from the algorithmic bytes of SURVEY s8d and the kernels' device time per step."""
    l_b, l_p, n_t = g["l_b"], g["l_p"], g["n_t"]
    b_sel = 2 * (4 * l_b + 4 * l_p + 2 * 2 * l_p * hkv * DH * 2)      # scores in, idx + K/V rows
    b_score = n_t * hq * DH * 2 + 2 * l_b * hkv * DH * 2 + 2 * 4 * l_b  # Q_qr + 2 K blocks + scores
    sel_ms = tim["select_ms"] / steps
    sc_ms = tim["score_ms"] / steps
    f_score = score_flops_host(g, hq)
    out = {}
    if sel_ms > 0:
        a = b_sel / (sel_ms / 1e3) / 1e9
        out["select_pack"] = {"bound": "hbm", "achieved": round(a, 1), "peak": hbm_peak, "unit": "GB/s",
                              "frac": round(a / hbm_peak, 4), "bytes_per_step": b_sel,
                              "ms_per_step": round(sel_ms, 4),
                              "note": "select (radix select + ordered scan, one CTA per block) + "
                                      "gather of the passing K/V rows; latency-bound at these sizes"}
    if sc_ms > 0:
        a = b_score / (sc_ms / 1e3) / 1e9
        out["score"] = {"bound": "fp32/fp64 CUDA cores (exact mode; intensity n_t*hq/hkv flop/B)",
                        "achieved_hbm": round(a, 1), "peak_hbm": hbm_peak, "unit": "GB/s",
                        "frac_hbm": round(a / hbm_peak, 4), "bytes_per_step": b_score,
                        "flops_per_step": f_score, "tflops": round(f_score / (sc_ms / 1e3) / 1e12, 2),
                        "ms_per_step": round(sc_ms, 4)}
    return out


def time_layer(torch, host, q, k, v, out, sel, stream, flush, steps, warmup):
    """warm-up, then `steps` layers bracketed by events (L2 flushed outside the events)."""
    for _ in range(warmup):
        host.layer(q, k, v, out, sel, stream)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush.zero_()
        ev[i][0].record(stream)
        host.layer(q, k, v, out, sel, stream)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def sweep_line(torch, spava, name, local, stream, flush, steps, pk, full=True):
    """One more single-GPU configuration on the N=1 line (BASELINE's 1/2/4/8 sweep config
    C4 at H=1, and C3 at H=1 for the 128K scaling curve): tokens/s, attention roofline and
    e2e through the host-buffer C-ABI call.  Inputs are drawn on the device (not compared)."""
    cfg = CONFIGS[name]
    g = geometry(cfg, 1)
    hq, hkv = cfg["hq"], cfg["hkv"]
    lc = spava.LayerConfig.make(g["n_v"], g["n_t"], 1, g["l_a"], g["l_p"], hq, hkv, DH)
    fab = spava.Fabric(lc, local)
    host = fab.host(0)
    dev = torch.device("cuda", local)
    gen = torch.Generator(device=dev).manual_seed(99)
    rows = host.rows
    q = torch.randn((rows, hq * DH), generator=gen, device=dev).to(torch.bfloat16)
    k = torch.randn((rows, hkv * DH), generator=gen, device=dev).to(torch.bfloat16)
    v = torch.randn((rows, hkv * DH), generator=gen, device=dev).to(torch.bfloat16)
    out = torch.empty((rows, hq * DH), dtype=torch.bfloat16, device=dev)
    sel = torch.empty((2, max(g["l_p"], 1)), dtype=torch.int32, device=dev)
    host.set_timing(True)
    step_ms = time_layer(torch, host, q, k, v, out, sel, stream, flush, steps, 1)
    tim = host.timing()
    host.set_timing(False)
    ms = sum(step_ms) / steps
    # timing covers warm-up + steps launches: normalise by the launch count
    n_layers = steps + 1
    ach = tim["attention_flops"] / (tim["attention_ms"] / 1e3) / 1e12
    res = {"workload": f"{name}: {cfg['desc']}", "hosts": 1, "n": g["n"], "l_b": g["l_b"], "l_p": g["l_p"],
           "heads": f"{hq}q/{hkv}kv", "value": g["n"] / (ms / 1e3), "unit": "tokens/s", "ms_per_step": round(ms, 3),
           "steps": steps,
           "roofline": {"bound": "tensor", "achieved": round(ach, 1), "peak": pk["bf16_burst"], "unit": "TFLOP/s",
                        "frac": round(ach / pk["bf16_burst"], 4),
                        "flops_per_step": tim["attention_flops"] / n_layers,
                        "kernel_ms_per_step": round(tim["attention_ms"] / n_layers, 3)}}
    if not full:  # device path only (N > 1: the same workload at H = 1, for the curve)
        host.close()
        fab.close()
        del q, k, v, out
        torch.cuda.empty_cache()
        return res
    try:  # e2e through the host-buffer entry point
        qh, kh, vh = q.cpu().pin_memory(), k.cpu().pin_memory(), v.cpu().pin_memory()
        oh = torch.empty(out.shape, dtype=out.dtype).pin_memory()
        selh = torch.empty(sel.shape, dtype=sel.dtype).pin_memory()
        host.layer_hostbuf(qh, kh, vh, oh, q, k, v, out, selh, sel, stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n2 = max(2, min(steps, 3))
        e0.record(stream)
        for _ in range(n2):
            host.layer_hostbuf(qh, kh, vh, oh, q, k, v, out, selh, sel, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / n2
        res["e2e"] = {"value": g["n"] / (ems / 1e3), "unit": "tokens/s", "ms_per_step": round(ems, 3),
                      "h2d_bytes_per_step": (q.numel() + k.numel() + v.numel()) * 2,
                      "d2h_bytes_per_step": out.numel() * 2}
        del qh, kh, vh, oh
    except Exception as e:  # pragma: no cover
        res["e2e"] = {"error": str(e)[:200]}
    # dense exact causal attention over the same sequence on one GPU (our kernel)
    try:
        n = g["n"]
        qd = torch.randn((n, hq * DH), generator=gen, device=dev).to(torch.bfloat16)
        kd = torch.randn((n, hkv * DH), generator=gen, device=dev).to(torch.bfloat16)
        vd = torch.randn((n, hkv * DH), generator=gen, device=dev).to(torch.bfloat16)
        del q, k, v, out
        segs = [dict(k=kd, v=vd, causal=True)]
        spava.attention(qd, segs, hq, hkv)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        spava.attention(qd, segs, hq, hkv)
        e1.record()
        torch.cuda.synchronize()
        dms = e0.elapsed_time(e1)
        res["dense_exact"] = {"ms": round(dms, 3), "tokens_per_s": n / (dms / 1e3),
                              "tflops": round(2.0 * n * n * hq * DH / (dms / 1e3) / 1e12, 1),
                              "spava_speedup": round(dms / ms, 2)}
        del qd, kd, vd
    except Exception as e:  # pragma: no cover
        res["dense_exact"] = {"error": str(e)[:200]}
    host.close()
    fab.close()
    torch.cuda.empty_cache()
    return res


def self_check(torch, spava, g, hq, hkv, Q, K, V, out, sel, rank, local):
    """N > 1: this rank's passing indices and outputs against a one-GPU spava_sim_layer of
    all H hosts on the same inputs (local fabric; bit-identical by construction)."""
    from oracle import layer_ref as LR

    H = g["hosts"]
    dev = torch.device("cuda", local)
    lc = spava.LayerConfig.make(g["n_v"], g["n_t"], H, g["l_a"], g["l_p"], hq, hkv, DH)
    fab = spava.Fabric(lc, local)
    hs, ins, outs, sels = [], [], [], []
    for h in range(H):
        hs.append(fab.host(h))
        rows = LR.host_rows(g, h)
        ins.append([torch.from_numpy(X[rows]).to(dev).to(torch.bfloat16) for X in (Q, K, V)])
        outs.append(torch.empty((hs[-1].rows, hq * DH), dtype=torch.bfloat16, device=dev))
        sels.append(torch.empty((2, max(g["l_p"], 1)), dtype=torch.int32, device=dev))
    fab.sim_layer(hs, [x[0] for x in ins], [x[1] for x in ins], [x[2] for x in ins], outs, sels)
    torch.cuda.synchronize()
    res = {"indices_equal": bool(torch.equal(sels[rank], sel)),
           "out_max_abs_diff": float((outs[rank].float() - out.float()).abs().max()),
           "out_bit_identical": bool(torch.equal(outs[rank], out)),
           "reference": "spava_sim_layer of all hosts on one GPU (local fabric), same inputs"}
    for h in hs:
        h.close()
    fab.close()
    del ins, outs, sels
    torch.cuda.empty_cache()
    return res


def run_spava_arm(args):
    import torch
    import torch.distributed as dist

    from oracle import layer_ref as LR
    from paper_2601_21444_b200 import spava

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world} (N > 1 runs one process per GPU "
                         "under torch.distributed.run)")
    torch.cuda.set_device(local)
    all_cpus = os.sched_getaffinity(0)
    numa_cpus = bind_gpu_numa(local)
    dev = torch.device("cuda", local)
    name, cfg, g = job_config(args, world)
    H = max(world, 1)
    hq, hkv = cfg["hq"], cfg["hkv"]
    lc = spava.LayerConfig.make(g["n_v"], g["n_t"], H, g["l_a"], g["l_p"], hq, hkv, DH)
    if world > 1:
        if os.environ.get("SPAVA_BENCH_ONE_GPU") == "1":
            if args.fabric != "peer":
                raise SystemExit("SPAVA_BENCH_ONE_GPU needs --fabric peer (NCCL refuses shared GPUs)")
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    fab, fabric, fabric_note, peer_err = make_fabric(spava, dist, lc, local, world, rank, args.fabric)
    host = fab.host(rank)
    rows = host.rows
    # the same synthetic layer as the reference arm (global rows, this host's share)
    Q, K, V = LR.layer_inputs(g, hq, hkv, seed=1234)
    hr = LR.host_rows(g, rank)
    q, k, v = [torch.from_numpy(X[hr]).to(dev).to(torch.bfloat16) for X in (Q, K, V)]
    assert q.shape[0] == rows
    out = torch.empty((rows, hq * DH), dtype=torch.bfloat16, device=dev)
    sel = torch.empty((2, max(g["l_p"], 1)), dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        host.layer(q, k, v, out, sel, stream)
    torch.cuda.synchronize()
    st = host.status()
    if st != 0:
        raise SystemExit(f"layer status {st}")

    # ---------------- timed region (device events per step; L2 flushed between steps)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    launches0 = spava.kernel_launches()
    host.set_timing(True)
    with ClockSampler(local) as clk:
        wall0 = time.perf_counter()
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            host.layer(q, k, v, out, sel, stream)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
    barrier()
    launches = spava.kernel_launches() - launches0
    tim = host.timing()
    host.set_timing(False)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = sum(step_ms) / args.steps
    t = torch.tensor([ms, tim["attention_ms"] / args.steps], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t[0])
    tokens = g["n"]  # one sequence of n tokens per step for the whole job
    value = tokens / (ms_max / 1e3)
    out_timed = out.clone()
    sel_timed = sel.clone()

    # ---------------- e2e through the C-ABI call with pinned host buffers
    qh = q.cpu().pin_memory()
    kh = k.cpu().pin_memory()
    vh = v.cpu().pin_memory()
    oh = torch.empty(out.shape, dtype=out.dtype).pin_memory()
    e2e_steps = max(3, min(args.steps, 10))
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(e2e_steps)]
    selh = torch.empty(sel.shape, dtype=sel.dtype).pin_memory()

    def step_host():
        # the C-ABI host-buffer entry point: copies pipelined with the layer's phases
        host.layer_hostbuf(qh, kh, vh, oh, q, k, v, out, selh, sel, stream)

    step_host()  # untimed warm-up of the copy streams
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    for i in range(e2e_steps):
        flush.zero_()
        ev2[i][0].record(stream)
        step_host()
        ev2[i][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_step_ms = [a.elapsed_time(b) for a, b in ev2]
    e2e_ms = sum(e2e_step_ms) / e2e_steps
    t2 = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t2, op=dist.ReduceOp.MAX)
    e2e_ms = float(t2[0])
    h2d = (q.numel() + k.numel() + v.numel()) * 2
    d2h = out.numel() * 2
    e2e_same = bool(torch.equal(oh.to(dev), out_timed))
    # copy floor: the same bytes as bare pinned copies (H2D and D2H on two streams at once),
    # i.e. the PCIe time the host-buffer layer hides its compute under
    s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    floor = []
    for _ in range(4):
        torch.cuda.synchronize()
        c0.record(stream)
        s_up.wait_stream(stream)
        s_dn.wait_stream(stream)
        with torch.cuda.stream(s_up):
            q.copy_(qh, non_blocking=True)
            k.copy_(kh, non_blocking=True)
            v.copy_(vh, non_blocking=True)
        with torch.cuda.stream(s_dn):
            oh.copy_(out, non_blocking=True)
        stream.wait_stream(s_up)
        stream.wait_stream(s_dn)
        c1.record(stream)
        torch.cuda.synchronize()
        floor.append(c0.elapsed_time(c1))
    copy_floor_ms = min(floor[1:])
    del qh, kh, vh, oh

    # ---------------- isolated kernel timing (scorer serialized on the step stream) so the
    # attention kernel's own efficiency is visible next to the overlapped timed region
    iso_steps = max(3, min(args.steps, 10))
    host.set_timing(2)
    torch.cuda.synchronize()
    for _ in range(iso_steps):
        flush.zero_()
        host.layer(q, k, v, out, sel, stream)
    torch.cuda.synchronize()
    tim_iso = host.timing()
    host.set_timing(False)

    # ---------------- N > 1: self-check against one GPU + per-rank exchange evidence
    rank_info = {"rank": rank, "device": torch.cuda.get_device_name(local), "fabric": fabric,
                 "peer_open_error": peer_err or None,
                 "nccl_ranks": world if fabric == "nccl" else 0, "ms_per_step": round(ms, 4),
                 "attention_ms_per_step": round(tim["attention_ms"] / args.steps, 4)}
    if world > 1:
        if not args.no_self_check:
            rank_info["self_check"] = self_check(torch, spava, g, hq, hkv, Q, K, V, out_timed, sel_timed,
                                                 rank, local)
        ranks = [None] * world
        dist.all_gather_object(ranks, rank_info)
    else:
        ranks = None
    del Q, K, V

    if rank != 0:
        if world > 1:
            torch.cuda.synchronize()
            dist.barrier()  # peers store into this rank's exchange buffer until their last layer
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---------------- roofline of the dominant kernel (attn_fwd_kernel)
    pk = peaks()
    attn_flops_step = tim["attention_flops"] / args.steps
    achieved = attn_flops_step / (tim["attention_ms"] / args.steps / 1e3) / 1e12
    clocks = clk.summary()
    # the step is milliseconds long at full clocks: the burst peak applies (MEASURED_PEAKS
    # recorded the sustained figure at a power-capped 1215 MHz median)
    peak = pk["bf16_burst"]
    traffic, traffic_src = None, None
    for tp in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_step.json")), reverse=True):
        try:
            with open(tp) as f:
                traffic = json.load(f).get(name, {}).get("dram_bytes_per_launch")
            if traffic:
                traffic_src = os.path.relpath(tp, ROOT)
                break
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_src": traffic_src,
                "kernel": "attn_fwd_kernel (tcgen05, all attention launches of the step)",
                "peak_src": f"{pk['src']} bf16 burst (MEASURED_PEAKS.json bf16_tflops; clocks at "
                            f"{clocks.get('sm_mhz')} of {clocks.get('sm_max_mhz')} MHz)",
                "peak_sustained": pk["bf16_sustained"],
                "frac_vs_sustained": round(achieved / pk["bf16_sustained"], 4),
                "flops_per_step": attn_flops_step,
                "kernel_ms_per_step": round(tim["attention_ms"] / args.steps, 4),
                "share_of_step": round(tim["attention_ms"] / args.steps / ms, 3),
                "score_ms_per_step": round(tim["score_ms"] / args.steps, 4),
                "select_ms_per_step": round(tim["select_ms"] / args.steps, 4),
                "merge_ms_per_step": round(tim["merge_ms"] / args.steps, 4),
                "note": "timed region: the scorer runs on a side stream concurrently with the query/"
                        "stage-1 attention, so attention launches share the SMs; 'isolated' times "
                        "the same launches with the scorer serialized"}
    iso_ms = tim_iso["attention_ms"] / iso_steps
    iso_ach = tim_iso["attention_flops"] / iso_steps / (iso_ms / 1e3) / 1e12
    roofline["isolated"] = {"achieved": round(iso_ach, 1), "frac": round(iso_ach / peak, 4),
                            "kernel_ms_per_step": round(iso_ms, 4),
                            "score_ms_per_step": round(tim_iso["score_ms"] / iso_steps, 4),
                            "select_ms_per_step": round(tim_iso["select_ms"] / iso_steps, 4),
                            "merge_ms_per_step": round(tim_iso["merge_ms"] / iso_steps, 4),
                            "steps": iso_steps}
    hbm = hbm_rooflines(g, hq, hkv, tim_iso, iso_steps, pk["hbm"])

    extra = {}
    cpu = None
    if world > 1 and not args.no_extras:
        # the same workload on ONE GPU (H = 1, local fabric), measured here on rank 0 while
        # the other ranks wait: the N = 1 point of this config's strong-scaling curve (the
        # driver's N = 1 run is BASELINE's C1 line; at N > 2 the job is C2 / C3)
        try:
            extra["same_workload_n1"] = sweep_line(torch, spava, name, local, stream, flush, 3, pk, full=False)
        except Exception as e:  # pragma: no cover
            extra["same_workload_n1"] = {"error": str(e)[:200]}
    if world == 1 and not args.no_extras:
        n = g["n"]
        gen = torch.Generator(device=dev).manual_seed(4321)
        # dense exact attention over the same sequence on one GPU (our kernel, full causal)
        qd = torch.randn((n, hq * DH), generator=gen, device=dev).to(torch.bfloat16)
        kd = torch.randn((n, hkv * DH), generator=gen, device=dev).to(torch.bfloat16)
        vd = torch.randn((n, hkv * DH), generator=gen, device=dev).to(torch.bfloat16)
        segs = [dict(k=kd, v=vd, causal=True)]
        for _ in range(2):
            spava.attention(qd, segs, hq, hkv)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        e0.record()
        for _ in range(reps):
            spava.attention(qd, segs, hq, hkv)
        e1.record()
        torch.cuda.synchronize()
        dms = e0.elapsed_time(e1) / reps
        dflops = 2.0 * n * n * hq * DH
        extra["dense_exact"] = {"tokens_per_s": n / (dms / 1e3), "ms": round(dms, 3),
                                "tflops": round(dflops / (dms / 1e3) / 1e12, 1),
                                "kernel": "attn_fwd_kernel, one causal segment over all n tokens",
                                "spava_speedup": round(dms / ms_max, 2)}
        try:
            import torch.nn.functional as F

            qs = qd.view(1, n, hq, DH).transpose(1, 2)
            ks = kd.view(1, n, hkv, DH).transpose(1, 2)
            vs = vd.view(1, n, hkv, DH).transpose(1, 2)
            F.scaled_dot_product_attention(qs, ks, vs, is_causal=True, enable_gqa=True)
            e0.record()
            for _ in range(reps):
                F.scaled_dot_product_attention(qs, ks, vs, is_causal=True, enable_gqa=True)
            e1.record()
            torch.cuda.synchronize()
            sms = e0.elapsed_time(e1) / reps
            extra["dense_torch_sdpa"] = {"tokens_per_s": n / (sms / 1e3), "ms": round(sms, 3),
                                         "tflops": round(dflops / (sms / 1e3) / 1e12, 1),
                                         "note": "library cross-check (torch SDPA / cuDNN), not our code"}
        except Exception as e:  # pragma: no cover
            extra["dense_torch_sdpa"] = {"error": str(e)[:200]}
        del qd, kd, vd
        # same layer with the tensor-core scorer (score_mode=1): not bit-faithful, so it is
        # reported beside the exact headline with its index agreement on these inputs
        try:
            lcf = spava.LayerConfig.make(g["n_v"], g["n_t"], 1, g["l_a"], g["l_p"], hq, hkv, DH, score_mode=1)
            fabf = spava.Fabric(lcf, local)
            hostf = fabf.host(0)
            outf = torch.empty_like(out)
            self_sel_f = torch.empty_like(sel)
            hostf.set_timing(True)
            fstep = time_layer(torch, hostf, q, k, v, outf, self_sel_f, stream, flush, args.steps, args.warmup)
            fms = sum(fstep) / args.steps
            hostf.set_timing(False)
            hostf.set_timing(2)
            hostf.layer(q, k, v, outf, self_sel_f, stream)
            torch.cuda.synchronize()
            ft = hostf.timing()
            hostf.set_timing(False)
            a_ex, a_f = sel_timed.cpu().numpy(), self_sel_f.cpu().numpy()
            lp = g["l_p"]
            common = sum(len(set(a_ex[r][:lp].tolist()) & set(a_f[r][:lp].tolist())) for r in range(2))
            extra["fast_scoring"] = {
                "tokens_per_s": g["n"] / (fms / 1e3), "ms_per_step": round(fms, 4),
                "score_ms_per_step_isolated": round(ft["score_ms"], 4),
                "index_agreement": round(common / (2 * lp), 6), "indices_differing": 2 * lp - common,
                "note": "score_mode=1: tcgen05 logits + exp2 scorer; same layer otherwise; indices "
                        "compared with the exact scorer on the same inputs"}
            hostf.close()
            fabf.close()
        except Exception as e:  # pragma: no cover
            extra["fast_scoring"] = {"error": str(e)[:200]}
        # the decoder layer around the path (f2): layer_norm, [Wq|Wk|Wv], Spava attention, Wo +
        # residual, layer_norm, ReLU MLP + residual (simhost.cpp:196-207, 431-436) at
        # Qwen2.5-VL-3B widths (d_model 2048, ffn 11008)
        try:
            D, FF = 2048, 11008
            gw = torch.Generator(device=dev).manual_seed(77)
            bfw = lambda *sh, sc: (torch.randn(*sh, generator=gw, device=dev) * sc).to(torch.bfloat16)
            xw = bfw(rows, D, sc=1.0)
            w_qkv = bfw(D, (hq + 2 * hkv) * DH, sc=D ** -0.5)
            w_o = bfw(hq * DH, D, sc=(hq * DH) ** -0.5)
            w_1 = bfw(D, FF, sc=D ** -0.5)
            w_2 = bfw(FF, D, sc=FF ** -0.5)
            g1 = torch.ones(D, device=dev)
            g2 = torch.ones(D, device=dev)
            wsd = host.decoder_layer(xw, w_qkv, w_o, w_1, w_2, g1, g2, stream)
            for _ in range(2):
                host.decoder_layer(xw, w_qkv, w_o, w_1, w_2, g1, g2, stream, wsd)
            torch.cuda.synchronize()
            nd = max(3, min(args.steps, 10))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(nd):
                host.decoder_layer(xw, w_qkv, w_o, w_1, w_2, g1, g2, stream, wsd)
            e1.record(stream)
            torch.cuda.synchronize()
            dms = e0.elapsed_time(e1) / nd
            gemm_fl = 2.0 * rows * D * ((hq + 2 * hkv) * DH + hq * DH / D * D + 2 * FF)
            extra["decoder_layer"] = {
                "tokens_per_s": g["n"] / (dms / 1e3), "ms": round(dms, 3),
                "gemm_tflop": round(gemm_fl / 1e12, 3),
                "note": "x += Spava-attention decoder layer (layer_norm, QKV, Spava, Wo, layer_norm, "
                        "ReLU MLP) at d_model 2048 / ffn 11008"}
            del xw, w_qkv, w_o, w_1, w_2, wsd
        except Exception as e:  # pragma: no cover
            extra["decoder_layer"] = {"error": str(e)[:200]}
        # BASELINE's sweep config (C4, 7B 256K) and the N = 4 / N = 8 configs (C2 64K, C3 128K)
        # at H = 1: the N = 1 points of the multi-GPU lines' workloads
        if not args.no_sweep:
            del q, k, v, out, out_timed
            torch.cuda.empty_cache()
            extra["sweep_h1"] = {}
            for sname in ("C2", "C3", "C4"):
                try:
                    extra["sweep_h1"][sname] = sweep_line(torch, spava, sname, local, stream, flush, 3, pk)
                except Exception as e:  # pragma: no cover
                    extra["sweep_h1"][sname] = {"error": str(e)[:200]}
        if not args.no_cpu:
            os.sched_setaffinity(0, all_cpus)  # the CPU reference gets every host core
            threads = os.cpu_count() or 1
            r = reference_job(g, hq, hkv, 4, 1, threads, max_s=args.cpu_budget)
            cpu = {"value": r["value"], "unit": "tokens/s", "cores": threads, "kind": r["kind"],
                   "sample": r["sample"], "gflops_per_s": round(r["gflops_per_s"], 2),
                   "layer_s": round(r["layer_s"], 1), "fraction_of_layer": round(r["frac"], 4)}

    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic N(0,1) bf16 activations",
        "config": dict(config_dict(name, cfg, g, H),
                       exchange=("local" if world == 1 else
                                 "peer (NVLink stores from the select / merge kernels + epoch flags)"
                                 if fabric == "peer" else "nccl allgather"),
                       exchange_note=fabric_note,
                       l2="flushed (256 MiB write) between timed steps, outside the events"),
        "e2e": {"value": tokens / (e2e_ms / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "host_cpus": numa_cpus,
                "step_ms": [round(x, 3) for x in e2e_step_ms],
                "outputs_equal_device_path": e2e_same,
                "copy_floor_ms": round(copy_floor_ms, 3),
                "copy_floor_note": "the step's H2D + D2H bytes as bare pinned copies on two streams "
                                   "(no compute): the PCIe bound of e2e"},
        "roofline": roofline,
        "hbm_roofline": hbm,
        "cpu_baseline": cpu,
        "gpu_launches": launches,
        "clocks": clocks,
        "wall_s_timed": round(wall, 4),
        "step_ms_minmax": [round(min(step_ms), 4), round(max(step_ms), 4)],
    }
    if ranks is not None:
        line["ranks"] = ranks
    line.update(extra)
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()
    host.close()
    fab.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default: C1 at N <= 2, C2 at N <= 4, C3 (128K tokens) above")
    ap.add_argument("--impl", default="spava", choices=["spava", "reference"])
    ap.add_argument("--fabric", default="peer", choices=["peer", "nccl"],
                    help="N>1 exchange: NVLink peer stores + flags (default) or NCCL allgathers")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds for the CPU baseline sample")
    ap.add_argument("--ref-max-s", type=float, default=150.0,
                    help="reference arm: run the whole layer when it fits this estimate, else a sample")
    ap.add_argument("--no-sweep", action="store_true", help="skip the C2/C3/C4 H=1 lines (N=1)")
    ap.add_argument("--no-self-check", action="store_true", help="N>1: skip the one-GPU comparison")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_spava_arm(args)


if __name__ == "__main__":
    main()
