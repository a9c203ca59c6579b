"""Is the per-host spread of a simulated H-host layer real or a clock artifact?  Runs the
sim (sim_layer_timed: every host's phases alone, in host order) while a thread samples the
SM clock and throttle reasons (NVML, ~1 ms), and prints per-host times with the clock
range seen -- dev tool.

    python tools/sim_clocks.py [C4] [hosts]
"""
import json
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2601_21444_b200 import spava  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "C4"
H = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = bench.CONFIGS[cfg_name]
dev = torch.device("cuda:0")
hq, hkv = cfg["hq"], cfg["hkv"]
pynvml.nvmlInit()
hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
samples, stop = [], threading.Event()


def sampler():
    while not stop.is_set():
        samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(hnd)))
        time.sleep(0.001)


g = bench.geometry(cfg, H, True)
lc = spava.LayerConfig.make(g["n_v"], g["n_t"], H, g["l_a"], g["l_p"], hq, hkv, 128)
fab = spava.Fabric(lc, 0)
hosts = [fab.host(h) for h in range(H)]
gen = torch.Generator(device=dev).manual_seed(7)
rows = hosts[0].rows
qs = [torch.randn(rows, hq * 128, device=dev, generator=gen).to(torch.bfloat16) for _ in range(H)]
ks = [torch.randn(rows, hkv * 128, device=dev, generator=gen).to(torch.bfloat16) for _ in range(H)]
vs = [torch.randn(rows, hkv * 128, device=dev, generator=gen).to(torch.bfloat16) for _ in range(H)]
outs = [torch.empty(rows, hq * 128, dtype=torch.bfloat16, device=dev) for _ in range(H)]
for _ in range(2):
    fab.sim_layer_timed(hosts, qs, ks, vs, outs)
for gap in (0.0, 2.0):
    th = threading.Thread(target=sampler)
    samples.clear()
    stop.clear()
    th.start()
    runs = []
    for _ in range(5):
        if gap:
            torch.cuda.synchronize()
            time.sleep(gap)
        runs.append(fab.sim_layer_timed(hosts, qs, ks, vs, outs))
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = [min(r[h] for r in runs) for h in range(H)]
    clk = sorted(s[1] for s in samples)
    reasons = sorted({s[2] for s in samples})
    print(json.dumps({"config": cfg_name, "hosts": H, "idle_gap_s": gap, "ms_per_host": [round(x, 3) for x in ms],
                      "max_over_min": round(max(ms) / min(ms), 3),
                      "runs_ms_per_host": [[round(x, 2) for x in r] for r in runs],
                      "sm_mhz_min_med_max": [clk[0], clk[len(clk) // 2], clk[-1]],
                      "throttle_reason_masks": [hex(x) for x in reasons]}), flush=True)
for h in hosts:
    h.close()
fab.close()
