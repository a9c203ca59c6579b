"""Library cross-check: flashinfer single prefill (dense causal, GQA 16/2, d=128, bf16) at 32K."""
import sys, time, torch
n, hq, hkv = 32768, 16, 2
dev = torch.device("cuda:0")
q = torch.randn(n, hq, 128, device=dev, dtype=torch.bfloat16)
k = torch.randn(n, hkv, 128, device=dev, dtype=torch.bfloat16)
v = torch.randn(n, hkv, 128, device=dev, dtype=torch.bfloat16)
import flashinfer
print("flashinfer", flashinfer.__version__, flush=True)
for backend in ("auto", "fa2", "cudnn", "trtllm-gen"):
    try:
        fn = lambda: flashinfer.single_prefill_with_kv_cache(q, k, v, causal=True, backend=backend)
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"backend={backend}: {ms:.3f} ms, {2.0 * n * n * hq * 128 / (ms / 1e3) / 1e12:.0f} TF/s", flush=True)
    except Exception as e:
        print(f"backend={backend}: error {str(e)[:200]}", flush=True)

# Blackwell backends of the ragged-KV batch wrapper: CUTLASS SM100 FMHA and the CuTe-DSL kernel
ws = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
qo = torch.tensor([0, n], dtype=torch.int32, device=dev)
for backend in ("cutlass", "cute-dsl"):
    try:
        w = flashinfer.prefill.BatchPrefillWithRaggedKVCacheWrapper(ws, "NHD", backend=backend)
        w.plan(qo, qo, hq, hkv, 128, causal=True, q_data_type=torch.bfloat16)
        fn = lambda: w.run(q, k, v)
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"ragged backend={backend}: {ms:.3f} ms, {2.0 * n * n * hq * 128 / (ms / 1e3) / 1e12:.0f} TF/s", flush=True)
    except Exception as e:
        print(f"ragged backend={backend}: error {str(e)[:300]}", flush=True)
