"""Dev probe: does a small fp64 kernel (2 warps/CTA) co-reside with the attention kernel?
Times attention alone, the fp64 kernel alone, and both on two streams."""
import sys, torch
sys.path.insert(0, '.')
from paper_2601_21444_b200 import spava
from torch.utils.cpp_extension import load_inline
src = r"""
__global__ void dfma_spin(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0;
  for (int i = 0; i < iters; ++i) { a = fma(a, 0.999, 1e-3); b = fma(b, 0.999, 1e-3); }
  if (a + b == 12345.0) out[blockIdx.x] = a;
}
void launch(torch::Tensor out, int blocks, int threads, int iters, int64_t stream) {
  dfma_spin<<<blocks, threads, 0, (cudaStream_t)stream>>>(out.data_ptr<double>(), iters);
}
"""
m = load_inline("cores", cpp_sources="void launch(torch::Tensor out, int blocks, int threads, int iters, int64_t stream);",
                cuda_sources=src.replace('void launch', '#include <torch/extension.h>\nvoid launch'),
                functions=["launch"], extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a"], verbose=False)
dev = torch.device("cuda:0")
hq, hkv, lb = 16, 2, 16064
q = torch.randn(lb, hq * 128, device=dev).to(torch.bfloat16)
k = torch.randn(lb, hkv * 128, device=dev).to(torch.bfloat16)
v = torch.randn(lb, hkv * 128, device=dev).to(torch.bfloat16)
out = torch.empty(4096, dtype=torch.float64, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def attn(): spava.attention(q, [dict(k=k, v=v, causal=True)], hq, hkv, stream=s1)
def dfma(threads): m.launch(out, 4096, threads, 4000, s2.cuda_stream)
def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); torch.cuda.synchronize(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)
for _ in range(2): attn(); dfma(64)
torch.cuda.synchronize()
for th in (64, 128, 256):
    ta = timed(attn); td = timed(lambda: dfma(th)); tb = timed(lambda: (attn(), dfma(th)))
    print(f"threads/CTA {th}: attention {ta:.3f} ms, fp64 kernel {td:.3f} ms, both concurrently {tb:.3f} ms (sum {ta+td:.3f})", flush=True)
