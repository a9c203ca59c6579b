#include <cstdio>
#include <cuda_bf16.h>
// mixed MUFU + F2FP: 8 ex2 + 4 f2fp per iteration
__global__ void k_mix(unsigned* out, int iters) {
  float a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i])); a[i] = y * -0.5f; }
#pragma unroll
    for (int i = 0; i < 8; i += 2) { __nv_bfloat162 b = __floats2bfloat162_rn(a[i], a[i + 1]); acc += *(unsigned*)&b; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_ex2bf(unsigned* out, int iters) {
  unsigned a[8]; for (int i = 0; i < 8; ++i) a[i] = 0x3f003f00u + threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) { unsigned y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(a[i])); a[i] = y ^ 0x80008000u; }
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += a[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  unsigned* o; cudaMalloc(&o, 148 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096, blocks = 148, thr = 512; float ms;
  k_mix<<<blocks, thr>>>(o, 16); cudaEventRecord(e0); k_mix<<<blocks, thr>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  double per = (double)blocks * thr * iters / (ms * 1e-3) / 148 / 1.965e9;  // iterations per clk per SM
  printf("mix: %.2f cycles per thread-iteration-group (8 ex2 + 4 f2fp) per 32 threads -> ex2 %.1f/clk, pairs %.1f/clk\n", 32.0 / per, per * 8, per * 4);
  k_ex2bf<<<blocks, thr>>>(o, 16); cudaEventRecord(e0); k_ex2bf<<<blocks, thr>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  printf("ex2.bf16x2: %.1f exps/clk/SM\n", (double)blocks * thr * iters * 16 / (ms * 1e-3) / 148 / 1.965e9);
}
