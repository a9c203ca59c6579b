// microbenchmark: per-SM throughput of MUFU.EX2, F2FP.BF16 pack, FFMA2, FFMA on sm_100a
#include <cstdio>
#include <cuda_bf16.h>
__global__ void k_ex2(float* out, int iters) {
  float a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[i])); a[i] = y * -0.5f; }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_f2fp(unsigned* out, int iters) {
  float a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; i += 2) { __nv_bfloat162 b = __floats2bfloat162_rn(a[i], a[i + 1]); unsigned u = *(unsigned*)&b; acc ^= u; a[i] = __int_as_float(__float_as_int(a[i]) ^ (u & 1)); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_ffma2(float* out, int iters) {
  float2 a[8]; for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x, i);
  float2 b = make_float2(1.0001f, 0.9999f), c = make_float2(1e-3f, 2e-3f);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], b, c);
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma(float* out, int iters) {
  float a[16]; for (int i = 0; i < 16; ++i) a[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], 1.0001f, 1e-3f);
  float s = 0; for (int i = 0; i < 16; ++i) s += a[i]; out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 1024 * 4 * 4);
  int iters = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w : {4, 8, 16, 32}) {
    int blocks = 148, thr = 32 * w;
    float ms;
    k_ex2<<<blocks, thr>>>(o, 16); cudaEventRecord(e0); k_ex2<<<blocks, thr>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * thr * iters * 8;
    printf("warps/SM %2d  ex2: %.1f /clk/SM", w, ops / (ms * 1e-3) / 148 / 1.965e9);
    k_f2fp<<<blocks, thr>>>((unsigned*)o, 16); cudaEventRecord(e0); k_f2fp<<<blocks, thr>>>((unsigned*)o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("  f2fp(pairs): %.1f /clk/SM", (double)blocks * thr * iters * 4 / (ms * 1e-3) / 148 / 1.965e9);
    k_ffma2<<<blocks, thr>>>(o, 16); cudaEventRecord(e0); k_ffma2<<<blocks, thr>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("  ffma2(fma): %.1f /clk/SM", (double)blocks * thr * iters * 16 / (ms * 1e-3) / 148 / 1.965e9);
    k_ffma<<<blocks, thr>>>(o, 16); cudaEventRecord(e0); k_ffma<<<blocks, thr>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("  ffma: %.1f /clk/SM\n", (double)blocks * thr * iters * 16 / (ms * 1e-3) / 148 / 1.965e9);
  }
}
