// rates.cu -- per-SM issue rates of the instructions the scorer / softmax lean on.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 rates.cu -o rates && ./rates
#include <cuda_bf16.h>
#include <cstdio>

#define BODY(NAME, T, INIT, OP, OUT)                                                    \
  __global__ void NAME(unsigned long long* out, int iters) {                            \
    T a[8];                                                                             \
    for (int i = 0; i < 8; ++i) a[i] = INIT;                                            \
    for (int it = 0; it < iters; ++it) {                                                \
      _Pragma("unroll") for (int i = 0; i < 8; ++i) { OP; }                             \
    }                                                                                   \
    unsigned long long s = 0;                                                           \
    for (int i = 0; i < 8; ++i) s += OUT;                                               \
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;                                     \
  }

BODY(k_ex2f32, float, threadIdx.x * 1e-3f + i,
     asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i])), (unsigned long long)__float_as_uint(a[i]))
BODY(k_ex2bf16x2, unsigned, 0x3f003f00u + threadIdx.x + i,
     asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i])), a[i])
BODY(k_cvt_f64_f32, float, threadIdx.x * 1e-3f + i,
     { double d; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(a[i])); asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(a[i]) : "d"(d)); },
     (unsigned long long)__float_as_uint(a[i]))
BODY(k_dfma, double, threadIdx.x * 1e-3 + i, a[i] = fma(a[i], 0.999, 1e-3),
     (unsigned long long)__double_as_longlong(a[i]))
BODY(k_drint, double, threadIdx.x * 1e-3 + i,
     asm volatile("cvt.rni.f64.f64 %0, %0;" : "+d"(a[i])), (unsigned long long)__double_as_longlong(a[i]))
BODY(k_d2i, double, threadIdx.x * 1e-3 + i,
     { int k; asm volatile("cvt.rni.s32.f64 %0, %1;" : "=r"(k) : "d"(a[i])); asm volatile("cvt.rn.f64.s32 %0, %1;" : "=d"(a[i]) : "r"(k)); },
     (unsigned long long)__double_as_longlong(a[i]))
BODY(k_ffma2, float2, make_float2(threadIdx.x * 1e-3f + i, 1.f),
     a[i] = __ffma2_rn(a[i], make_float2(0.999f, 0.999f), make_float2(1e-3f, 1e-3f)),
     (unsigned long long)__float_as_uint(a[i].x))
BODY(k_ffma, float, threadIdx.x * 1e-3f + i, a[i] = fmaf(a[i], 0.999f, 1e-3f),
     (unsigned long long)__float_as_uint(a[i]))
BODY(k_f2fp, unsigned, threadIdx.x + i,
     { __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(a[i]), __uint_as_float(a[i] + 7)); a[i] = *(unsigned*)&b; },
     a[i])
BODY(k_dmul, double, threadIdx.x * 1e-3 + i, a[i] = a[i] * 0.999,
     (unsigned long long)__double_as_longlong(a[i]))
BODY(k_ddiv, double, threadIdx.x * 1e-3 + i + 1.0, a[i] = 1.0 / a[i] + 0.5,
     (unsigned long long)__double_as_longlong(a[i]))

typedef void (*K)(unsigned long long*, int);
int main2();
int main() {
  main2();
  unsigned long long* o;
  cudaMalloc(&o, 148 * 4 * 1024 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct { const char* n; K k; double per; } ks[] = {
      {"ex2.approx.f32 (exps)", k_ex2f32, 1}, {"ex2.approx.bf16x2 (exps)", k_ex2bf16x2, 2},
      {"cvt f32->f64->f32 (pairs)", k_cvt_f64_f32, 1}, {"dfma", k_dfma, 1}, {"dmul", k_dmul, 1},
      {"cvt.rni.f64.f64", k_drint, 1}, {"cvt f64->s32->f64 (pairs)", k_d2i, 1},
      {"ffma2 (fmas)", k_ffma2, 2}, {"ffma", k_ffma, 1}, {"f2fp bf16x2 pack", k_f2fp, 1},
      {"1/x fp64 + add", k_ddiv, 1}};
  int blocks = 148 * 4, thr = 256, iters = 2048;
  for (auto& k : ks) {
    float ms;
    k.k<<<blocks, thr>>>(o, 8);
    cudaEventRecord(e0);
    k.k<<<blocks, thr>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * thr * iters * 8 * k.per;
    printf("%-28s %8.1f /clk/SM (at 1.965 GHz)\n", k.n, ops / (ms * 1e-3) / 148 / 1.965e9);
  }
  return 0;
}
// (appended) f16x2 ex2: one MUFU op for two halves?
BODY(k_ex2f16x2, unsigned, 0x3c003c00u + threadIdx.x + i,
     asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i])), a[i])
int main2() {
  unsigned long long* o;
  cudaMalloc(&o, 148 * 4 * 1024 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int blocks = 148 * 4, thr = 256, iters = 2048;
  float ms;
  k_ex2f16x2<<<blocks, thr>>>(o, 8);
  cudaEventRecord(e0);
  k_ex2f16x2<<<blocks, thr>>>(o, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("ex2.approx.f16x2 (exps)        %8.1f /clk/SM\n", (double)blocks * thr * iters * 16 / (ms * 1e-3) / 148 / 1.965e9);
  return 0;
}
