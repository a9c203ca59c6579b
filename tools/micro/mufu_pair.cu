// mufu_pair.cu -- which instruction classes co-issue with MUFU.EX2 on sm_100 (one warp per
// SMSP, 128 independent ex2 per iteration plus N independent ops of one other class).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 mufu_pair.cu -o mufu_pair
#include <cuda_bf16.h>
#include <cstdio>

template <int MODE>
__global__ void k(const float* in, unsigned* out, int iters, long long* cyc) {
  float s[128];
  unsigned o[64];
#pragma unroll
  for (int i = 0; i < 128; ++i) s[i] = in[(threadIdx.x + i) & 255];
#pragma unroll
  for (int i = 0; i < 64; ++i) o[i] = i;
  float mx[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 64; ++j) {
      float a, b;
      if (MODE != 8 && MODE != 10) {
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(a) : "f"(s[2 * j]));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"(s[2 * j + 1]));
      }
      if (MODE == 1) {  // F2FP pack
        __nv_bfloat162 bb = __floats2bfloat162_rn(s[2 * j], s[2 * j + 1]);
        o[j] ^= *reinterpret_cast<unsigned*>(&bb);
      } else if (MODE == 2) {  // FMNMX3
        mx[j & 7] = fmaxf(mx[j & 7], fmaxf(s[2 * j], s[2 * j + 1]));
      } else if (MODE == 3) {  // 2x FFMA2
        float2 t = __ffma2_rn(make_float2(s[2 * j], s[2 * j + 1]), make_float2(1.0001f, 1.0001f), make_float2(0.1f, 0.1f));
        t = __ffma2_rn(t, make_float2(1.0001f, 1.0001f), make_float2(0.1f, 0.1f));
        o[j] ^= __float_as_uint(t.x) + __float_as_uint(t.y);
      } else if (MODE == 4) {  // PRMT
        o[j] ^= __byte_perm(__float_as_uint(s[2 * j]), __float_as_uint(s[2 * j + 1]), 0x7632);
      } else if (MODE == 5) {  // FADD2
        float2 t = __fadd2_rn(make_float2(s[2 * j], s[2 * j + 1]), make_float2(__uint_as_float(o[j]), 1.f));
        o[j] = __float_as_uint(t.x) ^ __float_as_uint(t.y);
      }
      else if (MODE == 6) {  // 2 scalar FADD into 8 accumulators
        mx[j & 7] = __fadd_rn(mx[j & 7], s[2 * j]);
        mx[(j + 4) & 7] = __fadd_rn(mx[(j + 4) & 7], s[2 * j + 1]);
      } else if (MODE == 7) {  // FFMA2 accumulate (p*1 + acc) into 4 pair accumulators
        float2 t = __ffma2_rn(make_float2(s[2 * j], s[2 * j + 1]), make_float2(1.f, 1.f), make_float2(mx[2 * (j & 3)], mx[2 * (j & 3) + 1]));
        mx[2 * (j & 3)] = t.x; mx[2 * (j & 3) + 1] = t.y;
      } else if (MODE == 8) {  // 2 scalar FFMA
        s[2 * j] = fmaf(s[2 * j], 1.0001f, 0.1f);
        s[2 * j + 1] = fmaf(s[2 * j + 1], 1.0001f, 0.1f);
      } else if (MODE == 9) {  // FADD2 into 4 pair accumulators
        float2 t = __fadd2_rn(make_float2(s[2 * j], s[2 * j + 1]), make_float2(mx[2 * (j & 3)], mx[2 * (j & 3) + 1]));
        mx[2 * (j & 3)] = t.x; mx[2 * (j & 3) + 1] = t.y;
      } else if (MODE == 10) {  // 1 FFMA2 (scale)
        float2 t = __ffma2_rn(make_float2(s[2 * j], s[2 * j + 1]), make_float2(1.0001f, 1.0001f), make_float2(0.1f, 0.1f));
        s[2 * j] = t.x; s[2 * j + 1] = t.y;
      }
      if (MODE == 8 || MODE == 10) {
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(a) : "f"(s[2 * j]));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(b) : "f"(s[2 * j + 1]));
      }
      s[2 * j] = a;
      s[2 * j + 1] = b;
    }
  }
  const long long t1 = clock64();
  unsigned acc = 0;
#pragma unroll
  for (int i = 0; i < 64; ++i) acc ^= o[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc ^= __float_as_uint(mx[i]);
#pragma unroll
  for (int i = 0; i < 128; ++i) acc ^= __float_as_uint(s[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / iters;
}

int main() {
  float* in;
  unsigned* out;
  long long* cyc;
  cudaMalloc(&in, 256 * 4);
  cudaMemset(in, 0, 256 * 4);
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  long long h[148];
  auto run = [&](auto kern, const char* name, int warps) {
    kern<<<148, 32 * warps>>>(in, out, 4, cyc);
    kern<<<148, 32 * warps>>>(in, out, 200, cyc);
    cudaDeviceSynchronize();
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-34s warps/SM %2d: %6lld cycles per 128 ex2 per warp\n", name, warps, h[0]);
  };
  for (int w : {4}) {
    run(k<0>, "ex2 only", w);
    run(k<1>, "ex2 + 64 F2FP", w);
    run(k<2>, "ex2 + 64 fmaxf pairs", w);
    run(k<3>, "ex2 + 128 FFMA2", w);
    run(k<4>, "ex2 + 64 PRMT", w);
    run(k<5>, "ex2 + 64 FADD2 (+LOP3)", w);
    run(k<6>, "ex2 + 128 FADD acc", w);
    run(k<7>, "ex2 + 64 FFMA2 acc", w);
    run(k<8>, "ex2(ffma(x)) scalar", w);
    run(k<9>, "ex2 + 64 FADD2 acc", w);
    run(k<10>, "ex2(ffma2(x))", w);
  }
  return 0;
}
