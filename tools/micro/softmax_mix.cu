// softmax_mix.cu -- cycles per 128-element softmax row chunk for one warp per SMSP, for
// several instruction mixes (is the attention softmax body MUFU-bound or mix-bound?).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 softmax_mix.cu -o softmax_mix
#include <cuda_bf16.h>
#include <cstdio>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  const float2 magic = make_float2(0x1.8p23f, 0x1.8p23f);
  const float2 t = __fadd2_rn(x, magic);
  const float2 r = __fadd2_rn(t, make_float2(-0x1.8p23f, -0x1.8p23f));
  const float2 f = __fadd2_rn(x, make_float2(-r.x, -r.y));
  float2 p = __ffma2_rn(make_float2(0x1.c4c0d0p-5f, 0x1.c4c0d0p-5f), f, make_float2(0x1.f0e306p-3f, 0x1.f0e306p-3f));
  p = __ffma2_rn(p, f, make_float2(0x1.62f0d0p-1f, 0x1.62f0d0p-1f));
  p = __ffma2_rn(p, f, make_float2(0x1.fff66cp-1f, 0x1.fff66cp-1f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// MODE 0: MUFU only; 1: full mix (ffma2 scale, mufu, fadd2 sum, f2fp pack, fmnmx);
// 2: mix with 1 of 4 pairs emulated; 3: mix without pack; 4: mix with 1 of 8 pairs emulated
template <int MODE>
__global__ void k(const float* in, unsigned* out, int iters, long long* cyc) {
  float s[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) s[i] = in[(threadIdx.x + i) & 255] * 0.01f;
  float m = 0.f;
  float2 acc = make_float2(0.f, 0.f);
  unsigned pk = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float mx = -1e30f;
    unsigned pkv[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) {
      float2 x = make_float2(s[2 * j], s[2 * j + 1]);
      if (MODE != 0) mx = fmaxf(mx, fmaxf(x.x, x.y));
      x = __ffma2_rn(x, make_float2(1.4427f, 1.4427f), make_float2(-m, -m));
      float2 p;
      if ((MODE == 2 && (j & 3) == 3) || (MODE == 4 && (j & 7) == 7))
        p = exp2_poly2(x);
      else
        p = make_float2(ex2(x.x), ex2(x.y));
      if (MODE != 0) acc = __fadd2_rn(acc, p);
      if (MODE == 5 || MODE == 6) {
        const unsigned a = __float_as_uint(p.x) + (MODE == 5 ? 0x8000u : 0u);
        const unsigned b = __float_as_uint(p.y) + (MODE == 5 ? 0x8000u : 0u);
        pkv[j] = __byte_perm(a, b, 0x7632);
      } else if (MODE == 1 || MODE == 2 || MODE == 4) {
        __nv_bfloat162 b = __floats2bfloat162_rn(p.x, p.y);
        pkv[j] = *reinterpret_cast<unsigned*>(&b);
      } else {
        pkv[j] = __float_as_uint(p.x) ^ __float_as_uint(p.y);
      }
      s[2 * j] = p.x - 0.5f;  // keep the values live and changing
      s[2 * j + 1] = p.y - 0.5f;
    }
    m = mx * 1e-3f;
#pragma unroll
    for (int w = 32; w >= 1; w >>= 1)
#pragma unroll
      for (int j = 0; j < w; ++j) pkv[j] ^= pkv[j + w];
    pk ^= pkv[0];
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = pk ^ __float_as_uint(acc.x + acc.y);
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
    printf("%-40s warps/SM %2d: %6lld cycles per 128-element row-chunk per warp\n", name, warps, h[0]);
  };
  for (int w : {4, 8}) {
    run(k<0>, "mufu only", w);
    run(k<1>, "full mix", w);
    run(k<3>, "mix, no bf16 pack", w);
    run(k<5>, "mix, int round+prmt pack", w);
    run(k<6>, "mix, prmt truncation pack", w);
    run(k<2>, "mix, 1/4 pairs emulated", w);
    run(k<4>, "mix, 1/8 pairs emulated", w);
  }
  return 0;
}
