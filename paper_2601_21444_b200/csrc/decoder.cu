// decoder.cu -- the step on either side of the Spava attention:
// the reference decoder layer (simhost.cpp:196-207 project, :431-436 finish_group,
// model.cpp:60-75, matrix.cpp:128-150 layer_norm) around spava_host_layer:
//   xn = norm ? layer_norm(x, g1) : x
//   q, k, v = xn Wq, xn Wk, xn Wv                 (one GEMM against [Wq | Wk | Wv])
//   a = Spava attention layer (q, k, v)           (spava_host_layer, this library)
//   x += a Wo
//   f = norm ? layer_norm(x, g2) : x
//   x += relu(f W1) W2
// Rows are the host-local rows [anchor | lo | hi | query]; every operation is row-wise or
// a GEMM over rows, so applying it to the whole buffer equals the reference's per-part
// project / finish_group calls.  GEMMs are this library's tcgen05 kernel (gemm.cu: fp32
// accumulation in TMEM, ReLU and residual in its epilogue, q/k/v written by one GEMM);
// layer_norm is a one-warp-per-row kernel.
#include <cuda_bf16.h>

#include "spava_internal.h"

namespace spava {

namespace {

// one warp per row: mean / variance in fp32 over the row, out = (x - mean) * rsqrt(var +
// 1e-5) * g  (matrix.cpp:128-150 with the reference's eps)
__global__ void layer_norm_kernel(const __nv_bfloat16* x, long long ldx, const float* g, int d,
                                  __nv_bfloat16* y, long long ldy, int rows) {
  const int r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const __nv_bfloat16* xr = x + r * ldx;
  float s = 0.f, s2 = 0.f;
  for (int j = lane * 2; j < d; j += 64) {
    const float2 v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(xr + j));
    s += v.x + v.y;
    s2 += v.x * v.x + v.y * v.y;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  const float mean = s / d;
  const float var = fmaxf(s2 / d - mean * mean, 0.f);
  const float inv = rsqrtf(var + 1e-5f);
  __nv_bfloat16* yr = y + r * ldy;
  for (int j = lane * 2; j < d; j += 64) {
    const float2 v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(xr + j));
    const float g0 = g ? g[j] : 1.f, g1 = g ? g[j + 1] : 1.f;
    *reinterpret_cast<__nv_bfloat162*>(yr + j) =
        __floats2bfloat162_rn((v.x - mean) * inv * g0, (v.y - mean) * inv * g1);
  }
}

}  // namespace

cudaError_t launch_layer_norm(const void* x, long long ldx, const float* g, int d, void* y,
                              long long ldy, int rows, cudaStream_t stream) {
  if (d % 2 || rows <= 0) return rows <= 0 ? cudaSuccess : cudaErrorInvalidValue;
  layer_norm_kernel<<<(rows + 7) / 8, 256, 0, stream>>>(static_cast<const __nv_bfloat16*>(x), ldx, g, d,
                                                        static_cast<__nv_bfloat16*>(y), ldy, rows);
  return cudaGetLastError();
}

}  // namespace spava
