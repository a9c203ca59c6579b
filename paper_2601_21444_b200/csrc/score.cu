// score.cu -- query-aware importance scoring of one context block ("exact" mode).
//
// Reproduces score_block (simhost.cpp:209-224) -> score_context (approx.cpp:15-69) ->
// matmul_nt (matrix.cpp:73-86) operation by operation:
//   l_hij   = fp32 sum_c q[i,h,c]*k[j,h',c], c ascending        (h' = h / (hq/hkv))
//   mx_hi   = max_j double(l_hij) * scale   (fp64)
//   sum_hi  = sum_j exp(double(l_hij)*scale - mx_hi)            (fp64)
//   part_hj = ((0 + p_h0j) + p_h1j) + ...,  p = float(exp(..)/sum_hi)   (fp32, i ascending)
//   score_j = ((0 + part_0j) + part_1j) + ...                   (fp32, h ascending)
// Inputs are bf16, so every q*k product is exact in fp32 and one FFMA per term equals
// the reference's separate multiply and add bit for bit.  The only difference from the
// CPU reference is the *order* of the fp64 sum_hi (a parallel reduction here) and
// CUDA's fp64 exp vs glibc's: both perturb p below 1 fp32 ulp in rare elements.
// Three kernels: logits (CUDA-core SGEMM tile, c-sequential chains), per-row fp64
// statistics, and an ordered column sum fused with the ordered head sum.
#include <cuda_bf16.h>

#include "spava_internal.h"

namespace spava {

namespace {

constexpr int kLogitKeys = 64;   // keys per CTA
constexpr int kLogitRows = 128;  // query rows per pass
constexpr int kDh = 128;

inline long long ld_logits(int l_b) { return (static_cast<long long>(l_b) + 63) / 64 * 64; }

__device__ __forceinline__ float bf2f(__nv_bfloat16 x) { return __bfloat162float(x); }

// L[h][i][j] for j in [j0, j0+64), all i.  grid (ceil(l_b/64), hq), 256 threads.
__global__ void __launch_bounds__(256) logits_kernel(const __nv_bfloat16* __restrict__ q,
                                                     long long ldq, int n_t,
                                                     const __nv_bfloat16* __restrict__ k,
                                                     long long ldk, int l_b, int hq, int hkv,
                                                     float* __restrict__ L, long long ldL) {
  extern __shared__ float sm[];
  float* Ks = sm;                           // [kDh][kLogitKeys]
  float* Qs = sm + kDh * kLogitKeys;        // [kDh][kLogitRows]
  const int h = blockIdx.y;
  const int hk = h / (hq / hkv);
  const int j0 = blockIdx.x * kLogitKeys;
  const int tid = threadIdx.x;
  // K tile, transposed to [c][j]; lanes walk j so the smem stores are conflict-free.
  for (int idx = tid; idx < kLogitKeys * (kDh / 8); idx += 256) {
    const int j = idx % kLogitKeys, c0 = (idx / kLogitKeys) * 8;
    uint4 raw = make_uint4(0, 0, 0, 0);
    if (j0 + j < l_b)
      raw = *reinterpret_cast<const uint4*>(k + static_cast<long long>(j0 + j) * ldk + hk * kDh + c0);
    const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
    for (int t = 0; t < 8; ++t) Ks[(c0 + t) * kLogitKeys + j] = bf2f(e[t]);
  }
  const int tx = tid % 16;  // 4 keys each
  const int ty = tid / 16;  // 8 rows each
  for (int r0 = 0; r0 < n_t; r0 += kLogitRows) {
    __syncthreads();
    for (int idx = tid; idx < kLogitRows * (kDh / 8); idx += 256) {
      const int i = idx % kLogitRows, c0 = (idx / kLogitRows) * 8;
      uint4 raw = make_uint4(0, 0, 0, 0);
      if (r0 + i < n_t)
        raw = *reinterpret_cast<const uint4*>(q + static_cast<long long>(r0 + i) * ldq + h * kDh + c0);
      const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
      for (int t = 0; t < 8; ++t) Qs[(c0 + t) * kLogitRows + i] = bf2f(e[t]);
    }
    __syncthreads();
    float acc[8][4];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
#pragma unroll 4
    for (int c = 0; c < kDh; ++c) {  // ascending c: each acc is one sequential chain
      const float4 q0 = *reinterpret_cast<const float4*>(&Qs[c * kLogitRows + ty * 8]);
      const float4 q1 = *reinterpret_cast<const float4*>(&Qs[c * kLogitRows + ty * 8 + 4]);
      const float4 kv = *reinterpret_cast<const float4*>(&Ks[c * kLogitKeys + tx * 4]);
      const float qa[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
      const float ka[4] = {kv.x, kv.y, kv.z, kv.w};
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = __fmaf_rn(qa[a], ka[b], acc[a][b]);
    }
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int i = r0 + ty * 8 + a;
      if (i < n_t)
        *reinterpret_cast<float4*>(&L[(static_cast<long long>(h) * n_t + i) * ldL + j0 + tx * 4]) =
            make_float4(acc[a][0], acc[a][1], acc[a][2], acc[a][3]);
    }
  }
}

__device__ __forceinline__ bool is_pad(const uint8_t* pad, int n_valid, int j) {
  return j >= n_valid || (pad && pad[j]);
}

// One warp per (h, i): mx = double(max_j l)*scale (monotone, == max of products), sum.
__global__ void rowstats_kernel(const float* __restrict__ L, long long ldL, int n_rows, int l_b,
                                const uint8_t* __restrict__ pad, int n_valid, float scale,
                                double2* __restrict__ stats) {
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  const float* lr = L + static_cast<long long>(row) * ldL;
  float mxf = -INFINITY;
  for (int j = lane; j < l_b; j += 32)
    if (!is_pad(pad, n_valid, j)) mxf = fmaxf(mxf, lr[j]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mxf = fmaxf(mxf, __shfl_xor_sync(0xffffffffu, mxf, o));
  const double mx = static_cast<double>(mxf) * static_cast<double>(scale);
  double sum = 0.0;
  if (mxf != -INFINITY) {
    for (int j = lane; j < l_b; j += 32)
      if (!is_pad(pad, n_valid, j))
        sum += exp(__dsub_rn(__dmul_rn(static_cast<double>(lr[j]), static_cast<double>(scale)), mx));
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  }
  if (lane == 0) stats[row] = make_double2(mxf == -INFINITY ? -INFINITY : mx, sum);
}

// block (32, 8): thread (x, y) handles key j = blockIdx.x*32+x for heads y, y+8, ...
__global__ void colsum_kernel(const float* __restrict__ L, long long ldL, int n_t, int l_b, int hq,
                              const double2* __restrict__ stats, const uint8_t* __restrict__ pad,
                              int n_valid, float scale, int softmax, float* __restrict__ scores) {
  __shared__ float part[32][33];
  const int x = threadIdx.x, y = threadIdx.y;
  const int j = blockIdx.x * 32 + x;
  const bool inb = j < l_b;
  for (int h = y; h < hq; h += 8) {
    float acc = 0.f;
    if (inb) {
      for (int i = 0; i < n_t; ++i) {
        const float l = L[(static_cast<long long>(h) * n_t + i) * ldL + j];
        if (softmax) {
          const double2 st = stats[h * n_t + i];
          const double e = exp(__dsub_rn(__dmul_rn(static_cast<double>(l), static_cast<double>(scale)), st.x));
          acc = __fadd_rn(acc, __double2float_rn(__ddiv_rn(e, st.y)));
        } else {
          acc = __fadd_rn(acc, __fmul_rn(l, scale));
        }
      }
    }
    part[h][x] = acc;
  }
  __syncthreads();
  if (y == 0 && inb) {
    float total = 0.f;
    for (int h = 0; h < hq; ++h) total = __fadd_rn(total, part[h][x]);
    // pad keys -> -inf (approx.cpp:64-66); a block without visible keys is all pads
    scores[j] = is_pad(pad, n_valid, j) ? -INFINITY : total;
  }
}

}  // namespace

size_t score_workspace_bytes(int n_t, int l_b, int hq) {
  const size_t L = static_cast<size_t>(hq) * n_t * ld_logits(l_b) * sizeof(float);
  const size_t st = static_cast<size_t>(hq) * n_t * sizeof(double2);
  return L + st + 256;
}

cudaError_t launch_score_exact(const void* q, long long ldq, int n_t, const void* k,
                               long long ldk, int l_b, const uint8_t* pad, int n_valid, int hq,
                               int hkv, int dh, int softmax, float* scores, void* ws,
                               size_t ws_bytes, cudaStream_t stream) {
  if (dh != kDh || hq < 1 || hkv < 1 || hq % hkv || hq > 32 || n_t < 1)
    return cudaErrorInvalidValue;
  if (l_b <= 0) return cudaSuccess;
  if (ws_bytes < score_workspace_bytes(n_t, l_b, hq)) return cudaErrorInvalidValue;
  const long long ldL = ld_logits(l_b);
  float* L = static_cast<float*>(ws);
  double2* stats = reinterpret_cast<double2*>(
      reinterpret_cast<uintptr_t>(L + static_cast<size_t>(hq) * n_t * ldL + 63) & ~uintptr_t(63));
  const float scale = 1.0f / sqrtf(static_cast<float>(dh));
  static bool attr = false;
  const int smem = (kDh * kLogitKeys + kDh * kLogitRows) * sizeof(float);
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(logits_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 g1((l_b + kLogitKeys - 1) / kLogitKeys, hq);
  logits_kernel<<<g1, 256, smem, stream>>>(static_cast<const __nv_bfloat16*>(q), ldq, n_t,
                                            static_cast<const __nv_bfloat16*>(k), ldk, l_b, hq,
                                            hkv, L, ldL);
  const int rows = hq * n_t;
  if (softmax) rowstats_kernel<<<(rows + 7) / 8, 256, 0, stream>>>(L, ldL, rows, l_b, pad, n_valid, scale, stats);
  colsum_kernel<<<(l_b + 31) / 32, dim3(32, 8), 0, stream>>>(L, ldL, n_t, l_b, hq, stats, pad, n_valid,
                                                             scale, softmax, scores);
  return cudaGetLastError();
}

}  // namespace spava
