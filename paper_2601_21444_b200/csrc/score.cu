// score.cu -- query-aware importance scoring of context blocks ("exact" mode).
//
// Reproduces score_block (simhost.cpp:209-224) -> score_context (approx.cpp:15-69) ->
// matmul_nt (matrix.cpp:73-86) operation by operation:
//   l_hij   = fp32 sum_c q[i,h,c]*k[j,h',c], c ascending        (h' = h / (hq/hkv))
//   x_hij   = double(l_hij) * double(scale)                     (exact in fp64)
//   mx_hi   = max_j x_hij ;  sum_hi = sum_j exp(x_hij - mx_hi)  (fp64)
//   part_hj = ((0 + p_h0j) + p_h1j) + ...,  p = float(exp(x - mx)/sum)   (fp32, i ascending)
//   score_j = ((0 + part_0j) + part_1j) + ...                   (fp32, h ascending)
// Inputs are bf16, so every q*k product is exact in fp32 and one FFMA per term equals
// the reference's multiply-then-add bit for bit; the logit chains run c-ascending.
// Differences from the CPU reference are confined to (a) the summation order of the
// fp64 normaliser sum_hi (tile partials here) and (b) CUDA's fp64 exp vs glibc's; both
// move p only when it lies within ~1e-15 of an fp32 rounding midpoint.
// p = float(e/sum) is evaluated as e*(1/sum) with an exact-division fallback whenever
// the product lands within a few fp64 ulps of an fp32 midpoint (or in fp32 subnormals),
// so it equals the correctly rounded quotient.
//
// Kernels (both blocks of a host in one launch each):
//   logits_kernel : 128x128 CUDA-core SGEMM tile per CTA (8x8 register micro-tiles,
//                   c-chunks double-buffered in smem), writes L and per-(row, key-tile)
//                   softmax partials (tile max, fp64 sum of exp relative to it).
//   stats_kernel  : combines the partials into (mx, sum, 1/sum) per (block, head, row).
//   colsum_kernel : ordered column sums over query rows, then ordered sum over heads.
#include <cuda_bf16.h>

#include "spava_internal.h"

namespace spava {

namespace {

constexpr int kDh = 128;
constexpr int kTM = 128;  // query rows per CTA
constexpr int kTN = 128;  // keys per CTA
constexpr int kKC = 16;   // c-chunk
constexpr int kThr = 256;

inline long long ld_logits(int l_b) { return (static_cast<long long>(l_b) + kTN - 1) / kTN * kTN; }
inline int n_ktiles(int l_b) { return (l_b + kTN - 1) / kTN; }

struct ScoreArgs {
  const __nv_bfloat16* q;  // [n_t x ldq]
  long long ldq;
  const __nv_bfloat16* k[2];
  long long ldk;
  int n_valid[2];
  const uint8_t* pad[2];
  float* scores[2];
  int nblk, n_t, l_b, hq, hkv, softmax;
  float scale;
  float* L;          // [nblk][hq][n_t][ldL]
  long long ldL;
  double2* part;     // [nblk][hq][n_t][ntiles]  (tile max x, tile sum)
  double* stats;     // [nblk][hq][n_t][3]       (mx, sum, 1/sum)
  int ntiles;
};

__device__ __forceinline__ bool is_pad(const uint8_t* pad, int n_valid, int j) {
  return j >= n_valid || (pad && pad[j]);
}

__device__ __forceinline__ void load_chunk(const ScoreArgs& a, const __nv_bfloat16* k, int h, int hk,
                                           int r0, int j0, int c0, float4 (&qr)[2], float4 (&kr)[2]) {
  // 256 threads x 8 elements = 128 rows x 16 c for Q, same for K (lane walks the row
  // dimension so the transposed smem stores are conflict-free)
  const int tid = threadIdx.x;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int e = tid + u * kThr;  // 0..511: row = e % 128, c-quad = e / 128
    const int row = e % kTM, cq = (e / kTM) * 4;
    float4 qv = make_float4(0.f, 0.f, 0.f, 0.f), kv = qv;
    if (r0 + row < a.n_t) {
      const uint2 raw = *reinterpret_cast<const uint2*>(a.q + static_cast<long long>(r0 + row) * a.ldq +
                                                        h * kDh + c0 + cq);
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&raw);
      const float2 f0 = __bfloat1622float2(b[0]), f1 = __bfloat1622float2(b[1]);
      qv = make_float4(f0.x, f0.y, f1.x, f1.y);
    }
    if (j0 + row < a.l_b) {
      const uint2 raw = *reinterpret_cast<const uint2*>(k + static_cast<long long>(j0 + row) * a.ldk +
                                                        hk * kDh + c0 + cq);
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&raw);
      const float2 f0 = __bfloat1622float2(b[0]), f1 = __bfloat1622float2(b[1]);
      kv = make_float4(f0.x, f0.y, f1.x, f1.y);
    }
    qr[u] = qv;
    kr[u] = kv;
  }
}

__device__ __forceinline__ void store_chunk(float* Qs, float* Ks, const float4 (&qr)[2],
                                            const float4 (&kr)[2]) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int e = tid + u * kThr;
    const int row = e % kTM, cq = (e / kTM) * 4;
    Qs[(cq + 0) * kTM + row] = qr[u].x;
    Qs[(cq + 1) * kTM + row] = qr[u].y;
    Qs[(cq + 2) * kTM + row] = qr[u].z;
    Qs[(cq + 3) * kTM + row] = qr[u].w;
    Ks[(cq + 0) * kTN + row] = kr[u].x;
    Ks[(cq + 1) * kTN + row] = kr[u].y;
    Ks[(cq + 2) * kTN + row] = kr[u].z;
    Ks[(cq + 3) * kTN + row] = kr[u].w;
  }
}

// grid (ntiles, hq, nblk), 256 threads: L tile 128 rows x 128 keys, rows chunked by 128.
__global__ void __launch_bounds__(kThr, 2) logits_kernel(const __grid_constant__ ScoreArgs a) {
  __shared__ __align__(16) float Qs[2][kKC * kTM];
  __shared__ __align__(16) float Ks[2][kKC * kTN];
  const int tile = blockIdx.x, h = blockIdx.y, blk = blockIdx.z;
  const int hk = h / (a.hq / a.hkv);
  const int j0 = tile * kTN;
  const __nv_bfloat16* k = a.k[blk];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const double sc = static_cast<double>(a.scale);
  for (int r0 = 0; r0 < a.n_t; r0 += kTM) {
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    float4 qr[2], kr[2];
    load_chunk(a, k, h, hk, r0, j0, 0, qr, kr);
    store_chunk(Qs[0], Ks[0], qr, kr);
    __syncthreads();
    constexpr int kChunks = kDh / kKC;
    for (int ch = 0; ch < kChunks; ++ch) {
      const int cur = ch & 1;
      if (ch + 1 < kChunks) load_chunk(a, k, h, hk, r0, j0, (ch + 1) * kKC, qr, kr);
#pragma unroll
      for (int c = 0; c < kKC; ++c) {  // ascending c within the chunk, chunks ascending
        const float4 qa = *reinterpret_cast<const float4*>(&Qs[cur][c * kTM + ty * 4]);
        const float4 qb = *reinterpret_cast<const float4*>(&Qs[cur][c * kTM + 64 + ty * 4]);
        const float4 ka = *reinterpret_cast<const float4*>(&Ks[cur][c * kTN + tx * 4]);
        const float4 kb = *reinterpret_cast<const float4*>(&Ks[cur][c * kTN + 64 + tx * 4]);
        const float qv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
        const float kv[8] = {ka.x, ka.y, ka.z, ka.w, kb.x, kb.y, kb.z, kb.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = __fmaf_rn(qv[i], kv[j], acc[i][j]);
      }
      if (ch + 1 < kChunks) {
        store_chunk(Qs[cur ^ 1], Ks[cur ^ 1], qr, kr);
        __syncthreads();
      }
    }
    // ---- epilogue: L and per-(row, tile) softmax partials
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = r0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
      const bool rok = row < a.n_t;
      float* Lr = a.L + ((static_cast<long long>(blk) * a.hq + h) * a.n_t + (rok ? row : 0)) * a.ldL + j0;
      if (rok) {
        *reinterpret_cast<float4*>(Lr + tx * 4) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        *reinterpret_cast<float4*>(Lr + 64 + tx * 4) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
      }
      if (a.softmax) {
        float mxf = -INFINITY;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int key = j0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
          if (!is_pad(a.pad[blk], a.n_valid[blk], key)) mxf = fmaxf(mxf, acc[i][j]);
        }
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) mxf = fmaxf(mxf, __shfl_xor_sync(0xffffffffu, mxf, o));
        double s = 0.0;
        const double mt = static_cast<double>(mxf) * sc;
        if (mxf != -INFINITY) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int key = j0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
            if (!is_pad(a.pad[blk], a.n_valid[blk], key))
              s += exp(__dsub_rn(__dmul_rn(static_cast<double>(acc[i][j]), sc), mt));
          }
        }
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (tx == 0 && rok)
          a.part[((static_cast<long long>(blk) * a.hq + h) * a.n_t + row) * a.ntiles + tile] =
              make_double2(mxf == -INFINITY ? -INFINITY : mt, s);
      }
    }
    __syncthreads();
  }
}

// one warp per (blk, h, i): mx = max_t M_t ; sum = sum_t S_t * exp(M_t - mx)
__global__ void stats_kernel(const __grid_constant__ ScoreArgs a) {
  const long long rows = static_cast<long long>(a.nblk) * a.hq * a.n_t;
  const long long r = static_cast<long long>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const double2* p = a.part + r * a.ntiles;
  double mx = -INFINITY;
  for (int t = lane; t < a.ntiles; t += 32) mx = fmax(mx, p[t].x);
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  double s = 0.0;
  if (mx != -INFINITY)
    for (int t = lane; t < a.ntiles; t += 32)
      if (p[t].x != -INFINITY) s += p[t].y * exp(p[t].x - mx);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    a.stats[r * 3 + 0] = mx;
    a.stats[r * 3 + 1] = s;
    a.stats[r * 3 + 2] = 1.0 / s;
  }
}

// float(e / sum) with e*(1/sum) fast path; exact division when the product is within
// 8 fp64 ulps of an fp32 rounding midpoint or below FLT_MIN (different rounding point).
__device__ __forceinline__ float prob_f32(double e, double sum, double rinv) {
  const double y = __dmul_rn(e, rinv);
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(y));
  const long long low = static_cast<long long>(b & ((1ull << 29) - 1));
  const bool near_mid = (low > (1ll << 28) - 8) && (low < (1ll << 28) + 8);
  if (near_mid || y < 1.1754943508222875e-38) return __double2float_rn(__ddiv_rn(e, sum));
  return __double2float_rn(y);
}

// block (32, 8): thread (x, y) owns key j = blockIdx.x*32+x of block blockIdx.y for heads
// y, y+8, ...; rows i ascending per head, heads ascending for the total.
__global__ void __launch_bounds__(256) colsum_kernel(const __grid_constant__ ScoreArgs a) {
  __shared__ float part[32][33];
  const int x = threadIdx.x, y = threadIdx.y, blk = blockIdx.y;
  const int j = blockIdx.x * 32 + x;
  const bool inb = j < a.l_b;
  const double sc = static_cast<double>(a.scale);
  for (int h = y; h < a.hq; h += 8) {
    float acc = 0.f;
    if (inb) {
      const long long hb = (static_cast<long long>(blk) * a.hq + h) * a.n_t;
      const float* L = a.L + hb * a.ldL + j;
      const double* st = a.stats + hb * 3;
      if (a.softmax) {
        int i = 0;
        for (; i + 4 <= a.n_t; i += 4) {
          float p[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double e = exp(__dsub_rn(__dmul_rn(static_cast<double>(L[(i + u) * a.ldL]), sc),
                                           st[(i + u) * 3]));
            p[u] = prob_f32(e, st[(i + u) * 3 + 1], st[(i + u) * 3 + 2]);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) acc = __fadd_rn(acc, p[u]);
        }
        for (; i < a.n_t; ++i) {
          const double e = exp(__dsub_rn(__dmul_rn(static_cast<double>(L[i * a.ldL]), sc), st[i * 3]));
          acc = __fadd_rn(acc, prob_f32(e, st[i * 3 + 1], st[i * 3 + 2]));
        }
      } else {
        for (int i = 0; i < a.n_t; ++i) acc = __fadd_rn(acc, __fmul_rn(L[i * a.ldL], a.scale));
      }
    }
    part[h][x] = acc;
  }
  __syncthreads();
  if (y == 0 && inb) {
    float total = 0.f;
    for (int h = 0; h < a.hq; ++h) total = __fadd_rn(total, part[h][x]);
    // pad keys -> -inf (approx.cpp:64-66); a block without visible keys is all pads
    a.scores[blk][j] = is_pad(a.pad[blk], a.n_valid[blk], j) ? -INFINITY : total;
  }
}

}  // namespace

size_t score_workspace_bytes(int n_t, int l_b, int hq) {
  // sized for two blocks (lo + hi) scored in one launch
  const size_t L = 2ull * hq * n_t * ld_logits(l_b) * sizeof(float);
  const size_t part = 2ull * hq * n_t * n_ktiles(l_b) * sizeof(double2);
  const size_t st = 2ull * hq * n_t * 3 * sizeof(double);
  return L + part + st + 1024;
}

cudaError_t launch_score_exact2(int nblk, const void* q, long long ldq, int n_t,
                                const void* const* k, long long ldk, int l_b,
                                const uint8_t* const* pad, const int* n_valid, int hq, int hkv,
                                int dh, int softmax, float* const* scores, void* ws,
                                size_t ws_bytes, cudaStream_t stream) {
  if (dh != kDh || hq < 1 || hkv < 1 || hq % hkv || hq > 32 || n_t < 1 || nblk < 1 || nblk > 2)
    return cudaErrorInvalidValue;
  if (l_b <= 0) return cudaSuccess;
  if (ws_bytes < score_workspace_bytes(n_t, l_b, hq)) return cudaErrorInvalidValue;
  if ((ldq % 4) || (ldk % 4)) return cudaErrorInvalidValue;
  ScoreArgs a{};
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.ldq = ldq;
  for (int b = 0; b < nblk; ++b) {
    a.k[b] = static_cast<const __nv_bfloat16*>(k[b]);
    a.pad[b] = pad ? pad[b] : nullptr;
    a.n_valid[b] = n_valid[b];
    a.scores[b] = scores[b];
  }
  a.ldk = ldk;
  a.nblk = nblk;
  a.n_t = n_t;
  a.l_b = l_b;
  a.hq = hq;
  a.hkv = hkv;
  a.softmax = softmax;
  a.scale = 1.0f / sqrtf(static_cast<float>(dh));
  a.ldL = ld_logits(l_b);
  a.ntiles = n_ktiles(l_b);
  uint8_t* w = static_cast<uint8_t*>(ws);
  a.L = reinterpret_cast<float*>(w);
  w += 2ull * hq * n_t * a.ldL * sizeof(float);
  a.part = reinterpret_cast<double2*>((reinterpret_cast<uintptr_t>(w) + 255) & ~uintptr_t(255));
  w = reinterpret_cast<uint8_t*>(a.part) + 2ull * hq * n_t * a.ntiles * sizeof(double2);
  a.stats = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(w) + 255) & ~uintptr_t(255));
  logits_kernel<<<dim3(a.ntiles, hq, nblk), kThr, 0, stream>>>(a);
  if (softmax) {
    const long long rows = static_cast<long long>(nblk) * hq * n_t;
    stats_kernel<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, stream>>>(a);
  }
  colsum_kernel<<<dim3((l_b + 31) / 32, nblk), dim3(32, 8), 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_score_exact(const void* q, long long ldq, int n_t, const void* k,
                               long long ldk, int l_b, const uint8_t* pad, int n_valid, int hq,
                               int hkv, int dh, int softmax, float* scores, void* ws,
                               size_t ws_bytes, cudaStream_t stream) {
  const void* ks[1] = {k};
  const uint8_t* pads[1] = {pad};
  const int nv[1] = {n_valid};
  float* sc[1] = {scores};
  return launch_score_exact2(1, q, ldq, n_t, ks, ldk, l_b, pads, nv, hq, hkv, dh, softmax, sc, ws,
                             ws_bytes, stream);
}

}  // namespace spava
