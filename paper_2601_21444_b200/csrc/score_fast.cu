// score_fast.cu -- "fast" query-aware block scoring on the tensor cores (sm_100a).
//
// Same definition as score_block (simhost.cpp:209-224) -> score_context (approx.cpp:15-69):
//   score_j = sum_h sum_i softmax_j(q_hi . k_j * scale)          (softmax over the block's keys)
// but the logits come from tcgen05 bf16 MMAs with fp32 accumulation and the softmax is
// evaluated with exp2 on the MUFU, so scores differ from the reference in the last bits;
// passing-block indices agree except where two scores tie to within that error (the bench
// reports the agreement rate against the exact scorer).  Two passes over (block, 128-key
// tile) CTAs, each looping over the q-heads with the next head's MMA overlapping the
// current head's exps (S double-buffered in TMEM):
//   pass 0 (rowstats): S = Q_h K_t^T (lanes = query rows): per (row, tile) max and sum of
//                       2^(x - max) in the log2 domain           -> partials
//   combine          : lse2[blk][h][i] = log2 sum over tiles
//   pass 1 (colsum)  : S^T = K_t Q_h^T (lanes = keys): part_j = sum_i 2^(x_ij - lse2_i),
//                       score_j += part_j in head order            -> scores
// K tiles of every kv-head stay in smem for the CTA; Q_h tiles stream through a 2-stage
// TMA ring.  n_t <= 128 (one N=128 tile of query rows), hkv <= 4, dh = 128.
#include <cuda_bf16.h>

#include "score_fast_dev.cuh"

namespace spava {

namespace {

template <int kPass>
__global__ void __launch_bounds__(kFThreads, 1) score_fast_kernel(const __grid_constant__ FastArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  score_fast_cta<kPass>(a, blockIdx.x, blockIdx.y, smem);
}

// lse2[blk][h][i] = M + log2(sum_t s_t 2^(m_t - M)) over the key tiles of the block;
// one warp per row, lanes strided over the tiles
__global__ void score_fast_combine_kernel(FastArgs a, int rows) {
  const int r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float2* p = a.part + static_cast<long long>(r) * a.ntiles;
  float M = -INFINITY;
  for (int t = lane; t < a.ntiles; t += 32) M = fmaxf(M, p[t].x);
#pragma unroll
  for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  float s = 0.f;
  if (M != -INFINITY)
    for (int t = lane; t < a.ntiles; t += 32)
      if (p[t].x != -INFINITY) s += p[t].y * exp2f(p[t].x - M);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) a.lse2[r] = M + __log2f(s);
}

}  // namespace

size_t score_fast_workspace_bytes(int n_t, int l_b, int hq) {
  const size_t ntiles = (static_cast<size_t>(l_b) + 127) / 128;
  return 2ull * hq * n_t * ntiles * sizeof(float2) + 2ull * hq * n_t * sizeof(float) + 512;
}

cudaError_t launch_score_fast2(int nblk, const void* q, long long ldq, int n_t,
                               const void* const* k, long long ldk, int l_b,
                               const uint8_t* const* pad, const int* n_valid, int hq, int hkv,
                               int dh, float* const* scores, void* ws, size_t ws_bytes,
                               cudaStream_t stream, std::string* err) {
  if (dh != 128 || hq < 1 || hkv < 1 || hq % hkv || hq > kFMaxHq || hkv > kFMaxKv || n_t < 1 ||
      n_t > 128 || nblk < 1 || nblk > 2) {
    if (err) *err = "score_fast: needs dh == 128, n_t <= 128, hq <= 32, hkv <= 4";
    return cudaErrorInvalidValue;
  }
  if (l_b <= 0) return cudaSuccess;
  if (ws_bytes < score_fast_workspace_bytes(n_t, l_b, hq)) {
    if (err) *err = "score_fast: workspace too small";
    return cudaErrorInvalidValue;
  }
  FastArgs a{};
  if (!make_tmap_bf16(&a.tq, q, n_t, static_cast<long long>(hq) * 128, ldq, 128, err))
    return cudaErrorInvalidValue;
  for (int b = 0; b < nblk; ++b) {
    if (!make_tmap_bf16(&a.tk[b], k[b], l_b, static_cast<long long>(hkv) * 128, ldk, 128, err))
      return cudaErrorInvalidValue;
    a.n_valid[b] = n_valid[b];
    a.pad[b] = pad ? pad[b] : nullptr;
    a.scores[b] = scores[b];
  }
  a.n_t = n_t;
  a.l_b = l_b;
  a.hq = hq;
  a.hkv = hkv;
  a.ntiles = (l_b + 127) / 128;
  a.sl2 = (1.0f / sqrtf(128.f)) * 1.4426950408889634f;
  a.part = static_cast<float2*>(ws);
  a.lse2 = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) +
                                    ((2ull * hq * n_t * a.ntiles * sizeof(float2) + 255) & ~255ull));
  static std::atomic<uint32_t> attr[kMaxDevices] = {};
  for (int v = 0; v < 2; ++v) {
    const void* fn = v ? reinterpret_cast<const void*>(score_fast_kernel<1>)
                       : reinterpret_cast<const void*>(score_fast_kernel<0>);
    if (cudaError_t e = smem_optin(fn, static_cast<int>(kFSmemMaxBytes), attr, v); e != cudaSuccess) return e;
  }
  const dim3 grid(a.ntiles, nblk);
  const uint32_t smem = FSmem(hkv, hq).bytes();
  score_fast_kernel<0><<<grid, kFThreads, smem, stream>>>(a);
  const int rows = nblk * hq * n_t;
  score_fast_combine_kernel<<<(rows + 7) / 8, 256, 0, stream>>>(a, rows);
  score_fast_kernel<1><<<grid, kFThreads, smem, stream>>>(a);
  return cudaGetLastError();
}

}  // namespace spava
