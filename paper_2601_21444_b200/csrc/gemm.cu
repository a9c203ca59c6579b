// gemm.cu -- the decoder layer's GEMMs on tcgen05, no library.
//
// Row-major C[M x N] (+)= A[M x K] * B[K x N] in bf16 with fp32 accumulation in TMEM, the
// shapes of the reference decoder layer around the attention (simhost.cpp:196-207
// project, :431-436 finish_group): x [rows x d_model] times W_qkv / W_o / W_1 / W_2.
//
// Persistent warp-specialised kernel, one CTA per SM, 128 x 256 output tiles:
//   warp 0      TMA producer: A box (128 rows x 64 k, K-major) + 4 B boxes (64 k x 64 n,
//               N-major) per k-step into a 4-stage 128B-swizzled ring (48 KB / stage)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128 N=256 K=16 x4 per
//               stage), accumulating in one of two TMEM buffers (2 x 256 columns) so the
//               epilogue of tile i overlaps the main loop of tile i+1
//   warps 2-5   epilogue: tcgen05.ld 32 columns at a time (thread = TMEM lane = output
//               row), optional beta * C (the residual x += ...), optional ReLU, bf16
//               stores; the output columns may be routed to up to 3 buffers (the fused
//               [Wq | Wk | Wv] projection writes q, k and v directly).
// Tiles are rastered n-fastest so the ~148 CTAs in flight share their A row-blocks in L2.
#include <cuda_bf16.h>

#include "ptx.cuh"
#include "spava_internal.h"

namespace spava {

namespace {

constexpr int kGM = 128, kGN = 256, kGK = 64, kGStages = 4, kGThreads = 192;
constexpr uint32_t kGABytes = kGM * kGK * 2;     // 16 KB, one SW128 box
constexpr uint32_t kGBBox = kGK * 64 * 2;        // 8 KB: 64 k rows x 64 n
constexpr uint32_t kGBBytes = 4 * kGBBox;        // 32 KB
constexpr uint32_t kGStageBytes = kGABytes + kGBBytes;
constexpr uint32_t kGBar = kGStages * kGStageBytes;
constexpr uint32_t kGSmem = kGBar + 256 + 1024;

struct GemmArgs {
  CUtensorMap ta;  // A [M x K], box 64 k x 128 rows
  CUtensorMap tb;  // B [K x N], box 64 n x 64 k
  int M, N, K;
  int tiles_m, tiles_n;
  int nout;
  int col0[4];  // output r holds columns [col0[r], col0[r+1]) of C, col0[nout] = N
  __nv_bfloat16* out[3];
  long long ldo[3];
  float beta;  // 0: C = AB; else C = AB + beta * C (read from the same output)
  int relu;
};

__global__ void __launch_bounds__(kGThreads, 1) gemm_kernel(const __grid_constant__ GemmArgs g) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kGBar);
  uint64_t* full = bars;                 // [kGStages]
  uint64_t* empty = full + kGStages;     // [kGStages]
  uint64_t* acc_full = empty + kGStages; // [2]
  uint64_t* acc_empty = acc_full + 2;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = warp_id(), lane = lane_id();
  const int T = g.tiles_m * g.tiles_n;
  const int kb_n = (g.K + kGK - 1) / kGK;

  if (warp == 0 && elect_one()) {
    for (int s = 0; s < kGStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(acc_full + b, 1);
      mbar_init(acc_empty + b, 128);
    }
    fence_barrier_init();
    tma_prefetch_desc(&g.ta);
    tma_prefetch_desc(&g.tb);
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      uint32_t it = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x) {
        const int tm = t / g.tiles_n, tn = t % g.tiles_n;
        for (int kb = 0; kb < kb_n; ++kb, ++it) {
          const uint32_t s = it % kGStages;
          if (it >= kGStages) mbar_wait(empty + s, ((it / kGStages) - 1) & 1);
          uint8_t* st = smem + s * kGStageBytes;
          mbar_expect_tx(full + s, kGStageBytes);
          tma_load_2d(st, &g.ta, full + s, kb * kGK, tm * kGM);
          for (int j = 0; j < 4; ++j)
            tma_load_2d(st + kGABytes + j * kGBBox, &g.tb, full + s, tn * kGN + j * 64, kb * kGK);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      const uint32_t idesc = idesc_bf16_f32(kGM, kGN, 0, 1);  // A K-major, B N-major
      uint32_t it = 0, i = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x, ++i) {
        const uint32_t ab = i & 1;
        if (i >= 2) mbar_wait(acc_empty + ab, ((i >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + ab * kGN;
        for (int kb = 0; kb < kb_n; ++kb, ++it) {
          const uint32_t s = it % kGStages;
          mbar_wait(full + s, (it / kGStages) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * kGStageBytes), sb = sa + kGABytes;
#pragma unroll
          for (int kk = 0; kk < kGK / 16; ++kk) {
            const uint64_t a = sdesc_sw128(sa + kk * 32, 16, 1024);
            const uint64_t b = sdesc_sw128(sb + kk * 2048, kGBBox, 1024);
            mma_ss(d, a, b, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          }
          tc_commit(empty + s);
        }
        tc_commit(acc_full + ab);
      }
    }
  } else {
    // epilogue warpgroup: warp w reads TMEM lanes 32*(w%4) .. +31
    const int quad = warp & 3;
    const uint32_t t_lane = static_cast<uint32_t>(quad * 32) << 16;
    uint32_t i = 0;
    for (int t = blockIdx.x; t < T; t += gridDim.x, ++i) {
      const int tm = t / g.tiles_n, tn = t % g.tiles_n;
      const uint32_t ab = i & 1;
      mbar_wait(acc_full + ab, (i >> 1) & 1);
      tc_fence_after();
      const int row = tm * kGM + quad * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < kGN / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem + t_lane + ab * kGN + c * 32, r);
        tmem_wait_ld();
        const int col = tn * kGN + c * 32;
        if (row >= g.M || col >= g.N) continue;
        int o = 0;
        while (o + 1 < g.nout && col >= g.col0[o + 1]) ++o;
        __nv_bfloat16* dst = g.out[o] + static_cast<long long>(row) * g.ldo[o] + (col - g.col0[o]);
        const int ncols = min(32, g.N - col);
        if (ncols == 32) {
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint4 prev = make_uint4(0, 0, 0, 0);
            if (g.beta != 0.f) prev = reinterpret_cast<const uint4*>(dst)[q4];
            const uint32_t pw[4] = {prev.x, prev.y, prev.z, prev.w};
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float v0 = __uint_as_float(r[q4 * 8 + 2 * e]), v1 = __uint_as_float(r[q4 * 8 + 2 * e + 1]);
              if (g.beta != 0.f) {
                const float2 p2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pw[e]));
                v0 = fmaf(g.beta, p2.x, v0);
                v1 = fmaf(g.beta, p2.y, v1);
              }
              if (g.relu) {
                v0 = fmaxf(v0, 0.f);
                v1 = fmaxf(v1, 0.f);
              }
              __nv_bfloat162 b2 = __floats2bfloat162_rn(v0, v1);
              w[e] = *reinterpret_cast<uint32_t*>(&b2);
            }
            reinterpret_cast<uint4*>(dst)[q4] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) {  // compile-time indices: r stays in registers
            if (e >= ncols) break;
            float v = __uint_as_float(r[e]);
            if (g.beta != 0.f) v = fmaf(g.beta, __bfloat162float(dst[e]), v);
            if (g.relu) v = fmaxf(v, 0.f);
            dst[e] = __float2bfloat16_rn(v);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(acc_empty + ab);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

}  // namespace

// C (+)= A B, row-major bf16; outputs: nout column ranges [col0[r], col0[r+1]) of C go to
// out[r] (row stride ldo[r]); ranges must start at multiples of 32.  beta != 0 reads the
// previous C from the outputs (residual add); relu clamps at 0 after it.
cudaError_t launch_gemm_bf16(int M, int N, int K, const void* A, long long lda, const void* B, long long ldb,
                             int nout, const int* col0, void* const* out, const long long* ldo, float beta,
                             bool relu, cudaStream_t stream, std::string* err) {
  if (M <= 0 || N <= 0 || K <= 0 || nout < 1 || nout > 3 || lda % 8 || ldb % 8 || N % 8) {
    if (err) *err = "gemm: bad shape / strides (row strides and N multiples of 8)";
    return cudaErrorInvalidValue;
  }
  GemmArgs g{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.tiles_m = (M + kGM - 1) / kGM;
  g.tiles_n = (N + kGN - 1) / kGN;
  g.nout = nout;
  for (int r = 0; r < nout; ++r) {
    if (col0[r] % 32 || (r > 0 && col0[r] <= col0[r - 1]) || ldo[r] % 8 || !out[r]) {
      if (err) *err = "gemm: output ranges must be increasing multiples of 32 with 16-byte rows";
      return cudaErrorInvalidValue;
    }
    g.col0[r] = col0[r];
    g.out[r] = static_cast<__nv_bfloat16*>(out[r]);
    g.ldo[r] = ldo[r];
  }
  if (col0[0] != 0) {
    if (err) *err = "gemm: the first output range starts at column 0";
    return cudaErrorInvalidValue;
  }
  g.col0[nout] = N;
  g.beta = beta;
  g.relu = relu ? 1 : 0;
  if (!make_tmap_bf16(&g.ta, A, M, K, lda, kGM, err) || !make_tmap_bf16(&g.tb, B, K, N, ldb, kGK, err))
    return cudaErrorInvalidValue;
  static std::atomic<uint32_t> attr[kMaxDevices] = {};
  if (cudaError_t e = smem_optin(reinterpret_cast<const void*>(gemm_kernel), static_cast<int>(kGSmem), attr, 0);
      e != cudaSuccess)
    return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int tiles = g.tiles_m * g.tiles_n;
  gemm_kernel<<<std::min(tiles, sms), kGThreads, kGSmem, stream>>>(g);
  return cudaGetLastError();
}

}  // namespace spava
