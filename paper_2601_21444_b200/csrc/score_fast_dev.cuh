// score_fast_dev.cuh -- device body of the tensor-core ("fast") scorer, shared by the
// standalone scorer kernels (score_fast.cu) and the column-sum CTAs that ride in the query
// attention launch (attention.cu; the row statistics come from its online softmax).
#pragma once

#include <cuda_bf16.h>

#include "ptx.cuh"
#include "spava_internal.h"

namespace spava {

constexpr int kFThreads = 192;       // warps 0-3 softmax, 4 TMA, 5 MMA
constexpr int kFMaxKv = 4;
constexpr int kFMaxHq = 32;
constexpr uint32_t kFBox = 128 * 64 * 2;
constexpr uint32_t kFTile = 2 * kFBox;  // 128 rows x 128 dh bf16
// shared memory of one scorer CTA: K tiles of every kv-head, a 2-stage Q_h ring, the lse
// table of pass 1 ([hq][128] f32) and the barriers (byte offsets from a 1024-aligned base)
struct FSmem {
  static constexpr uint32_t k = 0;
  uint32_t q, lse, bar, total;
  __host__ __device__ FSmem(int hkv, int hq) {
    q = k + hkv * kFTile;
    lse = q + 2 * kFTile;
    bar = lse + hq * 128 * 4;
    total = bar + 128;
  }
  __host__ __device__ uint32_t bytes() const { return total + 1024; }  // + alignment slack
};
static constexpr uint32_t kFSmemMaxBytes = FSmem::k + kFMaxKv * kFTile + 2 * kFTile + kFMaxHq * 128 * 4 + 128 + 1024;


// One (block, 128-key tile) CTA of pass kPass.  Warps 0-3 compute, warp 4 TMA, warp 5 MMA;
// any further warps of the CTA only take part in the barriers.  `smem` is 1024-aligned.
// Pass 1 with a.ready != nullptr first waits (one thread, acquire) until *a.ready reached
// a.epoch: lse2 is produced inside the same launch (query attention, attention.cu).
template <int kPass>
__device__ __forceinline__ void score_fast_cta(const FastArgs& a, int kt, int blk, uint8_t* smem) {
  const FSmem L(a.hkv, a.hq);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint64_t* k_full = bars + 0;
  uint64_t* q_full = bars + 1;   // [2]
  uint64_t* q_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;   // [2]
  uint64_t* s_free = bars + 7;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);
  float* lse_tab = reinterpret_cast<float*>(smem + L.lse);

  const int warp = warp_id(), lane = lane_id();
  const int group = a.hq / a.hkv;

  if (kPass == 1 && a.ready) {
    if (threadIdx.x == 0) {
      unsigned long long t0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      while (true) {
        uint32_t v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.ready) : "memory");
        if (static_cast<int32_t>(v - a.epoch) >= 0) break;
        __nanosleep(100);
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 8000000000ull) __trap();
      }
    }
    __syncthreads();
  }
  if (kPass == 1) {
    // per-column (query row) log2-sum-exp of every head; rows >= n_t never contribute
    for (int e = threadIdx.x; e < a.hq * 128; e += kFThreads) {
      const int h = e >> 7, i = e & 127;
      lse_tab[e] = i < a.n_t ? __ldcg(a.lse2 + (static_cast<long long>(blk) * a.hq + h) * a.n_t + i) : INFINITY;
    }
  }
  if (warp == 4 && elect_one()) {
    mbar_init(k_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(q_full + s, 1);
      mbar_init(q_empty + s, 1);
      mbar_init(s_full + s, 1);
      mbar_init(s_free + s, 128);
    }
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    if (elect_one()) {
      mbar_expect_tx(k_full, a.hkv * kFTile);
      for (int g = 0; g < a.hkv; ++g)
        for (int c = 0; c < 2; ++c)
          tma_load_2d(smem + L.k + g * kFTile + c * kFBox, &a.tk[blk], k_full, g * 128 + c * 64, kt * 128);
      for (int h = 0; h < a.hq; ++h) {
        const int st = h & 1;
        if (h >= 2) mbar_wait(q_empty + st, ((h >> 1) - 1) & 1);
        mbar_expect_tx(q_full + st, kFTile);
        for (int c = 0; c < 2; ++c)
          tma_load_2d(smem + L.q + st * kFTile + c * kFBox, &a.tq, q_full + st, h * 128 + c * 64, 0);
      }
    }
  } else if (warp == 5) {
    if (elect_one()) {
      const uint32_t idesc = idesc_bf16_f32(128, 128, 0, 0);
      const uint32_t sk = smem_u32(smem + L.k), sq = smem_u32(smem + L.q);
      mbar_wait(k_full, 0);
      for (int h = 0; h < a.hq; ++h) {
        const int st = h & 1, b = h & 1;
        mbar_wait(q_full + st, (h >> 1) & 1);
        if (h >= 2) mbar_wait(s_free + b, ((h >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t kb = sk + (h / group) * kFTile, qb = sq + st * kFTile;
        // pass 0: A = Q_h (rows = queries), B = K tile; pass 1: A = K tile (rows = keys)
        const uint32_t abase = kPass == 0 ? qb : kb, bbase = kPass == 0 ? kb : qb;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * kFBox + (kk & 3) * 32;
          mma_ss(tmem + b * 128, sdesc_sw128(abase + off, 16, 1024), sdesc_sw128(bbase + off, 16, 1024),
                 idesc, kk > 0 ? 1u : 0u);
        }
        tc_commit(s_full + b);
        tc_commit(q_empty + st);
      }
    }
  } else if (warp < 4) {
    // thread = TMEM lane: pass 0 -> query row i; pass 1 -> key j of this tile
    const int r = warp * 32 + lane;
    const uint32_t t_lane = static_cast<uint32_t>(warp * 32) << 16;
    const int nv = min(a.n_valid[blk], a.l_b);
    const uint8_t* pad = a.pad[blk];
    const int j = kt * 128 + r;  // pass 1: this thread's key
    const float2 sl2v = make_float2(a.sl2, a.sl2);
    float score = 0.f;
    for (int h = 0; h < a.hq; ++h) {
      const int b = h & 1;
      mbar_wait(s_full + b, (h >> 1) & 1);
      tc_fence_after();
      uint32_t sr[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tmem + t_lane + b * 128 + 32 * c, sr[c]);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(s_free + b);  // the MMA of head h+2 may overwrite this buffer
      if (kPass == 0) {
        // columns = keys kt*128 + c*32 + e of this tile: visible iff < n_valid and not pad;
        // only a ragged or padded tile pays for the mask
        if (kt * 128 + 128 > nv || pad) {
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              const int jj = kt * 128 + c * 32 + e;
              if (!(jj < nv && !(pad && pad[jj]))) sr[c][e] = __float_as_uint(-INFINITY);
            }
        }
        float mp[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) mp[t] = -INFINITY;
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int e = 0; e < 32; e += 2)
            mp[(e / 2) & 7] = fmaxf(mp[(e / 2) & 7], fmaxf(__uint_as_float(sr[c][e]), __uint_as_float(sr[c][e + 1])));
        const float mraw = fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])),
                                 fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
        const float mx = mraw * a.sl2;  // sl2 > 0: max commutes with the scale
        float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                         make_float2(0.f, 0.f)};
        if (mx != -INFINITY) {
          const float2 negm = make_float2(-mx, -mx);
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const float2 x2 = __ffma2_rn(make_float2(__uint_as_float(sr[c][2 * e]),
                                                       __uint_as_float(sr[c][2 * e + 1])), sl2v, negm);
              acc[e & 3] = __fadd2_rn(acc[e & 3], make_float2(fast_exp2(x2.x), fast_exp2(x2.y)));
            }
        }
        const float2 s2 = __fadd2_rn(__fadd2_rn(acc[0], acc[1]), __fadd2_rn(acc[2], acc[3]));
        if (r < a.n_t)
          a.part[((static_cast<long long>(blk) * a.hq + h) * a.n_t + r) * a.ntiles + kt] =
              make_float2(mx, s2.x + s2.y);
      } else {
        const float* lt = lse_tab + h * 128;  // +inf for rows >= n_t -> 2^-inf = 0
        float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                         make_float2(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float2 l2 = *reinterpret_cast<const float2*>(lt + c * 32 + 2 * e);
            const float2 x2 = __ffma2_rn(make_float2(__uint_as_float(sr[c][2 * e]),
                                                     __uint_as_float(sr[c][2 * e + 1])),
                                         sl2v, make_float2(-l2.x, -l2.y));
            acc[e & 3] = __fadd2_rn(acc[e & 3], make_float2(fast_exp2(x2.x), fast_exp2(x2.y)));
          }
        const float2 s2 = __fadd2_rn(__fadd2_rn(acc[0], acc[1]), __fadd2_rn(acc[2], acc[3]));
        score = __fadd_rn(score, s2.x + s2.y);  // heads ascending (approx.cpp:57, simhost.cpp:222)
      }
    }
    if (kPass == 1 && j < a.l_b) {
      const bool is_pad = j >= a.n_valid[blk] || (pad && pad[j]);
      a.scores[blk][j] = is_pad ? -INFINITY : score;  // approx.cpp:64-66
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_dealloc(tmem, 256);
}

}  // namespace spava
