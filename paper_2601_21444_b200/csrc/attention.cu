// attention.cu -- fused segment attention for the Spava prefill on sm_100a.
//
// One kernel computes every attention call of the Spava layer
//   anchor_attention  (approx.cpp:134-138)  one causal segment
//   block_attention   (approx.cpp:140-154)  [anchor | passing(1..2 ranges) | own causal+pad]
//   query_attention   (approx.cpp:156-188)  [anchor slice | lo | hi | self causal], lse out
// i.e. attention_lse/mha_lse (attention.cpp:18-86, 158-178) over a segment table, with
// the reference's masking rules: key j of segment s is visible to query row i iff
// j < len(s) and (s not causal or j <= i).  Pads only ever sit at a segment's tail
// (partition.cpp:71-79), so a pad mask is a valid length.
//
// Blackwell structure (one CTA = 256 query rows of one q-head, or one split of them):
//   warp 8      TMA producer: Q tiles once, then K/V tiles of every visible segment into
//               a 2-stage 128B-swizzled smem ring (OOB rows zero-filled by TMA).
//   warp 9      TMEM allocator + single-thread tcgen05.mma issuer:
//                 S_t = Q_t K^T  (SS, M=128 N=128 K=16 x8, fp32 accum in TMEM)
//                 O_t += P_t V   (TS: P_t read from TMEM, V from smem, MN-major B)
//               ping-ponging the two Q tiles so the tensor pipe works on one tile while
//               the softmax warpgroup of the other runs.
//   warps 0-7   two softmax warpgroups (one per Q tile, thread = TMEM lane = query row):
//               tcgen05.ld S, mask, online softmax in exp2 domain with lazy (>2^8) O
//               rescale, P packed to bf16 and written back over S with tcgen05.st,
//               epilogue O/l (+ lse) straight from TMEM to HBM.
// GQA: q-head h reads kv-head h / (hq/hkv); consecutive CTAs share K/V tiles in L2.
// Split-KV (query attention has only 128 rows): a CTA handles a contiguous slice of the
// tile list and writes an (out, lse) partial, combined by the lse merge (merge.cu).
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "ptx.cuh"
#include "spava_internal.h"

namespace spava {

namespace {

constexpr int kStages = 2;
constexpr int kSoftmaxWarps = 8;
constexpr int kProducerWarp = 8;
constexpr int kMmaWarp = 9;
constexpr int kThreads = 320;
constexpr uint32_t kBoxBytes = 128 * 64 * 2;    // 128 rows x 64 bf16, one SW128 TMA box
constexpr uint32_t kTileBytes = 2 * kBoxBytes;  // 128 rows x 128 dh
constexpr uint32_t kTmemCols = 512;             // S0 | S1 | O0 | O1

struct Smem {
  static constexpr uint32_t q = 0;
  static constexpr uint32_t k = q + kTilesPerCta * kTileBytes;
  static constexpr uint32_t v = k + kStages * kTileBytes;
  static constexpr uint32_t bar = v + kStages * kTileBytes;
  static constexpr uint32_t total = bar + 256;
};
constexpr uint32_t kSmemBytes = Smem::total + 1024;  // + alignment slack

enum : int { kSkip = 0, kFull = 1, kPart = 2 };

__device__ __forceinline__ int seg_tiles(const AttnSeg& s, int imax) {
  const int klen = s.causal ? min(s.len, imax) : s.len;
  return klen > 0 ? (klen + kBlockN - 1) / kBlockN : 0;
}

// Masking mode of KV tile kt of segment s for the Q tile starting at row r0.
__device__ __forceinline__ int tile_mode(const AttnSeg& s, int kt, int r0, int nq) {
  if (r0 >= nq) return kSkip;
  const int k0 = kt * kBlockN;
  const bool tail = k0 + kBlockN > s.len;
  if (s.causal) {
    const int rlast = min(r0 + kBlockM, nq) - 1;
    if (k0 > rlast) return kSkip;
    return (k0 + kBlockN - 1 > r0 || tail) ? kPart : kFull;
  }
  return tail ? kPart : kFull;
}

struct Cursor {
  int seg, kt;
};

__device__ __forceinline__ Cursor cursor_at(const AttnProb& p, int imax, int t) {
  for (int s = 0; s < p.nseg; ++s) {
    const int n = seg_tiles(p.seg[s], imax);
    if (t < n) return {s, t};
    t -= n;
  }
  return {p.nseg, 0};
}

__device__ __forceinline__ void cursor_next(const AttnProb& p, int imax, Cursor& c) {
  ++c.kt;
  while (c.seg < p.nseg && c.kt >= seg_tiles(p.seg[c.seg], imax)) {
    ++c.seg;
    c.kt = 0;
  }
}

__global__ void __launch_bounds__(kThreads, 1) attn_fwd_kernel(const __grid_constant__ AttnParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::bar);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;    // [kStages]
  uint64_t* v_full = bars + 3;    // [kStages]
  uint64_t* kv_empty = bars + 5;  // [kStages]
  uint64_t* s_full = bars + 7;    // [2] S_t ready in TMEM
  uint64_t* p_full = bars + 9;    // [2] P_t written (and O_t corrected)
  uint64_t* o_full = bars + 11;   // [2] PV_t complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 13);

  const int warp = warp_id();
  const int lane = lane_id();

  // ---- decode the work item: problem, 256-row unit (heaviest first), head, split
  int pi = 0;
  while (pi + 1 < P.nprob && static_cast<int>(blockIdx.x) >= P.prob[pi + 1].work_begin) ++pi;
  const AttnProb& prob = P.prob[pi];
  int local = static_cast<int>(blockIdx.x) - prob.work_begin;
  const int split = local % prob.splits;
  local /= prob.splits;
  const int head = local % P.hq;
  local /= P.hq;
  const int unit = prob.units - 1 - local;
  const int i0 = unit * (kTilesPerCta * kBlockM);
  const int nq = prob.nq;
  const int imax = min(i0 + kTilesPerCta * kBlockM, nq);
  const int hk = head / (P.hq / P.hkv);

  int T = 0;
  for (int s = 0; s < prob.nseg; ++s) T += seg_tiles(prob.seg[s], imax);
  const int t_begin = static_cast<int>(static_cast<long long>(T) * split / prob.splits);
  const int t_end = static_cast<int>(static_cast<long long>(T) * (split + 1) / prob.splits);
  const int ntiles = t_end - t_begin;
  const CUtensorMap* tm = P.tmap[pi];

  if (warp == kProducerWarp && elect_one()) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(k_full + s, 1);
      mbar_init(v_full + s, 1);
      mbar_init(kv_empty + s, 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(s_full + t, 1);
      mbar_init(p_full + t, 128);
      mbar_init(o_full + t, 1);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tm[0]);
    for (int s = 0; s < prob.nseg; ++s) {
      tma_prefetch_desc(&tm[1 + 2 * s]);
      tma_prefetch_desc(&tm[2 + 2 * s]);
    }
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kProducerWarp) {
    // ======================================================== TMA producer
    if (elect_one()) {
      const bool has1 = i0 + kBlockM < nq;
      mbar_expect_tx(q_full, (has1 ? 2u : 1u) * kTileBytes);
      for (int qt = 0; qt < (has1 ? 2 : 1); ++qt)
        for (int c = 0; c < 2; ++c)
          tma_load_2d(smem + Smem::q + qt * kTileBytes + c * kBoxBytes, &tm[0], q_full,
                      head * kHeadDim + c * 64, i0 + qt * kBlockM);
      Cursor cur = cursor_at(prob, imax, t_begin);
      for (int it = 0; it < ntiles; ++it) {
        const int stage = it % kStages;
        if (it >= kStages) mbar_wait(kv_empty + stage, ((it / kStages) - 1) & 1);
        const CUtensorMap* km = &tm[1 + 2 * cur.seg];
        const CUtensorMap* vm = &tm[2 + 2 * cur.seg];
        mbar_expect_tx(k_full + stage, kTileBytes);
        for (int c = 0; c < 2; ++c)
          tma_load_2d(smem + Smem::k + stage * kTileBytes + c * kBoxBytes, km, k_full + stage,
                      hk * kHeadDim + c * 64, cur.kt * kBlockN);
        mbar_expect_tx(v_full + stage, kTileBytes);
        for (int c = 0; c < 2; ++c)
          tma_load_2d(smem + Smem::v + stage * kTileBytes + c * kBoxBytes, vm, v_full + stage,
                      hk * kHeadDim + c * 64, cur.kt * kBlockN);
        cursor_next(prob, imax, cur);
      }
    }
  } else if (warp == kMmaWarp) {
    // ======================================================== MMA issuer
    if (elect_one()) {
      const uint32_t idesc_qk = idesc_bf16_f32(128, 128, 0, 0);  // Q, K both K-major
      const uint32_t idesc_pv = idesc_bf16_f32(128, 128, 0, 1);  // P (TMEM), V MN-major
      const uint32_t sq = smem_u32(smem + Smem::q);
      const uint32_t sk = smem_u32(smem + Smem::k);
      const uint32_t sv = smem_u32(smem + Smem::v);
      auto issue_qk = [&](int qt, int stage) {
        const uint32_t d = tmem + qt * 128;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t koff = (kk >> 2) * kBoxBytes + (kk & 3) * 32;
          const uint64_t a = sdesc_sw128(sq + qt * kTileBytes + koff, 16, 1024);
          const uint64_t b = sdesc_sw128(sk + stage * kTileBytes + koff, 16, 1024);
          mma_ss(d, a, b, idesc_qk, kk > 0 ? 1u : 0u);
        }
      };
      auto issue_pv = [&](int qt, int stage, bool acc) {
        const uint32_t d = tmem + 256 + qt * 128;
        const uint32_t a = tmem + qt * 128;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t b = sdesc_sw128(sv + stage * kTileBytes + kk * 2048, kBoxBytes, 1024);
          mma_ts(d, a + kk * 8, b, idesc_pv, (acc || kk > 0) ? 1u : 0u);
        }
      };

      mbar_wait(q_full, 0);
      tc_fence_after();
      Cursor cur = cursor_at(prob, imax, t_begin);
      int mode[2] = {kSkip, kSkip};
      uint32_t p_cnt[2] = {0, 0};
      bool o_acc[2] = {false, false};
      if (ntiles > 0) {
        for (int qt = 0; qt < 2; ++qt)
          mode[qt] = tile_mode(prob.seg[cur.seg], cur.kt, i0 + qt * kBlockM, nq);
        mbar_wait(k_full + 0, 0);
        tc_fence_after();
        for (int qt = 0; qt < 2; ++qt)
          if (mode[qt] != kSkip) {
            issue_qk(qt, 0);
            tc_commit(s_full + qt);
          }
      }
      for (int it = 0; it < ntiles; ++it) {
        const int stage = it % kStages;
        const uint32_t ph = (it / kStages) & 1;
        const bool has_next = it + 1 < ntiles;
        Cursor nxt = cur;
        int nmode[2] = {kSkip, kSkip};
        const int nstage = (it + 1) % kStages;
        if (has_next) {
          cursor_next(prob, imax, nxt);
          for (int qt = 0; qt < 2; ++qt)
            nmode[qt] = tile_mode(prob.seg[nxt.seg], nxt.kt, i0 + qt * kBlockM, nq);
          mbar_wait(k_full + nstage, ((it + 1) / kStages) & 1);
        }
        mbar_wait(v_full + stage, ph);
        tc_fence_after();
        for (int qt = 0; qt < 2; ++qt) {
          if (mode[qt] != kSkip) {
            mbar_wait(p_full + qt, p_cnt[qt] & 1);
            tc_fence_after();
            issue_pv(qt, stage, o_acc[qt]);
            o_acc[qt] = true;
            ++p_cnt[qt];
            tc_commit(o_full + qt);
          }
          if (nmode[qt] != kSkip) {
            issue_qk(qt, nstage);
            tc_commit(s_full + qt);
          }
        }
        tc_commit(kv_empty + stage);
        cur = nxt;
        mode[0] = nmode[0];
        mode[1] = nmode[1];
      }
    }
  } else {
    // ======================================================== softmax warpgroups
    const int qt = warp >> 2;
    const int quad = warp & 3;
    const int row = i0 + qt * kBlockM + quad * 32 + lane;  // problem-local query row
    const uint32_t t_lane = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t tS = tmem + t_lane + qt * 128;
    const uint32_t tO = tmem + t_lane + 256 + qt * 128;
    const float sl2 = P.scale_log2;
    float m_ref = -INFINITY;
    float l = 0.f;
    uint32_t cnt = 0;
    Cursor cur = cursor_at(prob, imax, t_begin);
    for (int it = 0; it < ntiles; ++it, cursor_next(prob, imax, cur)) {
      const AttnSeg sg = prob.seg[cur.seg];
      const int mode = tile_mode(sg, cur.kt, i0 + qt * kBlockM, nq);
      if (mode == kSkip) continue;
      mbar_wait(s_full + qt, cnt & 1);
      tc_fence_after();
      uint32_t sr[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tS + 32 * c, sr[c]);
      tmem_wait_ld();
      if (mode == kPart) {
        const int k0 = cur.kt * kBlockN;
        int lim = sg.len - k0;
        if (sg.causal) lim = min(lim, row - k0 + 1);
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c * 32 + j >= lim) sr[c][j] = __float_as_uint(-INFINITY);
      }
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int j = 0; j < 32; ++j) mx = fmaxf(mx, __uint_as_float(sr[c][j]));
      const float m_new = fmaxf(m_ref, mx * sl2);
      float alpha = 1.f;
      bool rescale = false;
      if (m_new > m_ref + 8.f) {  // lazy rescale: keep a stale max while p <= 2^8
        alpha = exp2f(m_ref - m_new);
        m_ref = m_new;
        rescale = true;
      }
      const float m_use = (m_ref == -INFINITY) ? 0.f : m_ref;
      float sum0 = 0.f, sum1 = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float p0 = fast_exp2(fmaf(__uint_as_float(sr[c][2 * j]), sl2, -m_use));
          const float p1 = fast_exp2(fmaf(__uint_as_float(sr[c][2 * j + 1]), sl2, -m_use));
          sum0 += p0;
          sum1 += p1;
          __nv_bfloat162 b = __floats2bfloat162_rn(p0, p1);  // .x (low) = even key
          pk[j] = *reinterpret_cast<uint32_t*>(&b);
        }
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
            "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(tS + 16 * c),
            "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3]), "r"(pk[4]), "r"(pk[5]), "r"(pk[6]),
            "r"(pk[7]), "r"(pk[8]), "r"(pk[9]), "r"(pk[10]), "r"(pk[11]), "r"(pk[12]),
            "r"(pk[13]), "r"(pk[14]), "r"(pk[15]));
      }
      l = l * alpha + (sum0 + sum1);
      if (rescale && cnt > 0) {
        mbar_wait(o_full + qt, (cnt - 1) & 1);  // PV_{cnt-1} has landed in O
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t o[32];
          tmem_ld32(tO + 32 * c, o);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
          tmem_st32(tO + 32 * c, o);
        }
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_full + qt);
      ++cnt;
    }
    // ---- epilogue: O / l, lse
    if (cnt > 0) {
      mbar_wait(o_full + qt, (cnt - 1) & 1);
      tc_fence_after();
    }
    const bool valid_row = row < nq;
    const float inv = (l > 0.f) ? 1.f / l : 0.f;
    const long long obase = static_cast<long long>(split) * prob.split_stride_out +
                            static_cast<long long>(row) * prob.ldo + head * kHeadDim;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t o[32];
      if (cnt > 0) {
        tmem_ld32(tO + 32 * c, o);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) o[j] = 0u;
      }
      if (valid_row) {
        if (prob.out_f32) {
          float4* dst = reinterpret_cast<float4*>(static_cast<float*>(prob.out) + obase + 32 * c);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            dst[j] = make_float4(__uint_as_float(o[4 * j]) * inv, __uint_as_float(o[4 * j + 1]) * inv,
                                 __uint_as_float(o[4 * j + 2]) * inv,
                                 __uint_as_float(o[4 * j + 3]) * inv);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(prob.out) + obase + 32 * c);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(o[8 * j + 2 * e]) * inv,
                                                       __uint_as_float(o[8 * j + 2 * e + 1]) * inv);
              w[e] = *reinterpret_cast<uint32_t*>(&b);
            }
            dst[j] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
    }
    if (valid_row && prob.lse) {
      const float lse = (l > 0.f) ? (m_ref + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
      prob.lse[static_cast<long long>(split) * prob.split_stride_lse +
               static_cast<long long>(row) * prob.ld_lse + head] = lse;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc(tmem, kTmemCols);
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2D bf16 [rows x cols] row-major (row stride ld elements), box 64 cols x 128 rows, SW128.
bool make_tmap(CUtensorMap* m, const void* base, long long rows, long long cols, long long ld,
               std::string* err) {
  auto enc = tensor_map_encoder();
  if (!enc) {
    if (err) *err = "cuTensorMapEncodeTiled unavailable";
    return false;
  }
  if (rows < 1) rows = 1;  // empty segments are never loaded
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    if (err) *err = "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")";
    return false;
  }
  return true;
}

}  // namespace

cudaError_t launch_attention(const ProbView* probs, int nprob, int hq, int hkv, int dh,
                             cudaStream_t stream, std::string* err) {
  if (dh != kHeadDim) {
    if (err) *err = "attention: only dh == 128 is implemented";
    return cudaErrorInvalidValue;
  }
  if (nprob < 1 || nprob > kMaxProbs || hq < 1 || hkv < 1 || hq % hkv) {
    if (err) *err = "attention: bad problem count or head counts";
    return cudaErrorInvalidValue;
  }
  static AttnParams P;  // large; filled per launch (launch copies params)
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  std::memset(&P, 0, sizeof(P));
  P.hq = hq;
  P.hkv = hkv;
  P.scale_log2 = (1.0f / sqrtf(static_cast<float>(dh))) * 1.4426950408889634f;
  int work = 0;
  int np = 0;
  for (int i = 0; i < nprob; ++i) {
    const ProbView& v = probs[i];
    if (v.nq <= 0) continue;
    if (v.nseg < 0 || v.nseg > kMaxSegs || v.splits < 1) {
      if (err) *err = "attention: bad segment count / splits";
      return cudaErrorInvalidValue;
    }
    AttnProb& p = P.prob[np];
    p.nq = v.nq;
    p.nseg = v.nseg;
    p.units = (v.nq + kTilesPerCta * kBlockM - 1) / (kTilesPerCta * kBlockM);
    p.splits = v.splits;
    p.work_begin = work;
    p.out_f32 = v.out_f32;
    p.out = v.out;
    p.ldo = v.ldo;
    p.split_stride_out = v.split_stride_out;
    p.lse = v.lse;
    p.ld_lse = v.ld_lse;
    p.split_stride_lse = v.split_stride_lse;
    if (!make_tmap(&P.tmap[np][0], v.q, v.nq, static_cast<long long>(hq) * dh, v.ldq, err))
      return cudaErrorInvalidValue;
    for (int s = 0; s < v.nseg; ++s) {
      p.seg[s].len = v.seg[s].len;
      p.seg[s].causal = v.seg[s].causal;
      if (v.seg[s].causal && v.seg[s].len > v.nq) {
        if (err) *err = "attention: causal segment longer than the query";
        return cudaErrorInvalidValue;
      }
      if (!make_tmap(&P.tmap[np][1 + 2 * s], v.seg[s].k, v.seg[s].len,
                     static_cast<long long>(hkv) * dh, v.seg[s].ld, err) ||
          !make_tmap(&P.tmap[np][2 + 2 * s], v.seg[s].v, v.seg[s].len,
                     static_cast<long long>(hkv) * dh, v.seg[s].ld, err))
        return cudaErrorInvalidValue;
    }
    work += p.units * hq * p.splits;
    ++np;
  }
  P.nprob = np;
  P.total_work = work;
  if (work == 0) return cudaSuccess;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kSmemBytes));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  attn_fwd_kernel<<<work, kThreads, kSmemBytes, stream>>>(P);
  return cudaGetLastError();
}

}  // namespace spava
