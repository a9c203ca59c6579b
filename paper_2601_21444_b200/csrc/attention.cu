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
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "ptx.cuh"
#include "spava_internal.h"

namespace spava {

namespace {

constexpr int kVStages = 2;      // V ring depth
constexpr int kMaxKStages = 3;   // K ring depth (template parameter, <= 3)
constexpr int kProducerWarp = 8;
constexpr int kMmaWarp = 9;
constexpr int kThreads = 320;
constexpr uint32_t kBoxBytes = 128 * 64 * 2;    // 128 rows x 64 bf16, one SW128 TMA box
constexpr uint32_t kTileBytes = 2 * kBoxBytes;  // 128 rows x 128 dh
constexpr uint32_t kTmemCols = 512;             // S0 | S1 | O0 | O1

template <int KS>
struct Smem {
  static constexpr uint32_t q = 0;
  static constexpr uint32_t k = q + kTilesPerCta * kTileBytes;
  static constexpr uint32_t v = k + KS * kTileBytes;
  static constexpr uint32_t bar = v + kVStages * kTileBytes;
  static constexpr uint32_t total = bar + 256;
  static constexpr uint32_t bytes = total + 1024;  // + alignment slack
};

enum : int { kSkip = 0, kFull = 1, kPart = 2 };

// dev-only cycle accounting (variant 5): 0 mma wait K, 1 mma wait V, 2 mma wait P,
// 3 mma loop total, 4 softmax wait S, 5 softmax body, 6 softmax tiles, 7 rescales,
// 8 softmax S-load, 9 softmax max
__device__ unsigned long long g_attn_prof[16];
#define PROF_NOW() (kProf ? clock64() : 0ll)


// 2^x for finite x <= 8 (x clamped at -125), fp32 pair: x = n + f, n = rint(x) via the
// 1.5*2^23 magic add, 2^f (|f| <= 1/2) by a minimax cubic (max rel. err 7.8e-5), and n
// added to the exponent field.
// pair j (of 16 per 32-key chunk) takes the FMA-pipe exp2 when kEmu of every 16 do
__device__ __forceinline__ constexpr bool emu_slot(int j, int emu) {
  return emu > 0 && (j % (16 / (emu > 0 ? emu : 1))) == (16 / (emu > 0 ? emu : 1)) - 1;
}

__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 magic = make_float2(0x1.8p23f, 0x1.8p23f);
  const float2 t = __fadd2_rn(x, magic);
  const float2 r = __fadd2_rn(t, make_float2(-0x1.8p23f, -0x1.8p23f));
  const float2 f = __ffma2_rn(r, make_float2(-1.f, -1.f), x);
  float2 p = __ffma2_rn(make_float2(0x1.c4c0d0p-5f, 0x1.c4c0d0p-5f), f,
                        make_float2(0x1.f0e306p-3f, 0x1.f0e306p-3f));
  p = __ffma2_rn(p, f, make_float2(0x1.62f0d0p-1f, 0x1.62f0d0p-1f));
  p = __ffma2_rn(p, f, make_float2(0x1.fff66cp-1f, 0x1.fff66cp-1f));
  // bits(t) = bits(1.5*2^23) + n and bits(1.5*2^23) << 23 == 0 (mod 2^32): one IMAD per lane
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&pk)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3]), "r"(pk[4]), "r"(pk[5]), "r"(pk[6]),
      "r"(pk[7]), "r"(pk[8]), "r"(pk[9]), "r"(pk[10]), "r"(pk[11]), "r"(pk[12]), "r"(pk[13]),
      "r"(pk[14]), "r"(pk[15]));
}

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

template <int kEmu, int KS, bool kProf = false, bool kPipe = false, bool kSpec = true>
__global__ void __launch_bounds__(kThreads, 1) attn_fwd_kernel(const __grid_constant__ AttnParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  using SL = Smem<KS>;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SL::bar);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;                // [KS]
  uint64_t* k_empty = k_full + kMaxKStages;   // [KS] freed once both QK of the tile completed
  uint64_t* v_full = k_empty + kMaxKStages;   // [kVStages]
  uint64_t* v_empty = v_full + kVStages;      // [kVStages] freed once both PV completed
  uint64_t* s_full = v_empty + kVStages;      // [2] S_t ready in TMEM
  uint64_t* p_full = s_full + 2;              // [2] P_t written (and O_t corrected)
  uint64_t* o_full = p_full + 2;              // [2] PV_t complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 2);

  const int warp = warp_id();
  const int lane = lane_id();
  long long pr[14] = {};

  // ---- decode the work item: problem, 256-row unit (heaviest first), head, split
  int pi = 0;
  while (pi + 1 < P.nprob && static_cast<int>(blockIdx.x) >= P.prob[pi + 1].work_begin) ++pi;
  const AttnProb& prob = P.prob[pi];
  int local = static_cast<int>(blockIdx.x) - prob.work_begin;
  const int split = local % prob.splits;
  local /= prob.splits;
  // head pairing (nq <= 128, even GQA group): the two Q tiles are q-heads h, h+1 of one
  // kv group over the same rows, sharing every K/V tile
  const int pair = prob.head_pair;
  const int nheads = pair ? P.hq / 2 : P.hq;
  const int head = pair ? 2 * (local % nheads) : local % nheads;
  local /= nheads;
  const int unit = prob.units - 1 - local;
  const int i0 = pair ? 0 : unit * (kTilesPerCta * kBlockM);
  const int nq = prob.nq;
  const int imax = min(i0 + (pair ? kBlockM : kTilesPerCta * kBlockM), nq);
  const int hk = head / (P.hq / P.hkv);
  // Q tile t covers rows [r0(t), r0(t)+128) of q-head head + pair*t
#define TILE_R0(t) (pair ? 0 : i0 + (t) * kBlockM)
#define TILE_HEAD(t) (head + pair * (t))

  int T = 0;
  for (int s = 0; s < prob.nseg; ++s) T += seg_tiles(prob.seg[s], imax);
  const int t_begin = static_cast<int>(static_cast<long long>(T) * split / prob.splits);
  const int t_end = static_cast<int>(static_cast<long long>(T) * (split + 1) / prob.splits);
  const int ntiles = t_end - t_begin;
  const CUtensorMap* tm = P.tmap[pi];

  if (warp == kProducerWarp && elect_one()) {
    mbar_init(q_full, 1);
    for (int s = 0; s < KS; ++s) {
      mbar_init(k_full + s, 1);
      mbar_init(k_empty + s, 1);
    }
    for (int s = 0; s < kVStages; ++s) {
      mbar_init(v_full + s, 1);
      mbar_init(v_empty + s, 1);
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
      const bool has1 = TILE_R0(1) < nq;
      mbar_expect_tx(q_full, (has1 ? 2u : 1u) * kTileBytes);
      for (int qt = 0; qt < (has1 ? 2 : 1); ++qt)
        for (int c = 0; c < 2; ++c)
          tma_load_2d(smem + SL::q + qt * kTileBytes + c * kBoxBytes, &tm[0], q_full,
                      TILE_HEAD(qt) * kHeadDim + c * 64, TILE_R0(qt));
      Cursor cur = cursor_at(prob, imax, t_begin);
      for (int it = 0; it < ntiles; ++it) {
        const CUtensorMap* km = &tm[1 + 2 * cur.seg];
        const CUtensorMap* vm = &tm[2 + 2 * cur.seg];
        const int ks = it % KS, vs = it % kVStages;
        if (it >= KS) mbar_wait(k_empty + ks, ((it / KS) - 1) & 1);
        mbar_expect_tx(k_full + ks, kTileBytes);
        for (int c = 0; c < 2; ++c)
          tma_load_2d(smem + SL::k + ks * kTileBytes + c * kBoxBytes, km, k_full + ks,
                      hk * kHeadDim + c * 64, cur.kt * kBlockN);
        if (it >= kVStages) mbar_wait(v_empty + vs, ((it / kVStages) - 1) & 1);
        mbar_expect_tx(v_full + vs, kTileBytes);
        for (int c = 0; c < 2; ++c)
          tma_load_2d(smem + SL::v + vs * kTileBytes + c * kBoxBytes, vm, v_full + vs,
                      hk * kHeadDim + c * 64, cur.kt * kBlockN);
        cursor_next(prob, imax, cur);
      }
    }
  } else if (warp == kMmaWarp) {
    // ======================================================== MMA issuer
    if (elect_one()) {
      const uint32_t idesc_qk = idesc_bf16_f32(128, 128, 0, 0);  // Q, K both K-major
      const uint32_t idesc_pv = idesc_bf16_f32(128, 128, 0, 1);  // P (TMEM), V MN-major
      const uint32_t sq = smem_u32(smem + SL::q);
      const uint32_t sk = smem_u32(smem + SL::k);
      const uint32_t sv = smem_u32(smem + SL::v);
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
      const long long tm0 = PROF_NOW();
      Cursor cur = cursor_at(prob, imax, t_begin);
      int mode[2] = {kSkip, kSkip};
      uint32_t p_cnt[2] = {0, 0};
      bool o_acc[2] = {false, false};
      if (ntiles > 0) {
        for (int qt = 0; qt < 2; ++qt)
          mode[qt] = tile_mode(prob.seg[cur.seg], cur.kt, TILE_R0(qt), nq);
        mbar_wait(k_full + 0, 0);
        tc_fence_after();
        for (int qt = 0; qt < 2; ++qt)
          if (mode[qt] != kSkip) {
            issue_qk(qt, 0);
            tc_commit(s_full + qt);
          }
        tc_commit(k_empty + 0);
      }
      // Issue order per tile it: PV0(it) QK0(it+1) PV1(it) [free V(it)] QK1(it+1) [free K(it+1)].
      // P_t aliases S_t in TMEM, so QK_t(it+1) may only follow PV_t(it) (tcgen05 is in-order).
      for (int it = 0; it < ntiles; ++it) {
        const int vs = it % kVStages;
        const bool has_next = it + 1 < ntiles;
        Cursor nxt = cur;
        int nmode[2] = {kSkip, kSkip};
        const int kn = (it + 1) % KS;
        if (has_next) {
          cursor_next(prob, imax, nxt);
          for (int qt = 0; qt < 2; ++qt)
            nmode[qt] = tile_mode(prob.seg[nxt.seg], nxt.kt, TILE_R0(qt), nq);
          const long long tw = PROF_NOW();
          mbar_wait(k_full + kn, ((it + 1) / KS) & 1);
          if (kProf) pr[0] += PROF_NOW() - tw;
        }
        {
          const long long tw = PROF_NOW();
          mbar_wait(v_full + vs, (it / kVStages) & 1);
          if (kProf) pr[1] += PROF_NOW() - tw;
        }
        tc_fence_after();
        for (int qt = 0; qt < 2; ++qt) {
          if (mode[qt] != kSkip) {
            const long long tw = PROF_NOW();
            mbar_wait(p_full + qt, p_cnt[qt] & 1);
            if (kProf) pr[2] += PROF_NOW() - tw;
            tc_fence_after();
            issue_pv(qt, vs, o_acc[qt]);
            o_acc[qt] = true;
            ++p_cnt[qt];
            tc_commit(o_full + qt);
          }
          if (qt == 1) tc_commit(v_empty + vs);
          if (nmode[qt] != kSkip) {
            issue_qk(qt, kn);
            tc_commit(s_full + qt);
          }
        }
        if (has_next) tc_commit(k_empty + kn);
        cur = nxt;
        mode[0] = nmode[0];
        mode[1] = nmode[1];
      }
      if (kProf) pr[3] += PROF_NOW() - tm0;
    }
  } else if (warp < kProducerWarp) {
    // ======================================================== softmax warpgroups
    const int qt = warp >> 2;
    const int quad = warp & 3;
    const int row = TILE_R0(qt) + quad * 32 + lane;  // problem-local query row
    const int qhead = TILE_HEAD(qt);
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
      const int mode = tile_mode(sg, cur.kt, TILE_R0(qt), nq);
      if (mode == kSkip) continue;
      const long long tw0 = PROF_NOW();
      mbar_wait(s_full + qt, cnt & 1);
      const long long tw1 = PROF_NOW();
      if (kProf) pr[4] += tw1 - tw0;
      tc_fence_after();
      float alpha = 1.f;
      bool rescale = false;
      float2 sum2 = make_float2(0.f, 0.f);
      int lim = kBlockN;  // keys c < lim visible (kPart tiles only)
      if (mode == kPart) {
        const int k0 = cur.kt * kBlockN;
        lim = sg.len - k0;
        if (sg.causal) lim = min(lim, row - k0 + 1);
      }
      const float2 sl2v = make_float2(sl2, sl2);
      uint32_t sr[4][32];
      uint32_t pk[4][16];
      // exp + bf16 pack of one 32-key chunk against reference max m (-m in negm)
      // kPipe: exps are written back in place (sr[c] := p bits) and summed/packed by
      // chunk_pack one chunk later, so the FADD2/F2FP never sit right behind the MUFU
      // pair that feeds them (in-order issue stalled on MUFU latency there).
      auto chunk_exp_ip = [&](int c, float2 negm, bool emu) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 x2 = __ffma2_rn(
              make_float2(__uint_as_float(sr[c][2 * j]), __uint_as_float(sr[c][2 * j + 1])), sl2v, negm);
          float2 p2;
          if (kEmu > 0 && emu && emu_slot(j, kEmu))
            p2 = exp2_poly2(x2);
          else
            p2 = make_float2(fast_exp2(x2.x), fast_exp2(x2.y));  // -inf -> 0
          sr[c][2 * j] = __float_as_uint(p2.x);
          sr[c][2 * j + 1] = __float_as_uint(p2.y);
        }
      };
      auto chunk_pack = [&](int c, float2 (&sacc)[4]) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 p2 = make_float2(__uint_as_float(sr[c][2 * j]), __uint_as_float(sr[c][2 * j + 1]));
          sacc[j & 3] = __fadd2_rn(sacc[j & 3], p2);
          __nv_bfloat162 b = __floats2bfloat162_rn(p2.x, p2.y);
          pk[c][j] = *reinterpret_cast<uint32_t*>(&b);
        }
      };
      auto chunk_exp = [&](int c, float2 negm, bool emu, float2 (&sacc)[4]) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 x2 = __ffma2_rn(
              make_float2(__uint_as_float(sr[c][2 * j]), __uint_as_float(sr[c][2 * j + 1])), sl2v, negm);
          float2 p2;
          if (kEmu > 0 && emu && emu_slot(j, kEmu))
            p2 = exp2_poly2(x2);
          else
            p2 = make_float2(fast_exp2(x2.x), fast_exp2(x2.y));  // -inf -> 0
          sacc[j & 3] = __fadd2_rn(sacc[j & 3], p2);
          __nv_bfloat162 b = __floats2bfloat162_rn(p2.x, p2.y);  // .x (low) = even key
          pk[c][j] = *reinterpret_cast<uint32_t*>(&b);
        }
      };
      auto chunk_max = [&](int c, float (&mxp)[8]) {
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const int t = (j / 2) & 7;
          mxp[t] = fmaxf(mxp[t], fmaxf(__uint_as_float(sr[c][j]), __uint_as_float(sr[c][j + 1])));
        }
      };
      auto load_s = [&]() {
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(tS + 32 * c, sr[c]);
        tmem_wait_ld();
      };
      float mxp[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) mxp[t] = -INFINITY;
      float2 sacc[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) sacc[t] = make_float2(0.f, 0.f);
      bool done = false;
      load_s();
      if (kProf) pr[9] += PROF_NOW() - tw1;
      if (kSpec && mode == kFull && m_ref != -INFINITY) {
        // (kSpec only -- measured 1.5 % slower than max-first at C1, so off in production)
        // speculative pass against the running max m_ref: the tile max is folded in on the
        // side instead of sitting on the critical path; P is kept in registers and only
        // committed to TMEM if the tile max stayed within m_ref + 8 (P <= 2^8), the common
        // case after the first tiles; otherwise S is re-read and the exact path runs.
        const float2 negm = make_float2(-m_ref, -m_ref);
        if constexpr (kPipe) {
          chunk_max(0, mxp);
          chunk_exp_ip(0, negm, true);
#pragma unroll
          for (int c = 1; c < 4; ++c) {
            chunk_max(c, mxp);
            chunk_exp_ip(c, negm, true);
            chunk_pack(c - 1, sacc);
          }
          chunk_pack(3, sacc);
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            chunk_max(c, mxp);
            chunk_exp(c, negm, true, sacc);
          }
        }
        const float mx = fmaxf(fmaxf(fmaxf(mxp[0], mxp[1]), fmaxf(mxp[2], mxp[3])),
                               fmaxf(fmaxf(mxp[4], mxp[5]), fmaxf(mxp[6], mxp[7])));
        done = !(mx * sl2 > m_ref + 8.f);
        if (!done) {
#pragma unroll
          for (int t = 0; t < 4; ++t) sacc[t] = make_float2(0.f, 0.f);
          load_s();
        }
      } else if (mode == kPart) {
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c * 32 + j >= lim) sr[c][j] = __float_as_uint(-INFINITY);
      }
      if (kProf) pr[8] += PROF_NOW() - tw1;
      if (!done) {
        // max first, lazy rescale (keep a stale max while p <= 2^8), then exps
#pragma unroll
        for (int t = 0; t < 8; ++t) mxp[t] = -INFINITY;
#pragma unroll
        for (int c = 0; c < 4; ++c) chunk_max(c, mxp);
        const float mx = fmaxf(fmaxf(fmaxf(mxp[0], mxp[1]), fmaxf(mxp[2], mxp[3])),
                               fmaxf(fmaxf(mxp[4], mxp[5]), fmaxf(mxp[6], mxp[7])));
        const float m_new = fmaxf(m_ref, mx * sl2);
        if (m_new > m_ref + 8.f) {
          alpha = exp2f(m_ref - m_new);
          m_ref = m_new;
          rescale = true;
        }
        const float m_use = (m_ref == -INFINITY) ? 0.f : m_ref;
        const float2 negm = make_float2(-m_use, -m_use);
        if constexpr (kPipe) {
          chunk_exp_ip(0, negm, mode == kFull);
#pragma unroll
          for (int c = 1; c < 4; ++c) {
            chunk_exp_ip(c, negm, mode == kFull);
            chunk_pack(c - 1, sacc);
          }
          chunk_pack(3, sacc);
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) chunk_exp(c, negm, mode == kFull, sacc);
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_st16(tS + 16 * c, pk[c]);
      sum2 = __fadd2_rn(__fadd2_rn(sacc[0], sacc[1]), __fadd2_rn(sacc[2], sacc[3]));
      const long long tp3 = PROF_NOW();
      l = l * alpha + (sum2.x + sum2.y);
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
      if (kProf) {
        pr[12] += PROF_NOW() - tp3;
        pr[5] += PROF_NOW() - tw1;
        pr[6] += 1;
        pr[7] += rescale ? 1 : 0;
      }
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
                            static_cast<long long>(row) * prob.ldo + qhead * kHeadDim;
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
               static_cast<long long>(row) * prob.ld_lse + qhead] = lse;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (kProf && (warp == kMmaWarp || (warp < kProducerWarp && lane == 0)))
    for (int i = 0; i < 14; ++i)
      if (pr[i]) atomicAdd(&g_attn_prof[i], static_cast<unsigned long long>(pr[i]));
  if (warp == kMmaWarp) tmem_dealloc(tmem, kTmemCols);
#undef TILE_R0
#undef TILE_HEAD
}

// ============================================================================ variant family 4
// Ping-pong family with the score tile split across time: P is stored in the UPPER half of
// the S columns (64..127) and QK(j+1) is issued as two N=64 halves.  Half A (keys 0-63 ->
// S columns 0-63) is issued as soon as the softmax has pulled S(j) into registers (after
// its row max), i.e. while tile j's exps still run; P(j) is committed in two halves so
// PV(j) starts on keys 0-63 while the softmax is still on keys 64-127; half B of QK(j+1)
// (columns 64-127) follows PV(j) in the in-order tensor pipe.  The softmax of tile j+1
// then waits only for PV(j)_B + QK(j+1)_B after its last commit instead of a full PV+QK.
// The MMA warp is a small scheduler polling both Q tiles' barriers (no head-of-line
// blocking between the two softmax warpgroups).
template <int kEmu>
__global__ void __launch_bounds__(kThreads, 1) attn_fwd4_kernel(const __grid_constant__ AttnParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  using SL = Smem<2>;
  constexpr int KS = 2;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SL::bar);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;        // [2]
  uint64_t* k_empty = k_full + 2;     // [2]
  uint64_t* v_full = k_empty + 2;     // [2]
  uint64_t* v_empty = v_full + 2;     // [2]
  uint64_t* sA = v_empty + 2;         // [2 Q tiles] QK half A (S cols 0-63) landed
  uint64_t* sB = sA + 2;              // [2] QK half B (S cols 64-127) landed
  uint64_t* sfree = sB + 2;           // [2] softmax holds S(j) in registers (128 arrivals)
  uint64_t* pA = sfree + 2;           // [2] P keys 0-63 stored (and O corrected)
  uint64_t* pB = pA + 2;              // [2] P keys 64-127 stored
  uint64_t* o_full = pB + 2;          // [2] PV half B of the tile complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 2);

  const int warp = warp_id();
  const int lane = lane_id();

  int pi = 0;
  while (pi + 1 < P.nprob && static_cast<int>(blockIdx.x) >= P.prob[pi + 1].work_begin) ++pi;
  const AttnProb& prob = P.prob[pi];
  int local = static_cast<int>(blockIdx.x) - prob.work_begin;
  const int split = local % prob.splits;
  local /= prob.splits;
  const int pair = prob.head_pair;
  const int nheads = pair ? P.hq / 2 : P.hq;
  const int head = pair ? 2 * (local % nheads) : local % nheads;
  local /= nheads;
  const int unit = prob.units - 1 - local;
  const int i0 = pair ? 0 : unit * (kTilesPerCta * kBlockM);
  const int nq = prob.nq;
  const int imax = min(i0 + (pair ? kBlockM : kTilesPerCta * kBlockM), nq);
  const int hk = head / (P.hq / P.hkv);
#define TILE_R0(t) (pair ? 0 : i0 + (t) * kBlockM)
#define TILE_HEAD(t) (head + pair * (t))

  int T = 0;
  for (int s = 0; s < prob.nseg; ++s) T += seg_tiles(prob.seg[s], imax);
  const int t_begin = static_cast<int>(static_cast<long long>(T) * split / prob.splits);
  const int t_end = static_cast<int>(static_cast<long long>(T) * (split + 1) / prob.splits);
  const int ntiles = t_end - t_begin;
  const CUtensorMap* tm = P.tmap[pi];
  // Q tile t processes a prefix of the KV tiles (causal skips only trail the own segment)
  int nt[2] = {0, 0};
  {
    Cursor c = cursor_at(prob, imax, t_begin);
    for (int it = 0; it < ntiles; ++it, cursor_next(prob, imax, c))
      for (int qt = 0; qt < 2; ++qt)
        if (tile_mode(prob.seg[c.seg], c.kt, TILE_R0(qt), nq) != kSkip) nt[qt] = it + 1;
  }

  if (warp == kProducerWarp && elect_one()) {
    mbar_init(q_full, 1);
    for (int s = 0; s < KS; ++s) {
      mbar_init(k_full + s, 1);
      mbar_init(k_empty + s, 1);
      mbar_init(v_full + s, 1);
      mbar_init(v_empty + s, 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(sA + t, 1);
      mbar_init(sB + t, 1);
      mbar_init(sfree + t, 128);
      mbar_init(pA + t, 128);
      mbar_init(pB + t, 128);
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
    // ======================================================== TMA producer (as family 0)
    if (elect_one()) {
      const bool has1 = TILE_R0(1) < nq;
      mbar_expect_tx(q_full, (has1 ? 2u : 1u) * kTileBytes);
      for (int qt = 0; qt < (has1 ? 2 : 1); ++qt)
        for (int c = 0; c < 2; ++c)
          tma_load_2d(smem + SL::q + qt * kTileBytes + c * kBoxBytes, &tm[0], q_full,
                      TILE_HEAD(qt) * kHeadDim + c * 64, TILE_R0(qt));
      Cursor cur = cursor_at(prob, imax, t_begin);
      for (int it = 0; it < ntiles; ++it) {
        const CUtensorMap* km = &tm[1 + 2 * cur.seg];
        const CUtensorMap* vm = &tm[2 + 2 * cur.seg];
        const int ks = it % KS, vs = it % kVStages;
        if (it >= KS) mbar_wait(k_empty + ks, ((it / KS) - 1) & 1);
        mbar_expect_tx(k_full + ks, kTileBytes);
        for (int c = 0; c < 2; ++c)
          tma_load_2d(smem + SL::k + ks * kTileBytes + c * kBoxBytes, km, k_full + ks,
                      hk * kHeadDim + c * 64, cur.kt * kBlockN);
        if (it >= kVStages) mbar_wait(v_empty + vs, ((it / kVStages) - 1) & 1);
        mbar_expect_tx(v_full + vs, kTileBytes);
        for (int c = 0; c < 2; ++c)
          tma_load_2d(smem + SL::v + vs * kTileBytes + c * kBoxBytes, vm, v_full + vs,
                      hk * kHeadDim + c * 64, cur.kt * kBlockN);
        cursor_next(prob, imax, cur);
      }
    }
  } else if (warp == kMmaWarp) {
    // ======================================================== MMA scheduler
    if (elect_one()) {
      const uint32_t idesc_h = idesc_bf16_f32(128, 64, 0, 0);    // QK half: N = 64 keys
      const uint32_t idesc_pv = idesc_bf16_f32(128, 128, 0, 1);  // P (TMEM), V MN-major
      const uint32_t sq = smem_u32(smem + SL::q);
      const uint32_t sk = smem_u32(smem + SL::k);
      const uint32_t sv = smem_u32(smem + SL::v);
      // QK(j) half h of Q tile qt: S cols [64h, 64h+64) <- Q_qt x K(j) rows [64h, 64h+64)
      auto issue_qk_half = [&](int qt, int j, int h) {
        const int ks = j % KS;
        const uint32_t d = tmem + qt * 128 + h * 64;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t koff = (kk >> 2) * kBoxBytes + (kk & 3) * 32;
          mma_ss(d, sdesc_sw128(sq + qt * kTileBytes + koff, 16, 1024),
                 sdesc_sw128(sk + ks * kTileBytes + koff + h * 64 * 128, 16, 1024), idesc_h,
                 kk > 0 ? 1u : 0u);
        }
      };
      // PV(j) half h: O_qt += P[keys 64h..64h+63] x V(j) rows [64h, 64h+64)
      auto issue_pv_half = [&](int qt, int j, int h) {
        const int vs = j % kVStages;
        const uint32_t d = tmem + 256 + qt * 128;
        const uint32_t a = tmem + qt * 128 + 64;
#pragma unroll
        for (int kk = 4 * h; kk < 4 * h + 4; ++kk)
          mma_ts(d, a + kk * 8, sdesc_sw128(sv + vs * kTileBytes + kk * 2048, kBoxBytes, 1024), idesc_pv,
                 (j > 0 || kk > 0) ? 1u : 0u);
      };
      // K(j) / V(j) are released once every Q tile that uses tile j has issued its last MMA on it
      auto users = [&](int j) { return (nt[0] > j ? 1 : 0) + (nt[1] > j ? 1 : 0); };
      int k_done[KS] = {0, 0}, v_done[kVStages] = {0, 0};
      auto k_release = [&](int j) {
        if (++k_done[j % KS] == users(j)) {
          tc_commit(k_empty + j % KS);
          k_done[j % KS] = 0;
        }
      };
      auto v_release = [&](int j) {
        if (++v_done[j % kVStages] == users(j)) {
          tc_commit(v_empty + j % kVStages);
          v_done[j % kVStages] = 0;
        }
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      if (ntiles > 0) {
        mbar_wait(k_full, 0);
        tc_fence_after();
        for (int qt = 0; qt < 2; ++qt)
          if (nt[qt] > 0) {
            issue_qk_half(qt, 0, 0);
            tc_commit(sA + qt);
            issue_qk_half(qt, 0, 1);
            tc_commit(sB + qt);
            k_release(0);
          }
      }
      // per Q tile: current tile j and phase (0: QK_A(j+1) after sfree(j), 1: PV_A(j) after
      // pA(j), 2: PV_B(j) + QK_B(j+1) after pB(j))
      int j[2] = {0, 0}, ph[2] = {0, 0};
      bool a_issued[2] = {false, false};  // QK_A(j+1) issued for the current j
      auto finished = [&](int qt) { return j[qt] >= nt[qt]; };
      while (!(finished(0) && finished(1))) {
        for (int qt = 0; qt < 2; ++qt) {
          if (finished(qt)) continue;
          const int jj = j[qt];
          const bool next = jj + 1 < nt[qt];
          if (ph[qt] == 0) {
            if (!next) {
              ph[qt] = 1;
            } else if (mbar_try(sfree + qt, jj & 1) && mbar_try(k_full + (jj + 1) % KS, ((jj + 1) / KS) & 1)) {
              tc_fence_after();
              issue_qk_half(qt, jj + 1, 0);
              tc_commit(sA + qt);
              a_issued[qt] = true;
              ph[qt] = 1;
            }
          }
          if (ph[qt] == 1) {
            if (mbar_try(pA + qt, jj & 1) && mbar_try(v_full + jj % kVStages, (jj / kVStages) & 1)) {
              tc_fence_after();
              issue_pv_half(qt, jj, 0);
              ph[qt] = 2;
            }
          }
          if (ph[qt] == 2) {
            if (mbar_try(pB + qt, jj & 1)) {
              tc_fence_after();
              issue_pv_half(qt, jj, 1);
              tc_commit(o_full + qt);
              v_release(jj);
              if (next) {
                issue_qk_half(qt, jj + 1, 1);
                tc_commit(sB + qt);
                k_release(jj + 1);
              }
              a_issued[qt] = false;
              ph[qt] = 0;
              ++j[qt];
            }
          }
        }
      }
    }
  } else if (warp < kProducerWarp) {
    // ======================================================== softmax warpgroups
    const int qt = warp >> 2;
    const int quad = warp & 3;
    const int row = TILE_R0(qt) + quad * 32 + lane;
    const int qhead = TILE_HEAD(qt);
    const uint32_t t_lane = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t tS = tmem + t_lane + qt * 128;
    const uint32_t tO = tmem + t_lane + 256 + qt * 128;
    const float sl2 = P.scale_log2;
    const float2 sl2v = make_float2(sl2, sl2);
    float m_ref = -INFINITY;
    float l = 0.f;
    Cursor cur = cursor_at(prob, imax, t_begin);
    uint32_t sr[4][32];
    uint32_t pk[2][16];
    for (int it = 0; it < nt[qt]; ++it, cursor_next(prob, imax, cur)) {
      const AttnSeg sg = prob.seg[cur.seg];
      const int mode = tile_mode(sg, cur.kt, TILE_R0(qt), nq);
      mbar_wait(sA + qt, it & 1);
      mbar_wait(sB + qt, it & 1);
      tc_fence_after();
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
          for (int jv = 0; jv < 32; ++jv)
            if (c * 32 + jv >= lim) sr[c][jv] = __float_as_uint(-INFINITY);
      }
      float mxp[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) mxp[t] = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int jv = 0; jv < 32; jv += 2) {
          const int t = (jv / 2) & 7;
          mxp[t] = fmaxf(mxp[t], fmaxf(__uint_as_float(sr[c][jv]), __uint_as_float(sr[c][jv + 1])));
        }
      // S is in registers: the next tile's QK half A may overwrite S columns 0-63 now
      tc_fence_before();
      mbar_arrive(sfree + qt);
      const float mx = fmaxf(fmaxf(fmaxf(mxp[0], mxp[1]), fmaxf(mxp[2], mxp[3])),
                             fmaxf(fmaxf(mxp[4], mxp[5]), fmaxf(mxp[6], mxp[7])));
      float alpha = 1.f;
      bool rescale = false;
      const float m_new = fmaxf(m_ref, mx * sl2);
      if (m_new > m_ref + 8.f) {  // lazy rescale (P <= 2^8 otherwise)
        alpha = exp2f(m_ref - m_new);
        m_ref = m_new;
        rescale = true;
      }
      const float m_use = (m_ref == -INFINITY) ? 0.f : m_ref;
      const float2 negm = make_float2(-m_use, -m_use);
      float2 sacc[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) sacc[t] = make_float2(0.f, 0.f);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int c = 2 * h + cc;
#pragma unroll
          for (int jv = 0; jv < 16; ++jv) {
            const float2 x2 = __ffma2_rn(make_float2(__uint_as_float(sr[c][2 * jv]),
                                                     __uint_as_float(sr[c][2 * jv + 1])), sl2v, negm);
            float2 p2;
            if (kEmu > 0 && mode == kFull && emu_slot(jv, kEmu))
              p2 = exp2_poly2(x2);
            else
              p2 = make_float2(fast_exp2(x2.x), fast_exp2(x2.y));
            sacc[jv & 3] = __fadd2_rn(sacc[jv & 3], p2);
            __nv_bfloat162 bb = __floats2bfloat162_rn(p2.x, p2.y);
            pk[cc][jv] = *reinterpret_cast<uint32_t*>(&bb);
          }
        }
        // P keys [64h, 64h+64) -> S columns 64 + 32h .. (packed bf16 pairs)
        tmem_st16(tS + 64 + 32 * h, pk[0]);
        tmem_st16(tS + 64 + 32 * h + 16, pk[1]);
        if (h == 0 && rescale && it > 0) {
          // PV(it-1) is complete: S(it) half B only landed after it in the tensor pipe
          mbar_wait(o_full + qt, (it - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            tmem_ld32(tO + 32 * c, o);
            tmem_wait_ld();
#pragma unroll
            for (int jv = 0; jv < 32; ++jv) o[jv] = __float_as_uint(__uint_as_float(o[jv]) * alpha);
            tmem_st32(tO + 32 * c, o);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(h == 0 ? pA + qt : pB + qt);
      }
      const float2 sum2 = __fadd2_rn(__fadd2_rn(sacc[0], sacc[1]), __fadd2_rn(sacc[2], sacc[3]));
      l = l * alpha + (sum2.x + sum2.y);
    }
    // ---- epilogue: O / l, lse
    const int cnt = nt[qt];
    if (cnt > 0) {
      mbar_wait(o_full + qt, (cnt - 1) & 1);  // only PV(cnt-1) can still be in flight
      tc_fence_after();
    }
    const bool valid_row = row < nq;
    const float inv = (l > 0.f) ? 1.f / l : 0.f;
    const long long obase = static_cast<long long>(split) * prob.split_stride_out +
                            static_cast<long long>(row) * prob.ldo + qhead * kHeadDim;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t o[32];
      if (cnt > 0) {
        tmem_ld32(tO + 32 * c, o);
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int jv = 0; jv < 32; ++jv) o[jv] = 0u;
      }
      if (valid_row) {
        if (prob.out_f32) {
          float4* dst = reinterpret_cast<float4*>(static_cast<float*>(prob.out) + obase + 32 * c);
#pragma unroll
          for (int jv = 0; jv < 8; ++jv)
            dst[jv] = make_float4(__uint_as_float(o[4 * jv]) * inv, __uint_as_float(o[4 * jv + 1]) * inv,
                                  __uint_as_float(o[4 * jv + 2]) * inv, __uint_as_float(o[4 * jv + 3]) * inv);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(prob.out) + obase + 32 * c);
#pragma unroll
          for (int jv = 0; jv < 4; ++jv) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              __nv_bfloat162 bb = __floats2bfloat162_rn(__uint_as_float(o[8 * jv + 2 * e]) * inv,
                                                        __uint_as_float(o[8 * jv + 2 * e + 1]) * inv);
              w[e] = *reinterpret_cast<uint32_t*>(&bb);
            }
            dst[jv] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
    }
    if (valid_row && prob.lse) {
      const float lse = (l > 0.f) ? (m_ref + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
      prob.lse[static_cast<long long>(split) * prob.split_stride_lse +
               static_cast<long long>(row) * prob.ld_lse + qhead] = lse;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc(tmem, kTmemCols);
#undef TILE_R0
#undef TILE_HEAD
}

// ============================================================================ variant family 1
// One Q tile (128 rows of one q-head) per CTA with the score accumulator double-buffered
// in TMEM: S_0 | S_1 | O (384 of 512 columns).  The MMA warp issues QK(j+2) into the buffer
// of tile j right behind PV(j), so S(j+1) is already resident when the softmax finishes
// tile j: the per-tile critical loop is the softmax body alone (not body + PV + QK as in
// the ping-pong family, whose QK(j+1) must wait for PV(j) because P aliases S).
//   warps 0-3  softmax (thread = TMEM lane = query row), epilogue
//   warp 4     TMA producer (Q once, then K/V rings)
//   warp 5     TMEM allocator + single-thread tcgen05.mma issuer
constexpr int kThreads1 = 192;
constexpr int kKS1 = 3, kVS1 = 2;
struct Smem1 {
  static constexpr uint32_t q = 0;
  static constexpr uint32_t k = q + kTileBytes;
  static constexpr uint32_t v = k + kKS1 * kTileBytes;
  static constexpr uint32_t bar = v + kVS1 * kTileBytes;
  static constexpr uint32_t total = bar + 256;
  static constexpr uint32_t bytes = total + 1024;
};

template <int kEmu, bool kPipe>
__global__ void __launch_bounds__(kThreads1, 1) attn_fwd1_kernel(const __grid_constant__ AttnParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem1::bar);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;           // [kKS1]
  uint64_t* k_empty = k_full + kKS1;     // [kKS1]
  uint64_t* v_full = k_empty + kKS1;     // [kVS1]
  uint64_t* v_empty = v_full + kVS1;     // [kVS1]
  uint64_t* s_full = v_empty + kVS1;     // [2] S buffer b holds a fresh QK
  uint64_t* p_full = s_full + 2;         // [2] P written into buffer b (O corrected)
  uint64_t* o_full = p_full + 2;         // PV complete
  uint64_t* o_done = o_full + 1;         // every MMA of the CTA complete (epilogue)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 1);

  const int warp = warp_id();
  const int lane = lane_id();

  int pi = 0;
  while (pi + 1 < P.nprob && static_cast<int>(blockIdx.x) >= P.prob[pi + 1].work_begin) ++pi;
  const AttnProb& prob = P.prob[pi];
  int local = static_cast<int>(blockIdx.x) - prob.work_begin;
  const int split = local % prob.splits;
  local /= prob.splits;
  const int head = local % P.hq;
  local /= P.hq;
  const int unit = prob.units - 1 - local;  // heaviest (latest causal rows) first
  const int i0 = unit * kBlockM;
  const int nq = prob.nq;
  const int imax = min(i0 + kBlockM, nq);
  const int hk = head / (P.hq / P.hkv);

  int T = 0;
  for (int s = 0; s < prob.nseg; ++s) T += seg_tiles(prob.seg[s], imax);
  const int t_begin = static_cast<int>(static_cast<long long>(T) * split / prob.splits);
  const int t_end = static_cast<int>(static_cast<long long>(T) * (split + 1) / prob.splits);
  const int ntiles = t_end - t_begin;
  const CUtensorMap* tm = P.tmap[pi];

  if (warp == 4 && elect_one()) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kKS1; ++s) {
      mbar_init(k_full + s, 1);
      mbar_init(k_empty + s, 1);
    }
    for (int s = 0; s < kVS1; ++s) {
      mbar_init(v_full + s, 1);
      mbar_init(v_empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(s_full + b, 1);
      mbar_init(p_full + b, 128);
    }
    mbar_init(o_full, 1);
    mbar_init(o_done, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tm[0]);
    for (int s = 0; s < prob.nseg; ++s) {
      tma_prefetch_desc(&tm[1 + 2 * s]);
      tma_prefetch_desc(&tm[2 + 2 * s]);
    }
  }
  if (warp == 5) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 4) {
    // ======================================================== TMA producer
    if (elect_one()) {
      mbar_expect_tx(q_full, kTileBytes);
      for (int c = 0; c < 2; ++c)
        tma_load_2d(smem + Smem1::q + c * kBoxBytes, &tm[0], q_full, head * kHeadDim + c * 64, i0);
      Cursor cur = cursor_at(prob, imax, t_begin);
      for (int it = 0; it < ntiles; ++it) {
        const CUtensorMap* km = &tm[1 + 2 * cur.seg];
        const CUtensorMap* vm = &tm[2 + 2 * cur.seg];
        const int ks = it % kKS1, vs = it % kVS1;
        if (it >= kKS1) mbar_wait(k_empty + ks, ((it / kKS1) - 1) & 1);
        mbar_expect_tx(k_full + ks, kTileBytes);
        for (int c = 0; c < 2; ++c)
          tma_load_2d(smem + Smem1::k + ks * kTileBytes + c * kBoxBytes, km, k_full + ks,
                      hk * kHeadDim + c * 64, cur.kt * kBlockN);
        if (it >= kVS1) mbar_wait(v_empty + vs, ((it / kVS1) - 1) & 1);
        mbar_expect_tx(v_full + vs, kTileBytes);
        for (int c = 0; c < 2; ++c)
          tma_load_2d(smem + Smem1::v + vs * kTileBytes + c * kBoxBytes, vm, v_full + vs,
                      hk * kHeadDim + c * 64, cur.kt * kBlockN);
        cursor_next(prob, imax, cur);
      }
    }
  } else if (warp == 5) {
    // ======================================================== MMA issuer
    if (elect_one()) {
      const uint32_t idesc_qk = idesc_bf16_f32(128, 128, 0, 0);
      const uint32_t idesc_pv = idesc_bf16_f32(128, 128, 0, 1);
      const uint32_t sq = smem_u32(smem + Smem1::q);
      const uint32_t sk = smem_u32(smem + Smem1::k);
      const uint32_t sv = smem_u32(smem + Smem1::v);
      auto issue_qk = [&](int b, int it) {
        const int ks = it % kKS1;
        mbar_wait(k_full + ks, (it / kKS1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + b * 128;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t koff = (kk >> 2) * kBoxBytes + (kk & 3) * 32;
          mma_ss(d, sdesc_sw128(sq + koff, 16, 1024), sdesc_sw128(sk + ks * kTileBytes + koff, 16, 1024),
                 idesc_qk, kk > 0 ? 1u : 0u);
        }
        tc_commit(s_full + b);
        tc_commit(k_empty + ks);
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      if (ntiles > 0) issue_qk(0, 0);
      if (ntiles > 1) issue_qk(1, 1);
      for (int it = 0; it < ntiles; ++it) {
        const int b = it & 1, vs = it % kVS1;
        mbar_wait(v_full + vs, (it / kVS1) & 1);
        mbar_wait(p_full + b, (it >> 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + 256;
        const uint32_t a = tmem + b * 128;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(d, a + kk * 8, sdesc_sw128(sv + vs * kTileBytes + kk * 2048, kBoxBytes, 1024), idesc_pv,
                 (it > 0 || kk > 0) ? 1u : 0u);
        tc_commit(o_full);
        tc_commit(v_empty + vs);
        // QK(it+2) reuses buffer b: issued behind PV(it), the in-order tensor pipe keeps
        // P(it) intact until PV(it) has read it.
        if (it + 2 < ntiles) issue_qk(b, it + 2);
      }
      tc_commit(o_done);
    }
  } else {
    // ======================================================== softmax warpgroup
    const int quad = warp;
    const int row = i0 + quad * 32 + lane;
    const uint32_t t_lane = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t tO = tmem + t_lane + 256;
    const float sl2 = P.scale_log2;
    const float2 sl2v = make_float2(sl2, sl2);
    float m_ref = -INFINITY;
    float l = 0.f;
    Cursor cur = cursor_at(prob, imax, t_begin);
    uint32_t sr[4][32];
    uint32_t pk[4][16];
    for (int it = 0; it < ntiles; ++it, cursor_next(prob, imax, cur)) {
      const int b = it & 1;
      const uint32_t tS = tmem + t_lane + b * 128;
      const AttnSeg sg = prob.seg[cur.seg];
      const int mode = tile_mode(sg, cur.kt, i0, nq);
      mbar_wait(s_full + b, (it >> 1) & 1);
      tc_fence_after();
      auto load_s = [&]() {
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(tS + 32 * c, sr[c]);
        tmem_wait_ld();
      };
      auto chunk_max = [&](int c, float (&mxp)[8]) {
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const int t = (j / 2) & 7;
          mxp[t] = fmaxf(mxp[t], fmaxf(__uint_as_float(sr[c][j]), __uint_as_float(sr[c][j + 1])));
        }
      };
      auto chunk_exp = [&](int c, float2 negm, bool emu) {  // in place: sr[c] := p
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 x2 = __ffma2_rn(
              make_float2(__uint_as_float(sr[c][2 * j]), __uint_as_float(sr[c][2 * j + 1])), sl2v, negm);
          float2 p2;
          if (kEmu > 0 && emu && emu_slot(j, kEmu))
            p2 = exp2_poly2(x2);
          else
            p2 = make_float2(fast_exp2(x2.x), fast_exp2(x2.y));  // -inf -> 0
          sr[c][2 * j] = __float_as_uint(p2.x);
          sr[c][2 * j + 1] = __float_as_uint(p2.y);
        }
      };
      auto chunk_pack = [&](int c, float2 (&sacc)[4]) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 p2 = make_float2(__uint_as_float(sr[c][2 * j]), __uint_as_float(sr[c][2 * j + 1]));
          sacc[j & 3] = __fadd2_rn(sacc[j & 3], p2);
          __nv_bfloat162 bb = __floats2bfloat162_rn(p2.x, p2.y);
          pk[c][j] = *reinterpret_cast<uint32_t*>(&bb);
        }
      };
      auto exp_pack_all = [&](float2 negm, bool emu, float2 (&sacc)[4]) {
        if constexpr (kPipe) {
          chunk_exp(0, negm, emu);
#pragma unroll
          for (int c = 1; c < 4; ++c) {
            chunk_exp(c, negm, emu);
            chunk_pack(c - 1, sacc);
          }
          chunk_pack(3, sacc);
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            chunk_exp(c, negm, emu);
            chunk_pack(c, sacc);
          }
        }
      };
      float alpha = 1.f;
      bool rescale = false;
      float mxp[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) mxp[t] = -INFINITY;
      float2 sacc[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) sacc[t] = make_float2(0.f, 0.f);
      bool done = false;
      load_s();
      if (mode == kFull && m_ref != -INFINITY) {
        // speculative pass against the running max (see the ping-pong kernel)
        const float2 negm = make_float2(-m_ref, -m_ref);
#pragma unroll
        for (int c = 0; c < 4; ++c) chunk_max(c, mxp);
        exp_pack_all(negm, true, sacc);
        const float mx = fmaxf(fmaxf(fmaxf(mxp[0], mxp[1]), fmaxf(mxp[2], mxp[3])),
                               fmaxf(fmaxf(mxp[4], mxp[5]), fmaxf(mxp[6], mxp[7])));
        done = !(mx * sl2 > m_ref + 8.f);
        if (!done) {
#pragma unroll
          for (int t = 0; t < 8; ++t) mxp[t] = -INFINITY;
#pragma unroll
          for (int t = 0; t < 4; ++t) sacc[t] = make_float2(0.f, 0.f);
          load_s();
        }
      } else if (mode == kPart) {
        const int k0 = cur.kt * kBlockN;
        int lim = sg.len - k0;
        if (sg.causal) lim = min(lim, row - k0 + 1);
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c * 32 + j >= lim) sr[c][j] = __float_as_uint(-INFINITY);
      }
      if (!done) {
#pragma unroll
        for (int c = 0; c < 4; ++c) chunk_max(c, mxp);
        const float mx = fmaxf(fmaxf(fmaxf(mxp[0], mxp[1]), fmaxf(mxp[2], mxp[3])),
                               fmaxf(fmaxf(mxp[4], mxp[5]), fmaxf(mxp[6], mxp[7])));
        const float m_new = fmaxf(m_ref, mx * sl2);
        if (m_new > m_ref + 8.f) {
          alpha = exp2f(m_ref - m_new);
          m_ref = m_new;
          rescale = true;
        }
        const float m_use = (m_ref == -INFINITY) ? 0.f : m_ref;
        exp_pack_all(make_float2(-m_use, -m_use), mode == kFull, sacc);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_st16(tS + 16 * c, pk[c]);
      const float2 sum2 = __fadd2_rn(__fadd2_rn(sacc[0], sacc[1]), __fadd2_rn(sacc[2], sacc[3]));
      l = l * alpha + (sum2.x + sum2.y);
      if (rescale && it > 0) {
        mbar_wait(o_full, (it - 1) & 1);  // PV(it-1) has landed in O
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
      mbar_arrive(p_full + b);
    }
    // ---- epilogue: O / l, lse
    // S double-buffered: PV(n-1) and PV(n) may both be in flight, which a parity wait on
    // o_full cannot disambiguate -- wait for the MMA warp's final commit instead.
    mbar_wait(o_done, 0);
    tc_fence_after();
    const bool valid_row = row < nq;
    const float inv = (l > 0.f) ? 1.f / l : 0.f;
    const long long obase = static_cast<long long>(split) * prob.split_stride_out +
                            static_cast<long long>(row) * prob.ldo + head * kHeadDim;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t o[32];
      if (ntiles > 0) {
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
                                 __uint_as_float(o[4 * j + 2]) * inv, __uint_as_float(o[4 * j + 3]) * inv);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(prob.out) + obase + 32 * c);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              __nv_bfloat162 bb = __floats2bfloat162_rn(__uint_as_float(o[8 * j + 2 * e]) * inv,
                                                        __uint_as_float(o[8 * j + 2 * e + 1]) * inv);
              w[e] = *reinterpret_cast<uint32_t*>(&bb);
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
  if (warp == 5) tmem_dealloc(tmem, kTmemCols);
}

// ============================================================================ variant family 3
// Family 1 (one Q tile per CTA, S double-buffered: S_0 | S_1 | O) with the softmax split by
// COLUMNS over two warpgroups: warps 0-3 take keys 0-63 of every tile, warps 4-7 keys
// 64-127 of the same rows (a warp and its partner share TMEM lanes).  Each SMSP then holds
// two softmax warps working on the same tile with half the exps each, so one warp's MUFU
// stream fills the other's issue gaps, and the double-buffered S keeps the next tile's QK
// off the critical path.  The halves agree on the running max through a per-tile exchange
// in shared memory (named barrier of the 256 softmax threads); the row sum is combined in
// the epilogue.
constexpr int kThreads3 = 320;  // warps 0-7 softmax (2 column halves), 8 TMA, 9 MMA
struct Smem3 {
  static constexpr uint32_t q = 0;
  static constexpr uint32_t k = q + kTileBytes;
  static constexpr uint32_t v = k + kKS1 * kTileBytes;
  static constexpr uint32_t xch = v + kVS1 * kTileBytes;        // [2 buf][2 half][128] f32
  static constexpr uint32_t bar = xch + 2 * 2 * 128 * 4;
  static constexpr uint32_t total = bar + 256;
  static constexpr uint32_t bytes = total + 1024;
};

__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int kEmu>
__global__ void __launch_bounds__(kThreads3, 1) attn_fwd3_kernel(const __grid_constant__ AttnParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem3::bar);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;           // [kKS1]
  uint64_t* k_empty = k_full + kKS1;     // [kKS1]
  uint64_t* v_full = k_empty + kKS1;     // [kVS1]
  uint64_t* v_empty = v_full + kVS1;     // [kVS1]
  uint64_t* s_full = v_empty + kVS1;     // [2]
  uint64_t* p_full = s_full + 2;         // [2] both halves' P written (256 arrivals)
  uint64_t* o_full = p_full + 2;         // PV complete
  uint64_t* o_done = o_full + 1;         // every MMA complete (epilogue)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 1);
  float* xch = reinterpret_cast<float*>(smem + Smem3::xch);

  const int warp = warp_id();
  const int lane = lane_id();

  int pi = 0;
  while (pi + 1 < P.nprob && static_cast<int>(blockIdx.x) >= P.prob[pi + 1].work_begin) ++pi;
  const AttnProb& prob = P.prob[pi];
  int local = static_cast<int>(blockIdx.x) - prob.work_begin;
  const int split = local % prob.splits;
  local /= prob.splits;
  const int head = local % P.hq;
  local /= P.hq;
  const int unit = prob.units - 1 - local;
  const int i0 = unit * kBlockM;
  const int nq = prob.nq;
  const int imax = min(i0 + kBlockM, nq);
  const int hk = head / (P.hq / P.hkv);

  int T = 0;
  for (int s = 0; s < prob.nseg; ++s) T += seg_tiles(prob.seg[s], imax);
  const int t_begin = static_cast<int>(static_cast<long long>(T) * split / prob.splits);
  const int t_end = static_cast<int>(static_cast<long long>(T) * (split + 1) / prob.splits);
  const int ntiles = t_end - t_begin;
  const CUtensorMap* tm = P.tmap[pi];

  if (warp == 8 && elect_one()) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kKS1; ++s) {
      mbar_init(k_full + s, 1);
      mbar_init(k_empty + s, 1);
    }
    for (int s = 0; s < kVS1; ++s) {
      mbar_init(v_full + s, 1);
      mbar_init(v_empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(s_full + b, 1);
      mbar_init(p_full + b, 256);
    }
    mbar_init(o_full, 1);
    mbar_init(o_done, 1);
    fence_barrier_init();
    tma_prefetch_desc(&tm[0]);
    for (int s = 0; s < prob.nseg; ++s) {
      tma_prefetch_desc(&tm[1 + 2 * s]);
      tma_prefetch_desc(&tm[2 + 2 * s]);
    }
  }
  if (warp == 9) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    // ======================================================== TMA producer
    if (elect_one()) {
      mbar_expect_tx(q_full, kTileBytes);
      for (int c = 0; c < 2; ++c)
        tma_load_2d(smem + Smem3::q + c * kBoxBytes, &tm[0], q_full, head * kHeadDim + c * 64, i0);
      Cursor cur = cursor_at(prob, imax, t_begin);
      for (int it = 0; it < ntiles; ++it) {
        const CUtensorMap* km = &tm[1 + 2 * cur.seg];
        const CUtensorMap* vm = &tm[2 + 2 * cur.seg];
        const int ks = it % kKS1, vs = it % kVS1;
        if (it >= kKS1) mbar_wait(k_empty + ks, ((it / kKS1) - 1) & 1);
        mbar_expect_tx(k_full + ks, kTileBytes);
        for (int c = 0; c < 2; ++c)
          tma_load_2d(smem + Smem3::k + ks * kTileBytes + c * kBoxBytes, km, k_full + ks,
                      hk * kHeadDim + c * 64, cur.kt * kBlockN);
        if (it >= kVS1) mbar_wait(v_empty + vs, ((it / kVS1) - 1) & 1);
        mbar_expect_tx(v_full + vs, kTileBytes);
        for (int c = 0; c < 2; ++c)
          tma_load_2d(smem + Smem3::v + vs * kTileBytes + c * kBoxBytes, vm, v_full + vs,
                      hk * kHeadDim + c * 64, cur.kt * kBlockN);
        cursor_next(prob, imax, cur);
      }
    }
  } else if (warp == 9) {
    // ======================================================== MMA issuer (as family 1)
    if (elect_one()) {
      const uint32_t idesc_qk = idesc_bf16_f32(128, 128, 0, 0);
      const uint32_t idesc_pv = idesc_bf16_f32(128, 128, 0, 1);
      const uint32_t sq = smem_u32(smem + Smem3::q);
      const uint32_t sk = smem_u32(smem + Smem3::k);
      const uint32_t sv = smem_u32(smem + Smem3::v);
      auto issue_qk = [&](int b, int it) {
        const int ks = it % kKS1;
        mbar_wait(k_full + ks, (it / kKS1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + b * 128;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t koff = (kk >> 2) * kBoxBytes + (kk & 3) * 32;
          mma_ss(d, sdesc_sw128(sq + koff, 16, 1024), sdesc_sw128(sk + ks * kTileBytes + koff, 16, 1024),
                 idesc_qk, kk > 0 ? 1u : 0u);
        }
        tc_commit(s_full + b);
        tc_commit(k_empty + ks);
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      if (ntiles > 0) issue_qk(0, 0);
      if (ntiles > 1) issue_qk(1, 1);
      for (int it = 0; it < ntiles; ++it) {
        const int b = it & 1, vs = it % kVS1;
        mbar_wait(v_full + vs, (it / kVS1) & 1);
        mbar_wait(p_full + b, (it >> 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + 256;
        const uint32_t a = tmem + b * 128;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(d, a + kk * 8, sdesc_sw128(sv + vs * kTileBytes + kk * 2048, kBoxBytes, 1024), idesc_pv,
                 (it > 0 || kk > 0) ? 1u : 0u);
        tc_commit(o_full);
        tc_commit(v_empty + vs);
        if (it + 2 < ntiles) issue_qk(b, it + 2);
      }
      tc_commit(o_done);
    }
  } else {
    // ======================================================== softmax: 2 column halves
    const int half = warp >> 2;   // 0: keys 0-63 of each tile, 1: keys 64-127
    const int quad = warp & 3;
    const int rloc = quad * 32 + lane;
    const int row = i0 + rloc;
    const uint32_t t_lane = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t tO = tmem + t_lane + 256 + half * 64;  // this half rescales/stores O cols
    const float sl2 = P.scale_log2;
    const float2 sl2v = make_float2(sl2, sl2);
    float m_ref = -INFINITY;
    float l = 0.f;
    int xc = 0;  // exchange counter (identical in both halves: same decisions)
    // max of this half's 64 scores, combined with the partner half through smem
    auto exchange_max = [&](float mine) {
      float* buf = xch + (xc & 1) * 256;
      buf[half * 128 + rloc] = mine;
      named_bar_sync(1, 256);
      const float other = buf[(half ^ 1) * 128 + rloc];
      ++xc;
      return fmaxf(mine, other);
    };
    Cursor cur = cursor_at(prob, imax, t_begin);
    uint32_t sr[2][32];
    uint32_t pk[2][16];
    for (int it = 0; it < ntiles; ++it, cursor_next(prob, imax, cur)) {
      const int b = it & 1;
      const uint32_t tS = tmem + t_lane + b * 128;
      const AttnSeg sg = prob.seg[cur.seg];
      const int mode = tile_mode(sg, cur.kt, i0, nq);
      mbar_wait(s_full + b, (it >> 1) & 1);
      tc_fence_after();
      auto load_s = [&]() {
        tmem_ld32(tS + half * 64, sr[0]);
        tmem_ld32(tS + half * 64 + 32, sr[1]);
        tmem_wait_ld();
      };
      auto chunk_max = [&](int c, float (&mxp)[8]) {
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const int t = (j / 2) & 7;
          mxp[t] = fmaxf(mxp[t], fmaxf(__uint_as_float(sr[c][j]), __uint_as_float(sr[c][j + 1])));
        }
      };
      auto chunk_exp = [&](int c, float2 negm, bool emu) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 x2 = __ffma2_rn(
              make_float2(__uint_as_float(sr[c][2 * j]), __uint_as_float(sr[c][2 * j + 1])), sl2v, negm);
          float2 p2;
          if (kEmu > 0 && emu && emu_slot(j, kEmu))
            p2 = exp2_poly2(x2);
          else
            p2 = make_float2(fast_exp2(x2.x), fast_exp2(x2.y));
          sr[c][2 * j] = __float_as_uint(p2.x);
          sr[c][2 * j + 1] = __float_as_uint(p2.y);
        }
      };
      auto chunk_pack = [&](int c, float2 (&sacc)[4]) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 p2 = make_float2(__uint_as_float(sr[c][2 * j]), __uint_as_float(sr[c][2 * j + 1]));
          sacc[j & 3] = __fadd2_rn(sacc[j & 3], p2);
          __nv_bfloat162 bb = __floats2bfloat162_rn(p2.x, p2.y);
          pk[c][j] = *reinterpret_cast<uint32_t*>(&bb);
        }
      };
      auto exp_pack_all = [&](float2 negm, bool emu, float2 (&sacc)[4]) {
        chunk_exp(0, negm, emu);
        chunk_exp(1, negm, emu);
        chunk_pack(0, sacc);
        chunk_pack(1, sacc);
      };
      auto max8 = [](const float (&m)[8]) {
        return fmaxf(fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3])), fmaxf(fmaxf(m[4], m[5]), fmaxf(m[6], m[7])));
      };
      float alpha = 1.f;
      bool rescale = false;
      float mxp[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) mxp[t] = -INFINITY;
      float2 sacc[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) sacc[t] = make_float2(0.f, 0.f);
      bool done = false;
      load_s();
      if (mode == kFull && m_ref != -INFINITY) {
        const float2 negm = make_float2(-m_ref, -m_ref);
        chunk_max(0, mxp);
        chunk_max(1, mxp);
        exp_pack_all(negm, true, sacc);
        const float mx = exchange_max(max8(mxp));
        done = !(mx * sl2 > m_ref + 8.f);
        if (!done) {
#pragma unroll
          for (int t = 0; t < 8; ++t) mxp[t] = -INFINITY;
#pragma unroll
          for (int t = 0; t < 4; ++t) sacc[t] = make_float2(0.f, 0.f);
          load_s();
        }
      } else if (mode == kPart) {
        const int k0 = cur.kt * kBlockN + half * 64;
        int lim = sg.len - k0;
        if (sg.causal) lim = min(lim, row - k0 + 1);
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c * 32 + j >= lim) sr[c][j] = __float_as_uint(-INFINITY);
      }
      if (!done) {
        chunk_max(0, mxp);
        chunk_max(1, mxp);
        const float mx = exchange_max(max8(mxp));
        const float m_new = fmaxf(m_ref, mx * sl2);
        if (m_new > m_ref + 8.f) {
          alpha = exp2f(m_ref - m_new);
          m_ref = m_new;
          rescale = true;
        }
        const float m_use = (m_ref == -INFINITY) ? 0.f : m_ref;
        exp_pack_all(make_float2(-m_use, -m_use), mode == kFull, sacc);
      }
      tmem_st16(tS + half * 32, pk[0]);
      tmem_st16(tS + half * 32 + 16, pk[1]);
      const float2 sum2 = __fadd2_rn(__fadd2_rn(sacc[0], sacc[1]), __fadd2_rn(sacc[2], sacc[3]));
      l = l * alpha + (sum2.x + sum2.y);  // this half's share of the row sum
      if (rescale && it > 0) {
        mbar_wait(o_full, (it - 1) & 1);  // PV(it-1) has landed in O
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
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
      mbar_arrive(p_full + b);
    }
    // ---- epilogue: the row sum of both halves, O / l (this half's 64 columns), lse
    {
      float* buf = xch + (xc & 1) * 256;
      buf[half * 128 + rloc] = l;
      named_bar_sync(1, 256);
      l += buf[(half ^ 1) * 128 + rloc];
    }
    mbar_wait(o_done, 0);
    tc_fence_after();
    const bool valid_row = row < nq;
    const float inv = (l > 0.f) ? 1.f / l : 0.f;
    const long long obase = static_cast<long long>(split) * prob.split_stride_out +
                            static_cast<long long>(row) * prob.ldo + head * kHeadDim + half * 64;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t o[32];
      if (ntiles > 0) {
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
                                 __uint_as_float(o[4 * j + 2]) * inv, __uint_as_float(o[4 * j + 3]) * inv);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(prob.out) + obase + 32 * c);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              __nv_bfloat162 bb = __floats2bfloat162_rn(__uint_as_float(o[8 * j + 2 * e]) * inv,
                                                        __uint_as_float(o[8 * j + 2 * e + 1]) * inv);
              w[e] = *reinterpret_cast<uint32_t*>(&bb);
            }
            dst[j] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
    }
    if (valid_row && prob.lse && half == 0) {
      const float lse = (l > 0.f) ? (m_ref + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
      prob.lse[static_cast<long long>(split) * prob.split_stride_lse +
               static_cast<long long>(row) * prob.ld_lse + head] = lse;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 9) tmem_dealloc(tmem, kTmemCols);
}

// ============================================================================ variant family 2
// Two Q tiles (256 rows, or two q-heads of one GQA group) per CTA as in the ping-pong
// family, but with 64-key KV tiles so each Q tile's score accumulator fits TMEM twice:
// S_0[2] | S_1[2] (64 columns each) | O_0 | O_1 = 512 columns.  QK_t(j+2) is issued right
// behind PV_t(j) into the buffer PV_t(j) just drained, so S_t(j+1) is resident when softmax
// t finishes tile j: the two softmax warpgroups (one warp of each per SMSP) run back to back
// and interleave their MUFU streams instead of each waiting one PV+QK per tile.
constexpr int kBN2 = 64;
constexpr int kKS2 = 4, kVS2 = 4;
constexpr uint32_t kKvBox2 = kBN2 * 64 * 2;     // 64 rows x 64 bf16 (SW128 box)
constexpr uint32_t kKvTile2 = 2 * kKvBox2;      // 64 keys x 128 dh
struct Smem2 {
  static constexpr uint32_t q = 0;
  static constexpr uint32_t k = q + kTilesPerCta * kTileBytes;
  static constexpr uint32_t v = k + kKS2 * kKvTile2;
  static constexpr uint32_t bar = v + kVS2 * kKvTile2;
  static constexpr uint32_t total = bar + 256;
  static constexpr uint32_t bytes = total + 1024;
};

__device__ __forceinline__ int seg_tiles2(const AttnSeg& s, int imax) {
  const int klen = s.causal ? min(s.len, imax) : s.len;
  return klen > 0 ? (klen + kBN2 - 1) / kBN2 : 0;
}
__device__ __forceinline__ int tile_mode2(const AttnSeg& s, int kt, int r0, int nq) {
  if (r0 >= nq) return kSkip;
  const int k0 = kt * kBN2;
  const bool tail = k0 + kBN2 > s.len;
  if (s.causal) {
    const int rlast = min(r0 + kBlockM, nq) - 1;
    if (k0 > rlast) return kSkip;
    return (k0 + kBN2 - 1 > r0 || tail) ? kPart : kFull;
  }
  return tail ? kPart : kFull;
}
__device__ __forceinline__ Cursor cursor_at2(const AttnProb& p, int imax, int t) {
  for (int s = 0; s < p.nseg; ++s) {
    const int n = seg_tiles2(p.seg[s], imax);
    if (t < n) return {s, t};
    t -= n;
  }
  return {p.nseg, 0};
}
__device__ __forceinline__ void cursor_next2(const AttnProb& p, int imax, Cursor& c) {
  ++c.kt;
  while (c.seg < p.nseg && c.kt >= seg_tiles2(p.seg[c.seg], imax)) {
    ++c.seg;
    c.kt = 0;
  }
}

template <int kEmu>
__global__ void __launch_bounds__(kThreads, 1) attn_fwd2_kernel(const __grid_constant__ AttnParams P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem2::bar);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;          // [kKS2]
  uint64_t* k_empty = k_full + kKS2;    // [kKS2]
  uint64_t* v_full = k_empty + kKS2;    // [kVS2]
  uint64_t* v_empty = v_full + kVS2;    // [kVS2]
  uint64_t* s_full = v_empty + kVS2;    // [2 tiles][2 buffers]
  uint64_t* p_full = s_full + 4;        // [2][2]
  uint64_t* o_full = p_full + 4;        // [2] PV_t complete
  uint64_t* o_done = o_full + 2;        // every MMA of the CTA complete (epilogue)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 1);

  const int warp = warp_id();
  const int lane = lane_id();

  int pi = 0;
  while (pi + 1 < P.nprob && static_cast<int>(blockIdx.x) >= P.prob[pi + 1].work_begin) ++pi;
  const AttnProb& prob = P.prob[pi];
  int local = static_cast<int>(blockIdx.x) - prob.work_begin;
  const int split = local % prob.splits;
  local /= prob.splits;
  const int pair = prob.head_pair;
  const int nheads = pair ? P.hq / 2 : P.hq;
  const int head = pair ? 2 * (local % nheads) : local % nheads;
  local /= nheads;
  const int unit = prob.units - 1 - local;
  const int i0 = pair ? 0 : unit * (kTilesPerCta * kBlockM);
  const int nq = prob.nq;
  const int imax = min(i0 + (pair ? kBlockM : kTilesPerCta * kBlockM), nq);
  const int hk = head / (P.hq / P.hkv);
#define TILE_R0(t) (pair ? 0 : i0 + (t) * kBlockM)
#define TILE_HEAD(t) (head + pair * (t))

  int T = 0;
  for (int s = 0; s < prob.nseg; ++s) T += seg_tiles2(prob.seg[s], imax);
  const int t_begin = static_cast<int>(static_cast<long long>(T) * split / prob.splits);
  const int t_end = static_cast<int>(static_cast<long long>(T) * (split + 1) / prob.splits);
  const int ntiles = t_end - t_begin;
  const CUtensorMap* tm = P.tmap[pi];

  if (warp == kProducerWarp && elect_one()) {
    mbar_init(q_full, 1);
    for (int s = 0; s < kKS2; ++s) {
      mbar_init(k_full + s, 1);
      mbar_init(k_empty + s, 1);
    }
    for (int s = 0; s < kVS2; ++s) {
      mbar_init(v_full + s, 1);
      mbar_init(v_empty + s, 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(p_full + i, 128);
    }
    mbar_init(o_full + 0, 1);
    mbar_init(o_full + 1, 1);
    mbar_init(o_done, 1);
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
      const bool has1 = TILE_R0(1) < nq;
      mbar_expect_tx(q_full, (has1 ? 2u : 1u) * kTileBytes);
      for (int qt = 0; qt < (has1 ? 2 : 1); ++qt)
        for (int c = 0; c < 2; ++c)
          tma_load_2d(smem + Smem2::q + qt * kTileBytes + c * kBoxBytes, &tm[0], q_full,
                      TILE_HEAD(qt) * kHeadDim + c * 64, TILE_R0(qt));
      Cursor cur = cursor_at2(prob, imax, t_begin);
      for (int it = 0; it < ntiles; ++it) {
        const CUtensorMap* km = &tm[1 + 2 * cur.seg];
        const CUtensorMap* vm = &tm[2 + 2 * cur.seg];
        const int ks = it % kKS2, vs = it % kVS2;
        if (it >= kKS2) mbar_wait(k_empty + ks, ((it / kKS2) - 1) & 1);
        mbar_expect_tx(k_full + ks, kKvTile2);
        for (int c = 0; c < 2; ++c)
          tma_load_2d(smem + Smem2::k + ks * kKvTile2 + c * kKvBox2, km, k_full + ks,
                      hk * kHeadDim + c * 64, cur.kt * kBN2);
        if (it >= kVS2) mbar_wait(v_empty + vs, ((it / kVS2) - 1) & 1);
        mbar_expect_tx(v_full + vs, kKvTile2);
        for (int c = 0; c < 2; ++c)
          tma_load_2d(smem + Smem2::v + vs * kKvTile2 + c * kKvBox2, vm, v_full + vs,
                      hk * kHeadDim + c * 64, cur.kt * kBN2);
        cursor_next2(prob, imax, cur);
      }
    }
  } else if (warp == kMmaWarp) {
    // ======================================================== MMA issuer
    if (elect_one()) {
      const uint32_t idesc_qk = idesc_bf16_f32(128, kBN2, 0, 0);  // Q, K both K-major
      const uint32_t idesc_pv = idesc_bf16_f32(128, 128, 0, 1);   // P (TMEM), V MN-major
      const uint32_t sq = smem_u32(smem + Smem2::q);
      const uint32_t sk = smem_u32(smem + Smem2::k);
      const uint32_t sv = smem_u32(smem + Smem2::v);
      // per (tile, buffer) use counters -> mbarrier parities
      uint32_t s_cnt[2][2] = {{0, 0}, {0, 0}}, p_cnt[2][2] = {{0, 0}, {0, 0}};
      bool o_acc[2] = {false, false};
      auto issue_qk = [&](int qt, int b, int ks) {
        const uint32_t d = tmem + (qt * 2 + b) * kBN2;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t qoff = (kk >> 2) * kBoxBytes + (kk & 3) * 32;
          const uint32_t koff = (kk >> 2) * kKvBox2 + (kk & 3) * 32;
          mma_ss(d, sdesc_sw128(sq + qt * kTileBytes + qoff, 16, 1024),
                 sdesc_sw128(sk + ks * kKvTile2 + koff, 16, 1024), idesc_qk, kk > 0 ? 1u : 0u);
        }
        tc_commit(s_full + qt * 2 + b);
        ++s_cnt[qt][b];
      };
      auto issue_pv = [&](int qt, int b, int vs) {
        const uint32_t d = tmem + 256 + qt * 128;
        const uint32_t a = tmem + (qt * 2 + b) * kBN2;
#pragma unroll
        for (int kk = 0; kk < kBN2 / 16; ++kk)
          mma_ts(d, a + kk * 8, sdesc_sw128(sv + vs * kKvTile2 + kk * 2048, kKvBox2, 1024), idesc_pv,
                 (o_acc[qt] || kk > 0) ? 1u : 0u);
        o_acc[qt] = true;
        tc_commit(o_full + qt);
      };
      auto modes_at = [&](const Cursor& c, int (&m)[2]) {
        for (int qt = 0; qt < 2; ++qt) m[qt] = tile_mode2(prob.seg[c.seg], c.kt, TILE_R0(qt), nq);
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      // prologue: QK of tiles 0 and 1 into buffers 0 and 1
      Cursor cq = cursor_at2(prob, imax, t_begin);  // cursor of the next QK tile
      for (int it = 0; it < 2 && it < ntiles; ++it) {
        int m[2];
        modes_at(cq, m);
        const int ks = it % kKS2;
        mbar_wait(k_full + ks, (it / kKS2) & 1);
        tc_fence_after();
        for (int qt = 0; qt < 2; ++qt)
          if (m[qt] != kSkip) issue_qk(qt, it & 1, ks);
        tc_commit(k_empty + ks);
        cursor_next2(prob, imax, cq);
      }
      Cursor cp = cursor_at2(prob, imax, t_begin);  // cursor of the PV tile
      for (int it = 0; it < ntiles; ++it) {
        const int b = it & 1, vs = it % kVS2;
        int m[2], mn[2] = {kSkip, kSkip};
        modes_at(cp, m);
        const bool has_next = it + 2 < ntiles;
        const int ksn = (it + 2) % kKS2;
        if (has_next) modes_at(cq, mn);
        mbar_wait(v_full + vs, (it / kVS2) & 1);
        bool k_ready = false;
        for (int qt = 0; qt < 2; ++qt) {
          if (m[qt] != kSkip) {
            mbar_wait(p_full + qt * 2 + b, p_cnt[qt][b] & 1);
            ++p_cnt[qt][b];
            tc_fence_after();
            issue_pv(qt, b, vs);
          }
          if (qt == 1) tc_commit(v_empty + vs);
          // QK_t(it+2) into the buffer PV_t(it) just drained (in-order tensor pipe)
          if (has_next && mn[qt] != kSkip) {
            if (!k_ready) {
              mbar_wait(k_full + ksn, ((it + 2) / kKS2) & 1);
              tc_fence_after();
              k_ready = true;
            }
            issue_qk(qt, b, ksn);
          }
        }
        if (has_next) {
          tc_commit(k_empty + ksn);
          cursor_next2(prob, imax, cq);
        }
        cursor_next2(prob, imax, cp);
      }
      tc_commit(o_done);
    }
  } else if (warp < kProducerWarp) {
    // ======================================================== softmax warpgroups
    const int qt = warp >> 2;
    const int quad = warp & 3;
    const int row = TILE_R0(qt) + quad * 32 + lane;
    const int qhead = TILE_HEAD(qt);
    const uint32_t t_lane = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t tO = tmem + t_lane + 256 + qt * 128;
    const float sl2 = P.scale_log2;
    const float2 sl2v = make_float2(sl2, sl2);
    float m_ref = -INFINITY;
    float l = 0.f;
    uint32_t cnt = 0;                 // PV_t issued so far (o_full parity)
    uint32_t bcnt[2] = {0, 0};        // uses of S buffer b (s_full parity)
    Cursor cur = cursor_at2(prob, imax, t_begin);
    uint32_t sr[2][32];
    uint32_t pk[2][16];
    for (int it = 0; it < ntiles; ++it, cursor_next2(prob, imax, cur)) {
      const AttnSeg sg = prob.seg[cur.seg];
      const int mode = tile_mode2(sg, cur.kt, TILE_R0(qt), nq);
      if (mode == kSkip) continue;
      const int b = it & 1;
      const uint32_t tS = tmem + t_lane + (qt * 2 + b) * kBN2;
      mbar_wait(s_full + qt * 2 + b, bcnt[b] & 1);
      ++bcnt[b];
      tc_fence_after();
      auto load_s = [&]() {
        tmem_ld32(tS, sr[0]);
        tmem_ld32(tS + 32, sr[1]);
        tmem_wait_ld();
      };
      auto chunk_max = [&](int c, float (&mxp)[8]) {
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const int t = (j / 2) & 7;
          mxp[t] = fmaxf(mxp[t], fmaxf(__uint_as_float(sr[c][j]), __uint_as_float(sr[c][j + 1])));
        }
      };
      auto chunk_exp = [&](int c, float2 negm, bool emu) {  // in place: sr[c] := p
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 x2 = __ffma2_rn(
              make_float2(__uint_as_float(sr[c][2 * j]), __uint_as_float(sr[c][2 * j + 1])), sl2v, negm);
          float2 p2;
          if (kEmu > 0 && emu && emu_slot(j, kEmu))
            p2 = exp2_poly2(x2);
          else
            p2 = make_float2(fast_exp2(x2.x), fast_exp2(x2.y));  // -inf -> 0
          sr[c][2 * j] = __float_as_uint(p2.x);
          sr[c][2 * j + 1] = __float_as_uint(p2.y);
        }
      };
      auto chunk_pack = [&](int c, float2 (&sacc)[4]) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 p2 = make_float2(__uint_as_float(sr[c][2 * j]), __uint_as_float(sr[c][2 * j + 1]));
          sacc[j & 3] = __fadd2_rn(sacc[j & 3], p2);
          __nv_bfloat162 bb = __floats2bfloat162_rn(p2.x, p2.y);
          pk[c][j] = *reinterpret_cast<uint32_t*>(&bb);
        }
      };
      auto exp_pack_all = [&](float2 negm, bool emu, float2 (&sacc)[4]) {
        chunk_exp(0, negm, emu);
        chunk_exp(1, negm, emu);
        chunk_pack(0, sacc);
        chunk_pack(1, sacc);
      };
      float alpha = 1.f;
      bool rescale = false;
      float mxp[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) mxp[t] = -INFINITY;
      float2 sacc[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) sacc[t] = make_float2(0.f, 0.f);
      bool done = false;
      load_s();
      if (mode == kFull && m_ref != -INFINITY) {
        const float2 negm = make_float2(-m_ref, -m_ref);
        chunk_max(0, mxp);
        chunk_max(1, mxp);
        exp_pack_all(negm, true, sacc);
        const float mx = fmaxf(fmaxf(fmaxf(mxp[0], mxp[1]), fmaxf(mxp[2], mxp[3])),
                               fmaxf(fmaxf(mxp[4], mxp[5]), fmaxf(mxp[6], mxp[7])));
        done = !(mx * sl2 > m_ref + 8.f);
        if (!done) {
#pragma unroll
          for (int t = 0; t < 8; ++t) mxp[t] = -INFINITY;
#pragma unroll
          for (int t = 0; t < 4; ++t) sacc[t] = make_float2(0.f, 0.f);
          load_s();
        }
      } else if (mode == kPart) {
        const int k0 = cur.kt * kBN2;
        int lim = sg.len - k0;
        if (sg.causal) lim = min(lim, row - k0 + 1);
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c * 32 + j >= lim) sr[c][j] = __float_as_uint(-INFINITY);
      }
      if (!done) {
        chunk_max(0, mxp);
        chunk_max(1, mxp);
        const float mx = fmaxf(fmaxf(fmaxf(mxp[0], mxp[1]), fmaxf(mxp[2], mxp[3])),
                               fmaxf(fmaxf(mxp[4], mxp[5]), fmaxf(mxp[6], mxp[7])));
        const float m_new = fmaxf(m_ref, mx * sl2);
        if (m_new > m_ref + 8.f) {
          alpha = exp2f(m_ref - m_new);
          m_ref = m_new;
          rescale = true;
        }
        const float m_use = (m_ref == -INFINITY) ? 0.f : m_ref;
        exp_pack_all(make_float2(-m_use, -m_use), mode == kFull, sacc);
      }
      tmem_st16(tS, pk[0]);
      tmem_st16(tS + 16, pk[1]);
      const float2 sum2 = __fadd2_rn(__fadd2_rn(sacc[0], sacc[1]), __fadd2_rn(sacc[2], sacc[3]));
      l = l * alpha + (sum2.x + sum2.y);
      if (rescale && cnt > 0) {
        mbar_wait(o_full + qt, (cnt - 1) & 1);  // PV_t of the previous tile has landed
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
      mbar_arrive(p_full + qt * 2 + b);
      ++cnt;
    }
    // ---- epilogue: O / l, lse.  With S double-buffered, PV(n-1) and PV(n) may both be in
    // flight here, which a parity wait on o_full cannot disambiguate: wait for the one-shot
    // barrier the MMA warp commits after its last instruction instead.
    mbar_wait(o_done, 0);
    tc_fence_after();
    const bool valid_row = row < nq;
    const float inv = (l > 0.f) ? 1.f / l : 0.f;
    const long long obase = static_cast<long long>(split) * prob.split_stride_out +
                            static_cast<long long>(row) * prob.ldo + qhead * kHeadDim;
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
                                 __uint_as_float(o[4 * j + 2]) * inv, __uint_as_float(o[4 * j + 3]) * inv);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(prob.out) + obase + 32 * c);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              __nv_bfloat162 bb = __floats2bfloat162_rn(__uint_as_float(o[8 * j + 2 * e]) * inv,
                                                        __uint_as_float(o[8 * j + 2 * e + 1]) * inv);
              w[e] = *reinterpret_cast<uint32_t*>(&bb);
            }
            dst[j] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
    }
    if (valid_row && prob.lse) {
      const float lse = (l > 0.f) ? (m_ref + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
      prob.lse[static_cast<long long>(split) * prob.split_stride_lse +
               static_cast<long long>(row) * prob.ld_lse + qhead] = lse;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc(tmem, kTmemCols);
#undef TILE_R0
#undef TILE_HEAD
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
               std::string* err, int box_rows = 128) {
  auto enc = tensor_map_encoder();
  if (!enc) {
    if (err) *err = "cuTensorMapEncodeTiled unavailable";
    return false;
  }
  if (rows < 1) rows = 1;  // empty segments are never loaded
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
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

bool make_tmap_bf16(CUtensorMap* m, const void* base, long long rows, long long cols, long long ld,
                    int box_rows, std::string* err) {
  return make_tmap(m, base, rows, cols, ld, err, box_rows);
}

std::atomic<int> g_attn_variant{-1};  // -1: SPAVA_ATTN_VARIANT / default

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
  // kernel variants (SPAVA_ATTN_VARIANT): family 0 = ping-pong (2 Q tiles per CTA, 320
  // threads), family 1 = one Q tile per CTA with double-buffered S (192 threads).
  using KFn = void (*)(AttnParams);
  struct Var { KFn fn; uint32_t smem; int threads; int family; };
  static const Var variants[] = {
      {attn_fwd_kernel<0, 2, false, true, false>, Smem<2>::bytes, kThreads, 0},  // 0 production
      {attn_fwd1_kernel<0, true>, Smem1::bytes, kThreads1, 1},            // 1 single tile, S x2
      {attn_fwd_kernel<0, 2, true, true>, Smem<2>::bytes, kThreads, 0},   // 2 14 + cycle counters
      {attn_fwd1_kernel<4, true>, Smem1::bytes, kThreads1, 1},            // 3 1 + 25% FMA exp2
      {attn_fwd_kernel<4, 2, false, true>, Smem<2>::bytes, kThreads, 0},  // 4 14 + 25% FMA exp2
      {attn_fwd1_kernel<2, true>, Smem1::bytes, kThreads1, 1},            // 5 1 + 12.5% FMA exp2
      {attn_fwd_kernel<0, 2>, Smem<2>::bytes, kThreads, 0},               // 6 14 without the
                                                                          //   one-chunk-behind pack
      {attn_fwd2_kernel<0>, Smem2::bytes, kThreads, 2},                   // 7 64-key tiles, S x2
      {attn_fwd2_kernel<2>, Smem2::bytes, kThreads, 2},                   // 8 7 + 25% FMA exp2
      {attn_fwd2_kernel<1>, Smem2::bytes, kThreads, 2},                   // 9 7 + 12.5% FMA exp2
      {attn_fwd3_kernel<0>, Smem3::bytes, kThreads3, 1},                  // 10 1 + column-split softmax
      {attn_fwd3_kernel<4>, Smem3::bytes, kThreads3, 1},                  // 11 10 + 25% FMA exp2
      {attn_fwd4_kernel<0>, Smem<2>::bytes, kThreads, 0},                 // 12 0 + split QK / P halves
      {attn_fwd4_kernel<4>, Smem<2>::bytes, kThreads, 0},                 // 13 12 + 25% FMA exp2
      {attn_fwd_kernel<0, 2, false, true, true>, Smem<2>::bytes, kThreads, 0}};   // 14 0 + speculative
                                                                                  //  stale-max pass
  constexpr int kNumVar = sizeof(variants) / sizeof(variants[0]);
  static const int env_sel = [] {
    const char* e = getenv("SPAVA_ATTN_VARIANT");
    const int v = e ? atoi(e) : 0;
    return (v >= 0 && v < kNumVar) ? v : 0;
  }();
  const int forced = g_attn_variant.load();
  const int vsel = (forced >= 0 && forced < kNumVar) ? forced : env_sel;
  const Var& var = variants[vsel];
  const int rows_per_cta = var.family == 1 ? kBlockM : kTilesPerCta * kBlockM;
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
    p.head_pair = (var.family != 1 && v.nq <= kBlockM && (hq / hkv) % 2 == 0) ? 1 : 0;
    p.units = p.head_pair ? 1 : (v.nq + rows_per_cta - 1) / rows_per_cta;
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
      const int kv_box = var.family == 2 ? kBN2 : kBlockN;
      if (!make_tmap(&P.tmap[np][1 + 2 * s], v.seg[s].k, v.seg[s].len,
                     static_cast<long long>(hkv) * dh, v.seg[s].ld, err, kv_box) ||
          !make_tmap(&P.tmap[np][2 + 2 * s], v.seg[s].v, v.seg[s].len,
                     static_cast<long long>(hkv) * dh, v.seg[s].ld, err, kv_box))
        return cudaErrorInvalidValue;
    }
    work += p.units * (p.head_pair ? hq / 2 : hq) * p.splits;
    ++np;
  }
  P.nprob = np;
  P.total_work = work;
  if (work == 0) return cudaSuccess;
  static bool attr_set[kNumVar] = {};
  const KFn fn = var.fn;
  const uint32_t smem_bytes = var.smem;
  if (!attr_set[vsel]) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem_bytes));
    if (e != cudaSuccess) return e;
    attr_set[vsel] = true;
  }
  fn<<<work, var.threads, smem_bytes, stream>>>(P);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && err) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, fn);
    *err = std::string("attention launch: ") + cudaGetErrorString(e) + " (regs " +
           std::to_string(fa.numRegs) + ", maxThreads " + std::to_string(fa.maxThreadsPerBlock) +
           ", static smem " + std::to_string(fa.sharedSizeBytes) + ", local " +
           std::to_string(fa.localSizeBytes) + ", params " + std::to_string(sizeof(AttnParams)) + ")";
  }
  return e;
}

int attn_set_variant(int v) {
  if (v < -1 || v > 14) return -1;
  g_attn_variant.store(v);
  return 0;
}

// dev: read and reset the cycle counters of the profiling variant
void attn_prof_read(unsigned long long* out16) {
  cudaMemcpyFromSymbol(out16, g_attn_prof, sizeof(unsigned long long) * 16);
  static const unsigned long long z[16] = {};
  cudaMemcpyToSymbol(g_attn_prof, z, sizeof(z));
}

}  // namespace spava
