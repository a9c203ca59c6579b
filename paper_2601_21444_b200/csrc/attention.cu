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
#include <type_traits>

#include "fabric_dev.cuh"
#include "ptx.cuh"
#include "score_fast_dev.cuh"
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

// the first 16 words of a 32-word register row (P packed in place over S)
__device__ __forceinline__ void tmem_st16_lo(uint32_t taddr, const uint32_t (&pk)[32]) {
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

// kPParts: P of a tile is committed to TMEM in kPParts key ranges, each signalled on its own
// mbarrier, and the MMA warp issues the PV K-steps of a range as soon as it is in, so the
// tensor pipe overlaps the tail of the softmax of the same tile (the per-tile loop
// softmax -> PV -> QK shortens by (1 - 1/kPParts) of a PV).
// kRegs > 0: 384 threads (3 warpgroups); the producer/MMA warpgroup gives registers back
// (setmaxnreg.dec to 56) and the two softmax warpgroups take kRegs each (setmaxnreg.inc), so
// a softmax thread holds its S row, packed P and a deeper software pipeline without spills.
// kSeq: the exp phases of the two softmax warpgroups strictly alternate (named barriers 1/2),
// so each runs with the SM's MUFU to itself and the two stay in anti-phase with the MMAs.
// kLd2: S is read from TMEM in two halves, the max of the first overlapping the second load.
// kWG = 2: FOUR softmax warpgroups (576 threads), two per Q tile, each taking 64 of the 128
// key columns of every S tile: per-tile softmax latency halves (64 exps per thread), the two
// halves exchange their row maxima through shared memory (named barrier per Q tile) and
// keep partial row sums that are added in the epilogue; each half commits its two P ranges.
template <int kEmu, int KS, bool kProf = false, bool kPipe = false, bool kSpec = true, int kPParts = 1,
          int kRegs = 0, bool kSeq = false, bool kLd2 = false, int kWG = 1, bool kStats = true,
          bool kHalfQK = false>
__global__ void __launch_bounds__(kWG == 2 ? 576 : kRegs > 0 ? 384 : kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ AttnParams P) {
  static_assert(!kHalfQK || (kWG == 1 && !kSpec && !kLd2 && kPParts == 4),
                "split QK: production softmax path only");
  static_assert(kPParts == 1 || (kPipe && !kSpec && (kPParts == 2 || kPParts == 4)),
                "split P needs the max-first pipelined softmax");
  static_assert(kWG == 1 || (kPipe && !kSpec && kPParts == 4 && kRegs == 0 && !kSeq && !kLd2),
                "column-split softmax: max-first pipelined body with P in 4 ranges only");
  constexpr int kProdW = kWG == 2 ? 16 : kProducerWarp;
  constexpr int kMmaW = kProdW + 1;
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
  uint64_t* p_full = s_full + 2;              // [2][4] P_t key range written (O_t corrected)
  uint64_t* o_full = p_full + 8;              // [2] PV_t complete
  uint64_t* s_loaded = o_full + 2;            // [2] kHalfQK: S_t(j) is in the softmax registers
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_loaded + 2);

  // trailing CTAs of a stage launch (peer fabric): the receive-side query merge
  if constexpr (kWG == 1) {
  if (P.job.ctas > 0 && static_cast<int>(blockIdx.x) >= P.total_work &&
      static_cast<int>(blockIdx.x) < P.total_work + P.job.ctas) {
    merge_job(P.job, static_cast<int>(blockIdx.x) - P.total_work, reinterpret_cast<float*>(smem));
    return;
  }
  // trailing CTAs of a query launch (fast scoring fused, N1): the column-sum pass of the
  // tensor-core scorer over (block, 128-key tile), once this launch's attention CTAs have
  // produced the lo / hi row statistics (K tiles of the blocks are L2-resident by then)
  if (P.sj.ctas > 0 && static_cast<int>(blockIdx.x) >= P.total_work + P.job.ctas) {
    const int t = static_cast<int>(blockIdx.x) - P.total_work - P.job.ctas;
    score_fast_cta<1>(P.sj.fa, t % P.sj.fa.ntiles, t / P.sj.fa.ntiles, smem);
    return;
  }
  }  // kWG == 1 (the launcher keeps trailing jobs on the production kernel)
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

  if (warp == kProdW && elect_one()) {
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
      for (int pp = 0; pp < kPParts; ++pp) mbar_init(p_full + 4 * t + pp, 128);
      mbar_init(o_full + t, 1);
      mbar_init(s_loaded + t, 128);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tm[0]);
    for (int s = 0; s < prob.nseg; ++s) {
      tma_prefetch_desc(&tm[1 + 2 * s]);
      tma_prefetch_desc(&tm[2 + 2 * s]);
    }
  }
  if (warp == kMmaW) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Role branches: the register budget changes at the top of each warpgroup's branch and the
  // branches only rejoin at the teardown, so ptxas allocates each role within its budget.
  if (warp >= kProdW) {
  if constexpr (kRegs > 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
  if (warp == kProdW) {
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
  } else if (warp == kMmaW) {
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
      // kHalfQK: S_t(j+1) as two N = 64 halves.  Keys 64..127 land in S columns 64..127,
      // which hold no P, so that half is issued as soon as the softmax has S_t(j) in
      // registers (s_loaded) and runs under its exps; only keys 0..63 (columns 0..63, where
      // P_t(j) sits) still follow PV_t(j) -- the chain after the last P range shrinks from
      // 1.25 to 0.75 MMA times.
      const uint32_t idesc_qk64 = idesc_bf16_f32(128, 64, 0, 0);
      auto issue_qk_half = [&](int qt, int stage, int h) {
        const uint32_t d = tmem + qt * 128 + 64 * h;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t koff = (kk >> 2) * kBoxBytes + (kk & 3) * 32;
          const uint64_t a = sdesc_sw128(sq + qt * kTileBytes + koff, 16, 1024);
          const uint64_t b = sdesc_sw128(sk + stage * kTileBytes + koff + h * 8192u, 16, 1024);
          mma_ss(d, a, b, idesc_qk64, kk > 0 ? 1u : 0u);
        }
      };
      // PV K-steps [kk0, kk0 + n) (16 keys each; P of K-step kk at S columns 8kk..8kk+7)
      auto issue_pv = [&](int qt, int stage, bool acc, int kk0, int n) {
        const uint32_t d = tmem + 256 + qt * 128;
        const uint32_t a = tmem + qt * 128;
#pragma unroll
        for (int k = 0; k < n; ++k) {
          const int kk = kk0 + k;
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
          if constexpr (kHalfQK) {
            if (nmode[qt] != kSkip) {
              if (mode[qt] != kSkip) {  // S_qt(it) exists: wait until the softmax holds it
                mbar_wait(s_loaded + qt, p_cnt[qt] & 1);
                tc_fence_after();
              }
              issue_qk_half(qt, kn, 1);
            }
          }
          if (mode[qt] != kSkip) {
#pragma unroll
            for (int pp = 0; pp < kPParts; ++pp) {
              const long long tw = PROF_NOW();
              mbar_wait(p_full + 4 * qt + pp, p_cnt[qt] & 1);
              if (kProf) pr[2] += PROF_NOW() - tw;
              tc_fence_after();
              issue_pv(qt, vs, o_acc[qt], pp * (8 / kPParts), 8 / kPParts);
            }
            o_acc[qt] = true;
            ++p_cnt[qt];
            tc_commit(o_full + qt);
          }
          if (qt == 1) tc_commit(v_empty + vs);
          if (nmode[qt] != kSkip) {
            if constexpr (kHalfQK)
              issue_qk_half(qt, kn, 0);
            else
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
  }
  } else {
    if constexpr (kRegs > 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegs));
    // ======================================================== softmax warpgroups
    if constexpr (kWG == 2) {
    // ---- column-split softmax: warpgroup g takes Q tile g & 1, key columns [64 h, 64 h + 64)
    // of every S tile (h = g >> 1); TMEM lanes are per warp-in-warpgroup, so both halves of a
    // Q tile address the same 128 lanes.
    const int g = warp >> 2;
    const int qt = g & 1;
    const int half = g >> 1;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const int row = TILE_R0(qt) + r;
    const int qhead = TILE_HEAD(qt);
    const uint32_t t_lane = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t tS = tmem + t_lane + qt * 128;
    const uint32_t tO = tmem + t_lane + 256 + qt * 128 + 64 * half;
    float* xmax = reinterpret_cast<float*>(smem + SL::total);  // [2 parity][2 qt][2 half][128]
    float* xl = xmax + 1024;  // [2 qt][2 half][3][128]  (10 KB in all, Smem<2>::bytes + 10240)
    const float sl2 = P.scale_log2;
    const float2 sl2v = make_float2(sl2, sl2);
    float m_ref = -INFINITY;
    const bool seg_stats = prob.seg_lse2 != nullptr;
    float l_seg[2] = {0.f, 0.f};
    float l = 0.f;
    uint32_t cnt = 0;
    Cursor cur = cursor_at(prob, imax, t_begin);
    for (int it = 0; it < ntiles; ++it, cursor_next(prob, imax, cur)) {
      const AttnSeg sg = prob.seg[cur.seg];
      const int mode = tile_mode(sg, cur.kt, TILE_R0(qt), nq);
      if (mode == kSkip) continue;  // same decision in both halves (it depends on rows only)
      mbar_wait(s_full + qt, cnt & 1);
      tc_fence_after();
      uint32_t sr[2][32];
      tmem_ld32(tS + 64 * half, sr[0]);
      tmem_ld32(tS + 64 * half + 32, sr[1]);
      tmem_wait_ld();
      if (mode == kPart) {
        const int k0 = cur.kt * kBlockN + 64 * half;
        int lim = sg.len - k0;
        if (sg.causal) lim = min(lim, row - k0 + 1);
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (c * 32 + j >= lim) sr[c][j] = __float_as_uint(-INFINITY);
      }
      float mxp[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) mxp[t] = -INFINITY;
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int j = 0; j < 32; j += 2)
          mxp[(j / 2) & 7] = fmaxf(mxp[(j / 2) & 7], fmaxf(__uint_as_float(sr[c][j]), __uint_as_float(sr[c][j + 1])));
      const float mxl = fmaxf(fmaxf(fmaxf(mxp[0], mxp[1]), fmaxf(mxp[2], mxp[3])),
                              fmaxf(fmaxf(mxp[4], mxp[5]), fmaxf(mxp[6], mxp[7])));
      // row max of the whole tile: exchange with the other half (slot by tile parity: the
      // partner reads slot j before either half can reach tile j + 2's write of it).  The
      // barrier also orders this half's S loads before the other half's P stores, which
      // land in S columns [32 h', 32 h' + 32) -- half 0's S columns 32..63 for h' = 1.
      float* xm = xmax + ((cnt & 1) * 2 + qt) * 2 * 128;
      xm[half * 128 + r] = mxl;
      named_bar_sync(1 + qt, 256);
      const float mx = fmaxf(mxl, xm[(half ^ 1) * 128 + r]);
      const float m_new = fmaxf(m_ref, mx * sl2);
      float alpha = 1.f;
      const bool rescale = m_new > m_ref + 8.f;  // identical in both halves
      if (rescale) {
        alpha = exp2f(m_ref - m_new);
        m_ref = m_new;
      }
      if (rescale && cnt > 0) {
        // each half corrects its 64 O columns; both are done before either releases a P
        // range (the PV K-steps write all 128 columns)
        mbar_wait(o_full + qt, (cnt - 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
          uint32_t o[8];
          tmem_ld8(tO + 8 * c, o);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
          tmem_st8(tO + 8 * c, o);
        }
        tmem_wait_st();
        tc_fence_before();
        named_bar_sync(1 + qt, 256);
      }
      const float m_use = (m_ref == -INFINITY) ? 0.f : m_ref;
      const float2 negm = make_float2(-m_use, -m_use);
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 x2 = __ffma2_rn(
              make_float2(__uint_as_float(sr[c][2 * j]), __uint_as_float(sr[c][2 * j + 1])), sl2v, negm);
          float2 p2;
          if (kEmu > 0 && mode == kFull && emu_slot(j, kEmu))
            p2 = exp2_poly2(x2);
          else
            p2 = make_float2(fast_exp2(x2.x), fast_exp2(x2.y));  // -inf -> 0
          sr[c][2 * j] = __float_as_uint(p2.x);
          sr[c][2 * j + 1] = __float_as_uint(p2.y);
        }
      float2 sacc[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) sacc[t] = make_float2(0.f, 0.f);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        // pack in place (word j <- keys 2j, 2j+1; reads never hit an already packed word)
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 p2 = make_float2(__uint_as_float(sr[c][2 * j]), __uint_as_float(sr[c][2 * j + 1]));
          sacc[j & 3] = __fadd2_rn(sacc[j & 3], p2);
          __nv_bfloat162 b = __floats2bfloat162_rn(p2.x, p2.y);
          sr[c][j] = *reinterpret_cast<uint32_t*>(&b);
        }
        tmem_st16_lo(tS + 32 * half + 16 * c, sr[c]);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(p_full + 4 * qt + 2 * half + c);
      }
      const float2 sum2 = __fadd2_rn(__fadd2_rn(sacc[0], sacc[1]), __fadd2_rn(sacc[2], sacc[3]));
      l = l * alpha + (sum2.x + sum2.y);
      if (seg_stats) {
        l_seg[0] *= alpha;
        l_seg[1] *= alpha;
        if (cur.seg == prob.stat_seg[0]) l_seg[0] += sum2.x + sum2.y;
        if (cur.seg == prob.stat_seg[1]) l_seg[1] += sum2.x + sum2.y;
      }
      ++cnt;
    }
    // ---- epilogue: row sums of both halves (half 0 + half 1), O / l of this half's columns
    if (cnt > 0) {
      mbar_wait(o_full + qt, (cnt - 1) & 1);
      tc_fence_after();
    }
    float* xq = xl + qt * 2 * 3 * 128;
    xq[(half * 3 + 0) * 128 + r] = l;
    xq[(half * 3 + 1) * 128 + r] = l_seg[0];
    xq[(half * 3 + 2) * 128 + r] = l_seg[1];
    named_bar_sync(1 + qt, 256);
    const float lt = xq[0 * 128 + r] + xq[3 * 128 + r];
    const float ls0 = xq[1 * 128 + r] + xq[4 * 128 + r];
    const float ls1 = xq[2 * 128 + r] + xq[5 * 128 + r];
    const bool valid_row = row < nq;
    const float inv = (lt > 0.f) ? 1.f / lt : 0.f;
    const long long obase = static_cast<long long>(split) * prob.split_stride_out +
                            static_cast<long long>(row) * prob.ldo + qhead * kHeadDim + 64 * half;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
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
              __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(o[8 * j + 2 * e]) * inv,
                                                       __uint_as_float(o[8 * j + 2 * e + 1]) * inv);
              w[e] = *reinterpret_cast<uint32_t*>(&b);
            }
            dst[j] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
    }
    if (valid_row && half == 0 && prob.lse) {
      const float lse = (lt > 0.f) ? (m_ref + __log2f(lt)) * 0.69314718055994530942f : -INFINITY;
      prob.lse[static_cast<long long>(split) * prob.split_stride_lse +
               static_cast<long long>(row) * prob.ld_lse + qhead] = lse;
    }
    if (valid_row && half == 0 && seg_stats) {
      const float lsv[2] = {ls0, ls1};
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2)
        if (prob.stat_seg[s2] >= 0)
          prob.seg_lse2[((static_cast<long long>(s2) * prob.splits + split) * nq + row) * P.hq + qhead] =
              lsv[s2] > 0.f ? m_ref + __log2f(lsv[s2]) : -INFINITY;
    }
    } else {
    const int qt = warp >> 2;
    const int quad = warp & 3;
    const int row = TILE_R0(qt) + quad * 32 + lane;  // problem-local query row
    const int qhead = TILE_HEAD(qt);
    const uint32_t t_lane = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t tS = tmem + t_lane + qt * 128;
    const uint32_t tO = tmem + t_lane + 256 + qt * 128;
    const float sl2 = P.scale_log2;
    float m_ref = -INFINITY;
    // fused fast scorer: sum of 2^(x - m_ref) over the keys of block lo / hi alone (same
    // reference max and lazy rescale as l), i.e. the scorer's per-row softmax statistics
    // (kStats = false: an instance without them -- two fewer live registers in the softmax
    // loop, which runs at the 168-register cap of 320 threads)
    const bool seg_stats = kStats && prob.seg_lse2 != nullptr;
    float l_seg[2] = {0.f, 0.f};
    float l = 0.f;
    uint32_t cnt = 0;
    // kSeq: tiles processed by this and by the other warpgroup (skipped tiles are the causal
    // tail, so the k-th processed tiles of both line up); tokens only for k < n_min.
    int n_ot = 0, n_min = 0;
    if constexpr (kSeq) {
      int n_me = 0;
      Cursor c2 = cursor_at(prob, imax, t_begin);
      for (int it = 0; it < ntiles; ++it, cursor_next(prob, imax, c2)) {
        n_me += tile_mode(prob.seg[c2.seg], c2.kt, TILE_R0(qt), nq) != kSkip;
        n_ot += tile_mode(prob.seg[c2.seg], c2.kt, TILE_R0(qt ^ 1), nq) != kSkip;
      }
      n_min = min(n_me, n_ot);
    }
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
      auto mask_chunk = [&](int c) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c * 32 + j >= lim) sr[c][j] = __float_as_uint(-INFINITY);
      };
      auto rescale_o = [&](float a) {
        mbar_wait(o_full + qt, (cnt - 1) & 1);  // PV_{cnt-1} has landed in O
        tc_fence_after();
        if constexpr (kPParts > 1) {  // the S row is still live: 8 columns at a time
#pragma unroll 1
          for (int c = 0; c < 16; ++c) {
            uint32_t o[8];
            tmem_ld8(tO + 8 * c, o);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 8; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * a);
            tmem_st8(tO + 8 * c, o);
          }
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            tmem_ld32(tO + 32 * c, o);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * a);
            tmem_st32(tO + 32 * c, o);
          }
        }
      };
      float mxp[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) mxp[t] = -INFINITY;
      float2 sacc[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) sacc[t] = make_float2(0.f, 0.f);
      bool done = false;
      if constexpr (kLd2) {
        static_assert(!kSpec, "kLd2 is a max-first path");
#pragma unroll
        for (int t = 0; t < 8; ++t) mxp[t] = -INFINITY;
        tmem_ld32(tS, sr[0]);
        tmem_ld32(tS + 32, sr[1]);
        tmem_wait_ld();
        tmem_ld32(tS + 64, sr[2]);
        tmem_ld32(tS + 96, sr[3]);
        if (mode == kPart) {
          mask_chunk(0);
          mask_chunk(1);
        }
        chunk_max(0, mxp);
        chunk_max(1, mxp);
        tmem_wait_ld();
        if (mode == kPart) {
          mask_chunk(2);
          mask_chunk(3);
        }
        chunk_max(2, mxp);
        chunk_max(3, mxp);
      } else {
        load_s();
        if constexpr (kHalfQK) {  // S columns 64..127 may now take the next tile's keys 64..127
          tc_fence_before();
          mbar_arrive(s_loaded + qt);
        }
      }
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
      } else if (!kLd2 && mode == kPart) {
#pragma unroll
        for (int c = 0; c < 4; ++c) mask_chunk(c);
      }
      if (kProf) pr[8] += PROF_NOW() - tw1;
      if (!done) {
        // max first, lazy rescale (keep a stale max while p <= 2^8), then exps
        if constexpr (!kLd2) {
#pragma unroll
          for (int t = 0; t < 8; ++t) mxp[t] = -INFINITY;
#pragma unroll
          for (int c = 0; c < 4; ++c) chunk_max(c, mxp);
        }
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
        if constexpr (kPParts > 1) {
          // O is corrected before any P range is released (PV_{cnt-1} already landed: it
          // was issued before the QK whose commit signalled s_full), then each key range
          // of P is stored and signalled as soon as it is packed.
          if (rescale && cnt > 0) rescale_o(alpha);
          constexpr int kCpp = 4 / kPParts;  // 32-key chunks per range
          const int k = static_cast<int>(cnt);
          if constexpr (kSeq) {  // wait for the other warpgroup's exp phase of the turn before
            if (qt == 0 ? (k >= 1 && k - 1 < n_min) : (k < n_min)) named_bar_sync(qt == 0 ? 2 : 1, 256);
          }
          const long long te0 = PROF_NOW();
          // the exp phase is instantiated twice when some exps go to the FMA pipe (kEmu):
          // fully visible tiles take the mixed MUFU / polynomial body, partial tiles the
          // MUFU-only one -- one uniform branch per tile, none inside the unrolled body
          auto exp_phase = [&](auto emu_tag) {
            constexpr bool kE = decltype(emu_tag)::value;
            chunk_exp_ip(0, negm, kE);
#pragma unroll
            for (int c = 1; c < 4; ++c) {
              chunk_exp_ip(c, negm, kE);
              if (kSeq && c == 3) {  // exps done: hand the MUFUs to the other warpgroup
                // warpgroup 0's turn k is awaited by warpgroup 1 iff k < n_min; warpgroup 1's
                // turn k by warpgroup 0 iff k < n_min and warpgroup 0 has a turn k + 1
                if (qt == 0 ? (k < n_min) : (k < n_min && k + 1 < n_ot)) named_bar_arrive(qt == 0 ? 1 : 2, 256);
              }
              chunk_pack(c - 1, sacc);
              tmem_st16(tS + 16 * (c - 1), pk[c - 1]);
              if (c % kCpp == 0) {
                const long long ts0 = PROF_NOW();
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(p_full + 4 * qt + c / kCpp - 1);
                if (kProf) pr[11] += PROF_NOW() - ts0;
              }
            }
            chunk_pack(3, sacc);
            tmem_st16(tS + 48, pk[3]);
          };
          if (kEmu > 0 && mode == kFull)
            exp_phase(std::true_type{});
          else
            exp_phase(std::false_type{});
          if (kProf) pr[10] += PROF_NOW() - te0;
        } else if constexpr (kPipe) {
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
      if constexpr (kPParts == 1) {
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_st16(tS + 16 * c, pk[c]);
      }
      sum2 = __fadd2_rn(__fadd2_rn(sacc[0], sacc[1]), __fadd2_rn(sacc[2], sacc[3]));
      const long long tp3 = PROF_NOW();
      l = l * alpha + (sum2.x + sum2.y);
      if (seg_stats) {
        l_seg[0] *= alpha;
        l_seg[1] *= alpha;
        if (cur.seg == prob.stat_seg[0]) l_seg[0] += sum2.x + sum2.y;
        if (cur.seg == prob.stat_seg[1]) l_seg[1] += sum2.x + sum2.y;
      }
      if (kPParts == 1 && rescale && cnt > 0) rescale_o(alpha);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(p_full + 4 * qt + kPParts - 1);
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
    if (valid_row && seg_stats) {
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2)
        if (prob.stat_seg[s2] >= 0)
          prob.seg_lse2[((static_cast<long long>(s2) * prob.splits + split) * nq + row) * P.hq + qhead] =
              l_seg[s2] > 0.f ? m_ref + __log2f(l_seg[s2]) : -INFINITY;
    }
    }  // kWG
  }

  if (P.sj.ctas > 0) __threadfence();  // seg_lse2 stores, before this CTA is counted
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (P.sj.ctas > 0) {
    // the last split CTA of each head group combines that group's per-split statistics into
    // lse2[blk][h][i]; the last group to finish releases the column-sum CTAs
    // (counter[g]: splits done of group g; counter[ngroups]: groups done)
    const AttnProb& q0 = P.prob[0];
    const int grp = (static_cast<int>(blockIdx.x) - q0.work_begin) / q0.splits;
    const int ngroups = P.total_work / q0.splits;
    __shared__ int last_sh;
    if (threadIdx.x == 0) {
      __threadfence();
      last_sh = atomicAdd(P.sj.counter + grp, 1u) == static_cast<unsigned>(q0.splits) - 1;
    }
    __syncthreads();
    if (last_sh) {
      __threadfence();
      const FastArgs& fa = P.sj.fa;
      const int nh = q0.head_pair ? 2 : 1;
      const int h0 = q0.head_pair ? 2 * grp : grp;
      for (int e = threadIdx.x; e < 2 * nh * fa.n_t; e += blockDim.x) {
        const int b2 = e / (nh * fa.n_t), h2 = h0 + (e / fa.n_t) % nh, i2 = e % fa.n_t;
        float* dst = fa.lse2 + (static_cast<long long>(b2) * fa.hq + h2) * fa.n_t + i2;
        if (q0.stat_seg[b2] < 0) {  // block without visible keys: every score is a pad (-inf)
          *dst = -INFINITY;
          continue;
        }
        const float* src = q0.seg_lse2 + (static_cast<long long>(b2) * q0.splits * q0.nq + i2) * fa.hq + h2;
        const long long sstride = static_cast<long long>(q0.nq) * fa.hq;
        float M = -INFINITY, S = 0.f;  // online log2-sum-exp over the splits
        for (int sp = 0; sp < q0.splits; sp += 8) {
          float v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = sp + u < q0.splits ? __ldcg(src + (sp + u) * sstride) : -INFINITY;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (v[u] == -INFINITY) continue;
            if (v[u] > M) {
              S = S * exp2f(M - v[u]) + 1.f;
              M = v[u];
            } else {
              S += exp2f(v[u] - M);
            }
          }
        }
        *dst = M + __log2f(S);  // -inf for a row without visible keys
      }
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) {
        atomicExch(P.sj.counter + grp, 0u);
        if (atomicAdd(P.sj.counter + ngroups, 1u) == static_cast<unsigned>(ngroups) - 1) {
          __threadfence();
          atomicExch(P.sj.counter + ngroups, 0u);
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(P.sj.ready), "r"(fa.epoch) : "memory");
        }
      }
    }
  }
  if (kProf && (warp == kMmaW || (warp < kProdW && lane == 0)))
    for (int i = 0; i < 14; ++i)
      if (pr[i]) atomicAdd(&g_attn_prof[i], static_cast<unsigned long long>(pr[i]));
  if (warp == kMmaW) tmem_dealloc(tmem, kTmemCols);
#undef TILE_R0
#undef TILE_HEAD
}

#ifdef SPAVA_DEV_VARIANTS
// ---------------------------------------------------------------------------------------
// CTA-pair form (2-SM tcgen05.mma.cta_group::2): a cluster of two CTAs computes two q-heads
// of one KV group over the same 256 rows, so both see the same segment / causal tile
// sequence.  The rank-0 CTA issues every MMA for the pair (M = 256: each CTA's own Q tile
// rows, D in each CTA's TMEM); the B operand is split along N -- each CTA loads and holds
// half of every K tile (64 keys) and half of every V tile (64 of the 128 dh columns) -- so
// K/V TMA traffic, smem footprint and the MMA's smem operand reads per SM are halved.
// Commits multicast to both CTAs; P readiness is counted on the rank-0 CTA's barriers by
// the softmax threads of both.  The softmax / epilogue code is the production kernel's.
constexpr uint32_t kHalfTile = kTileBytes / 2;  // 64 keys x 128 dh (K half) or 128 keys x 64 dh (V half)
template <int KS>
struct SmemP {
  static constexpr uint32_t q = 0;
  static constexpr uint32_t k = q + kTilesPerCta * kTileBytes;
  static constexpr uint32_t v = k + KS * kHalfTile;
  static constexpr uint32_t bar = v + KS * kHalfTile;
  static constexpr uint32_t total = bar + 256;
  static constexpr uint32_t bytes = total + 1024;
};

constexpr int kPairStages = 4;  // K / V half-tile ring depth of the pair kernel
template <int KS>
__global__ void __launch_bounds__(kThreads, 1) attn_pair_kernel(const __grid_constant__ AttnParams P) {
  constexpr int kPParts = 4;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  using SL = SmemP<KS>;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SL::bar);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;        // [KS]   counted on rank 0
  uint64_t* k_empty = k_full + KS;    // [KS]   both CTAs (multicast commit)
  uint64_t* v_full = k_empty + KS;    // [KS]   rank 0
  uint64_t* v_empty = v_full + KS;    // [KS]   both
  uint64_t* s_full = v_empty + KS;    // [2]    both
  uint64_t* p_full = s_full + 2;      // [2][4] rank 0, 256 arrivals (both CTAs' softmax)
  uint64_t* o_full = p_full + 8;      // [2]    both
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 2);
  static_assert((1 + 4 * KS + 12) * 8 + 4 <= 256, "barrier area");
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int warp = warp_id();
  const int lane = lane_id();

  // ---- decode the pair's work item: problem, 256-row unit (heaviest first), head group, split
  const int w = static_cast<int>(blockIdx.x >> 1);
  int pi = 0;
  while (pi + 1 < P.nprob && w >= P.prob[pi + 1].work_begin) ++pi;
  const AttnProb& prob = P.prob[pi];
  int local = w - prob.work_begin;
  const int split = local % prob.splits;
  local /= prob.splits;
  const int pair = prob.head_pair;  // nq <= 128: a CTA's two Q tiles are heads h, h+1
  const int ngroups = pair ? P.hq / 4 : P.hq / 2;
  const int g = local % ngroups;
  local /= ngroups;
  const int head = pair ? 4 * g + 2 * static_cast<int>(rank) : 2 * g + static_cast<int>(rank);
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
  const CUtensorMap* tm = P.tmap[pi];  // [0] Q, [1+2s] K (64-key boxes), [2+2s] V

  if (warp == kProducerWarp && elect_one()) {
    mbar_init(q_full, 1);
    for (int s = 0; s < KS; ++s) {
      mbar_init(k_full + s, 1);
      mbar_init(k_empty + s, 1);
      mbar_init(v_full + s, 1);
      mbar_init(v_empty + s, 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(s_full + t, 1);
      for (int pp = 0; pp < kPParts; ++pp) mbar_init(p_full + 4 * t + pp, 256);
      mbar_init(o_full + t, 1);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tm[0]);
    for (int s = 0; s < prob.nseg; ++s) {
      tma_prefetch_desc(&tm[1 + 2 * s]);
      tma_prefetch_desc(&tm[2 + 2 * s]);
    }
  }
  if (warp == kMmaWarp) tmem_alloc2(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers exist before any remote arrive / TMA signal
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kProducerWarp) {
    // ======================================================== TMA producer (both CTAs)
    if (elect_one()) {
      const bool has1 = TILE_R0(1) < nq;
      if (leader) mbar_expect_tx(q_full, 2u * (has1 ? 2u : 1u) * kTileBytes);
      for (int qt = 0; qt < (has1 ? 2 : 1); ++qt)
        for (int c = 0; c < 2; ++c)
          tma_load_2d_pair(smem + SL::q + qt * kTileBytes + c * kBoxBytes, &tm[0], q_full,
                           TILE_HEAD(qt) * kHeadDim + c * 64, TILE_R0(qt));
      Cursor cur = cursor_at(prob, imax, t_begin);
      for (int it = 0; it < ntiles; ++it) {
        const CUtensorMap* km = &tm[1 + 2 * cur.seg];
        const CUtensorMap* vm = &tm[2 + 2 * cur.seg];
        const int st = it % KS;
        if (it >= KS) mbar_wait(k_empty + st, ((it / KS) - 1) & 1);
        if (leader) mbar_expect_tx(k_full + st, kTileBytes);  // both halves
        for (int c = 0; c < 2; ++c)  // keys [kt*128 + rank*64, +64), dh half c
          tma_load_2d_pair(smem + SL::k + st * kHalfTile + c * (kBoxBytes / 2), km, k_full + st,
                           hk * kHeadDim + c * 64, cur.kt * kBlockN + static_cast<int>(rank) * 64);
        if (it >= KS) mbar_wait(v_empty + st, ((it / KS) - 1) & 1);
        if (leader) mbar_expect_tx(v_full + st, kTileBytes);
        tma_load_2d_pair(smem + SL::v + st * kHalfTile, vm, v_full + st,
                         hk * kHeadDim + static_cast<int>(rank) * 64, cur.kt * kBlockN);  // dh half `rank`
        cursor_next(prob, imax, cur);
      }
    }
  } else if (warp == kMmaWarp) {
    // ======================================================== MMA issuer (rank 0 for the pair)
    if (leader && elect_one()) {
      const uint32_t idesc_qk = idesc_bf16_f32(256, 128, 0, 0);
      const uint32_t idesc_pv = idesc_bf16_f32(256, 128, 0, 1);
      const uint32_t sq = smem_u32(smem + SL::q);
      const uint32_t sk = smem_u32(smem + SL::k);
      const uint32_t sv = smem_u32(smem + SL::v);
      auto issue_qk = [&](int qt, int stage) {
        const uint32_t d = tmem + qt * 128;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t a = sdesc_sw128(sq + qt * kTileBytes + (kk >> 2) * kBoxBytes + (kk & 3) * 32, 16, 1024);
          const uint64_t b = sdesc_sw128(sk + stage * kHalfTile + (kk >> 2) * (kBoxBytes / 2) + (kk & 3) * 32, 16, 1024);
          mma_ss2(d, a, b, idesc_qk, kk > 0 ? 1u : 0u);
        }
      };
      auto issue_pv = [&](int qt, int stage, bool acc, int kk0, int n) {
        const uint32_t d = tmem + 256 + qt * 128;
        const uint32_t a = tmem + qt * 128;
#pragma unroll
        for (int k = 0; k < n; ++k) {
          const int kk = kk0 + k;
          const uint64_t b = sdesc_sw128(sv + stage * kHalfTile + kk * 2048, kHalfTile, 1024);
          mma_ts2(d, a + kk * 8, b, idesc_pv, (acc || kk > 0) ? 1u : 0u);
        }
      };
      mbar_wait(q_full, 0);
      tc_fence_after();
      Cursor cur = cursor_at(prob, imax, t_begin);
      int mode[2] = {kSkip, kSkip};
      uint32_t p_cnt[2] = {0, 0};
      bool o_acc[2] = {false, false};
      if (ntiles > 0) {
        for (int qt = 0; qt < 2; ++qt) mode[qt] = tile_mode(prob.seg[cur.seg], cur.kt, TILE_R0(qt), nq);
        mbar_wait(k_full + 0, 0);
        tc_fence_after();
        for (int qt = 0; qt < 2; ++qt)
          if (mode[qt] != kSkip) {
            issue_qk(qt, 0);
            tc_commit_pair(s_full + qt);
          }
        tc_commit_pair(k_empty + 0);
      }
      for (int it = 0; it < ntiles; ++it) {
        const int st = it % KS;
        const bool has_next = it + 1 < ntiles;
        Cursor nxt = cur;
        int nmode[2] = {kSkip, kSkip};
        const int kn = (it + 1) % KS;
        if (has_next) {
          cursor_next(prob, imax, nxt);
          for (int qt = 0; qt < 2; ++qt) nmode[qt] = tile_mode(prob.seg[nxt.seg], nxt.kt, TILE_R0(qt), nq);
          mbar_wait(k_full + kn, ((it + 1) / KS) & 1);
        }
        mbar_wait(v_full + st, (it / KS) & 1);
        tc_fence_after();
        for (int qt = 0; qt < 2; ++qt) {
          if (mode[qt] != kSkip) {
#pragma unroll
            for (int pp = 0; pp < kPParts; ++pp) {
              mbar_wait(p_full + 4 * qt + pp, p_cnt[qt] & 1);
              tc_fence_after();
              issue_pv(qt, st, o_acc[qt], pp * (8 / kPParts), 8 / kPParts);
            }
            o_acc[qt] = true;
            ++p_cnt[qt];
            tc_commit_pair(o_full + qt);
          }
          if (qt == 1) tc_commit_pair(v_empty + st);
          if (nmode[qt] != kSkip) {
            issue_qk(qt, kn);
            tc_commit_pair(s_full + qt);
          }
        }
        if (has_next) tc_commit_pair(k_empty + kn);
        cur = nxt;
        mode[0] = nmode[0];
        mode[1] = nmode[1];
      }
    }
  } else {
    // ======================================================== softmax warpgroups (both CTAs)
    const int qt = warp >> 2;
    const int quad = warp & 3;
    const int row = TILE_R0(qt) + quad * 32 + lane;
    const int qhead = TILE_HEAD(qt);
    const uint32_t t_lane = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t tS = tmem + t_lane + qt * 128;
    const uint32_t tO = tmem + t_lane + 256 + qt * 128;
    const float sl2 = P.scale_log2;
    const float2 sl2v = make_float2(sl2, sl2);
    float m_ref = -INFINITY, l = 0.f;
    uint32_t cnt = 0;
    Cursor cur = cursor_at(prob, imax, t_begin);
    for (int it = 0; it < ntiles; ++it, cursor_next(prob, imax, cur)) {
      const AttnSeg sg = prob.seg[cur.seg];
      const int mode = tile_mode(sg, cur.kt, TILE_R0(qt), nq);
      if (mode == kSkip) continue;
      mbar_wait(s_full + qt, cnt & 1);
      tc_fence_after();
      uint32_t sr[4][32];
      uint32_t pk[4][16];
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
      float mxp[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) mxp[t] = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const int t = (j / 2) & 7;
          mxp[t] = fmaxf(mxp[t], fmaxf(__uint_as_float(sr[c][j]), __uint_as_float(sr[c][j + 1])));
        }
      const float mx = fmaxf(fmaxf(fmaxf(mxp[0], mxp[1]), fmaxf(mxp[2], mxp[3])),
                             fmaxf(fmaxf(mxp[4], mxp[5]), fmaxf(mxp[6], mxp[7])));
      float alpha = 1.f;
      bool rescale = false;
      const float m_new = fmaxf(m_ref, mx * sl2);
      if (m_new > m_ref + 8.f) {
        alpha = exp2f(m_ref - m_new);
        m_ref = m_new;
        rescale = true;
      }
      const float m_use = (m_ref == -INFINITY) ? 0.f : m_ref;
      const float2 negm = make_float2(-m_use, -m_use);
      if (rescale && cnt > 0) {
        mbar_wait(o_full + qt, (cnt - 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < 16; ++c) {
          uint32_t o[8];
          tmem_ld8(tO + 8 * c, o);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
          tmem_st8(tO + 8 * c, o);
        }
      }
      float2 sacc[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) sacc[t] = make_float2(0.f, 0.f);
      auto chunk_exp = [&](int c) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 x2 = __ffma2_rn(
              make_float2(__uint_as_float(sr[c][2 * j]), __uint_as_float(sr[c][2 * j + 1])), sl2v, negm);
          sr[c][2 * j] = __float_as_uint(fast_exp2(x2.x));
          sr[c][2 * j + 1] = __float_as_uint(fast_exp2(x2.y));
        }
      };
      auto chunk_pack = [&](int c) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 p2 = make_float2(__uint_as_float(sr[c][2 * j]), __uint_as_float(sr[c][2 * j + 1]));
          sacc[j & 3] = __fadd2_rn(sacc[j & 3], p2);
          __nv_bfloat162 b = __floats2bfloat162_rn(p2.x, p2.y);
          pk[c][j] = *reinterpret_cast<uint32_t*>(&b);
        }
      };
      chunk_exp(0);
#pragma unroll
      for (int c = 1; c < 4; ++c) {
        chunk_exp(c);
        chunk_pack(c - 1);
        tmem_st16(tS + 16 * (c - 1), pk[c - 1]);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive_leader(p_full + 4 * qt + c - 1);
      }
      chunk_pack(3);
      tmem_st16(tS + 48, pk[3]);
      const float2 sum2 = __fadd2_rn(__fadd2_rn(sacc[0], sacc[1]), __fadd2_rn(sacc[2], sacc[3]));
      l = l * alpha + (sum2.x + sum2.y);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive_leader(p_full + 4 * qt + 3);
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
                                 __uint_as_float(o[4 * j + 2]) * inv, __uint_as_float(o[4 * j + 3]) * inv);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(prob.out) + obase + 32 * c);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t wv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(o[8 * j + 2 * e]) * inv,
                                                       __uint_as_float(o[8 * j + 2 * e + 1]) * inv);
              wv[e] = *reinterpret_cast<uint32_t*>(&b);
            }
            dst[j] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
          }
        }
      }
    }
    if (valid_row && prob.lse) {
      const float lse = (l > 0.f) ? (m_ref + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
      prob.lse[static_cast<long long>(split) * prob.split_stride_lse + static_cast<long long>(row) * prob.ld_lse +
               qhead] = lse;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the pair's last MMAs (issued by rank 0) are done with both TMEMs
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc2(tmem, kTmemCols);
#undef TILE_R0
#undef TILE_HEAD
}

template <int KS>
struct SmemPS {
  static constexpr uint32_t q = 0;
  static constexpr uint32_t k = q + kTilesPerCta * kTileBytes;
  static constexpr uint32_t v = k + KS * kHalfTile;
  static constexpr uint32_t p = v + KS * kHalfTile;  // P_0 | P_1, 32 KB each
  static constexpr uint32_t bar = p + kTilesPerCta * kTileBytes;
  static constexpr uint32_t total = bar + 256;
  static constexpr uint32_t bytes = total + 1024;
};

// Pair kernel with P in shared memory (SS PV): S_t is free as soon as the softmax has read
// it, so QK_t(j+1) no longer waits for PV_t(j) -- the softmax -> PV -> QK chain of the
// TMEM-aliased form is cut; the halved B operands leave the smem bandwidth for P.
template <int KS>
__global__ void __launch_bounds__(kThreads, 1) attn_pair_ps_kernel(const __grid_constant__ AttnParams P) {
  constexpr int kPParts = 4;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  using SL = SmemPS<KS>;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SL::bar);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;        // [KS]   counted on rank 0
  uint64_t* k_empty = k_full + KS;    // [KS]   both CTAs (multicast commit)
  uint64_t* v_full = k_empty + KS;    // [KS]   rank 0
  uint64_t* v_empty = v_full + KS;    // [KS]   both
  uint64_t* s_full = v_empty + KS;    // [2]    both
  uint64_t* p_full = s_full + 2;      // [2][4] rank 0, 256 arrivals (both CTAs' softmax)
  uint64_t* o_full = p_full + 8;      // [2]    both: PV done (O landed, P buffer free)
  uint64_t* s_free = o_full + 2;      // [2]    rank 0, 256 arrivals: S loaded by both CTAs
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_free + 2);
  static_assert((1 + 4 * KS + 14) * 8 + 4 <= 256, "barrier area");
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int warp = warp_id();
  const int lane = lane_id();

  // ---- decode the pair's work item: problem, 256-row unit (heaviest first), head group, split
  const int w = static_cast<int>(blockIdx.x >> 1);
  int pi = 0;
  while (pi + 1 < P.nprob && w >= P.prob[pi + 1].work_begin) ++pi;
  const AttnProb& prob = P.prob[pi];
  int local = w - prob.work_begin;
  const int split = local % prob.splits;
  local /= prob.splits;
  const int pair = prob.head_pair;  // nq <= 128: a CTA's two Q tiles are heads h, h+1
  const int ngroups = pair ? P.hq / 4 : P.hq / 2;
  const int g = local % ngroups;
  local /= ngroups;
  const int head = pair ? 4 * g + 2 * static_cast<int>(rank) : 2 * g + static_cast<int>(rank);
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
  const CUtensorMap* tm = P.tmap[pi];  // [0] Q, [1+2s] K (64-key boxes), [2+2s] V

  if (warp == kProducerWarp && elect_one()) {
    mbar_init(q_full, 1);
    for (int s = 0; s < KS; ++s) {
      mbar_init(k_full + s, 1);
      mbar_init(k_empty + s, 1);
      mbar_init(v_full + s, 1);
      mbar_init(v_empty + s, 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(s_full + t, 1);
      for (int pp = 0; pp < kPParts; ++pp) mbar_init(p_full + 4 * t + pp, 256);
      mbar_init(o_full + t, 1);
      mbar_init(s_free + t, 256);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tm[0]);
    for (int s = 0; s < prob.nseg; ++s) {
      tma_prefetch_desc(&tm[1 + 2 * s]);
      tma_prefetch_desc(&tm[2 + 2 * s]);
    }
  }
  if (warp == kMmaWarp) tmem_alloc2(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers exist before any remote arrive / TMA signal
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kProducerWarp) {
    // ======================================================== TMA producer (both CTAs)
    if (elect_one()) {
      const bool has1 = TILE_R0(1) < nq;
      if (leader) mbar_expect_tx(q_full, 2u * (has1 ? 2u : 1u) * kTileBytes);
      for (int qt = 0; qt < (has1 ? 2 : 1); ++qt)
        for (int c = 0; c < 2; ++c)
          tma_load_2d_pair(smem + SL::q + qt * kTileBytes + c * kBoxBytes, &tm[0], q_full,
                           TILE_HEAD(qt) * kHeadDim + c * 64, TILE_R0(qt));
      Cursor cur = cursor_at(prob, imax, t_begin);
      for (int it = 0; it < ntiles; ++it) {
        const CUtensorMap* km = &tm[1 + 2 * cur.seg];
        const CUtensorMap* vm = &tm[2 + 2 * cur.seg];
        const int st = it % KS;
        if (it >= KS) mbar_wait(k_empty + st, ((it / KS) - 1) & 1);
        if (leader) mbar_expect_tx(k_full + st, kTileBytes);  // both halves
        for (int c = 0; c < 2; ++c)  // keys [kt*128 + rank*64, +64), dh half c
          tma_load_2d_pair(smem + SL::k + st * kHalfTile + c * (kBoxBytes / 2), km, k_full + st,
                           hk * kHeadDim + c * 64, cur.kt * kBlockN + static_cast<int>(rank) * 64);
        if (it >= KS) mbar_wait(v_empty + st, ((it / KS) - 1) & 1);
        if (leader) mbar_expect_tx(v_full + st, kTileBytes);
        tma_load_2d_pair(smem + SL::v + st * kHalfTile, vm, v_full + st,
                         hk * kHeadDim + static_cast<int>(rank) * 64, cur.kt * kBlockN);  // dh half `rank`
        cursor_next(prob, imax, cur);
      }
    }
  } else if (warp == kMmaWarp) {
    // ======================================================== MMA issuer (rank 0 for the pair)
    if (leader && elect_one()) {
      const uint32_t idesc_qk = idesc_bf16_f32(256, 128, 0, 0);
      const uint32_t idesc_pv = idesc_bf16_f32(256, 128, 0, 1);
      const uint32_t sq = smem_u32(smem + SL::q);
      const uint32_t sk = smem_u32(smem + SL::k);
      const uint32_t sv = smem_u32(smem + SL::v);
      auto issue_qk = [&](int qt, int stage) {
        const uint32_t d = tmem + qt * 128;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t a = sdesc_sw128(sq + qt * kTileBytes + (kk >> 2) * kBoxBytes + (kk & 3) * 32, 16, 1024);
          const uint64_t b = sdesc_sw128(sk + stage * kHalfTile + (kk >> 2) * (kBoxBytes / 2) + (kk & 3) * 32, 16, 1024);
          mma_ss2(d, a, b, idesc_qk, kk > 0 ? 1u : 0u);
        }
      };
      auto issue_pv = [&](int qt, int stage, bool acc, int kk0, int n) {
        const uint32_t d = tmem + 256 + qt * 128;
        const uint32_t a = tmem + qt * 128;
#pragma unroll
        for (int k = 0; k < n; ++k) {
          const int kk = kk0 + k;
          const uint64_t b = sdesc_sw128(sv + stage * kHalfTile + kk * 2048, kHalfTile, 1024);
          mma_ts2(d, a + kk * 8, b, idesc_pv, (acc || kk > 0) ? 1u : 0u);
        }
      };
      const uint32_t sp = smem_u32(smem + SL::p);
      // PV with P from shared memory (SS): A = P_t, laid out like a Q tile
      auto issue_pv_s = [&](int qt, int stage, bool acc, int kk0, int n) {
        const uint32_t d = tmem + 256 + qt * 128;
#pragma unroll
        for (int k = 0; k < n; ++k) {
          const int kk = kk0 + k;
          const uint64_t a = sdesc_sw128(sp + qt * kTileBytes + (kk >> 2) * kBoxBytes + (kk & 3) * 32, 16, 1024);
          const uint64_t b = sdesc_sw128(sv + stage * kHalfTile + kk * 2048, kHalfTile, 1024);
          mma_ss2(d, a, b, idesc_pv, (acc || kk > 0) ? 1u : 0u);
        }
      };
      (void)issue_pv;
      mbar_wait(q_full, 0);
      tc_fence_after();
      // step j: QK(j) of both Q tiles as soon as K(j) is in and the softmax has LOADED S(j-1)
      // (P lives in shared memory, so S is free right after its tcgen05.ld), then PV(j-1)
      Cursor cur = cursor_at(prob, imax, t_begin);
      int mode_prev[2] = {kSkip, kSkip};
      uint32_t n_qk[2] = {0, 0}, p_cnt[2] = {0, 0};
      bool o_acc[2] = {false, false};
      auto pv_step = [&](int jj) {  // PV of tile jj (ring slot jj % KS)
        const int st = jj % KS;
        mbar_wait(v_full + st, (jj / KS) & 1);
        tc_fence_after();
        for (int qt = 0; qt < 2; ++qt)
          if (mode_prev[qt] != kSkip) {
#pragma unroll
            for (int pp = 0; pp < kPParts; ++pp) {
              mbar_wait(p_full + 4 * qt + pp, p_cnt[qt] & 1);
              tc_fence_after();
              issue_pv_s(qt, st, o_acc[qt], pp * (8 / kPParts), 8 / kPParts);
            }
            o_acc[qt] = true;
            ++p_cnt[qt];
            tc_commit_pair(o_full + qt);
          }
        tc_commit_pair(v_empty + st);
      };
      for (int it = 0; it < ntiles; ++it, cursor_next(prob, imax, cur)) {
        const int st = it % KS;
        int mode[2];
        for (int qt = 0; qt < 2; ++qt) mode[qt] = tile_mode(prob.seg[cur.seg], cur.kt, TILE_R0(qt), nq);
        mbar_wait(k_full + st, (it / KS) & 1);
        tc_fence_after();
        for (int qt = 0; qt < 2; ++qt)
          if (mode[qt] != kSkip) {
            if (n_qk[qt] > 0) {
              mbar_wait(s_free + qt, (n_qk[qt] - 1) & 1);
              tc_fence_after();
            }
            issue_qk(qt, st);
            tc_commit_pair(s_full + qt);
            ++n_qk[qt];
          }
        tc_commit_pair(k_empty + st);
        if (it > 0) pv_step(it - 1);
        mode_prev[0] = mode[0];
        mode_prev[1] = mode[1];
      }
      if (ntiles > 0) pv_step(ntiles - 1);
    }
  } else {
    // ======================================================== softmax warpgroups (both CTAs)
    const int qt = warp >> 2;
    const int quad = warp & 3;
    const int row = TILE_R0(qt) + quad * 32 + lane;
    const int qhead = TILE_HEAD(qt);
    const uint32_t t_lane = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t tS = tmem + t_lane + qt * 128;
    const uint32_t tO = tmem + t_lane + 256 + qt * 128;
    const float sl2 = P.scale_log2;
    const float2 sl2v = make_float2(sl2, sl2);
    float m_ref = -INFINITY, l = 0.f;
    uint32_t cnt = 0;
    Cursor cur = cursor_at(prob, imax, t_begin);
    for (int it = 0; it < ntiles; ++it, cursor_next(prob, imax, cur)) {
      const AttnSeg sg = prob.seg[cur.seg];
      const int mode = tile_mode(sg, cur.kt, TILE_R0(qt), nq);
      if (mode == kSkip) continue;
      mbar_wait(s_full + qt, cnt & 1);
      tc_fence_after();
      uint32_t sr[4][32];
      uint32_t pk[4][16];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32(tS + 32 * c, sr[c]);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive_leader(s_free + qt);  // S is in registers: QK(next) may overwrite it
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
      float mxp[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) mxp[t] = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const int t = (j / 2) & 7;
          mxp[t] = fmaxf(mxp[t], fmaxf(__uint_as_float(sr[c][j]), __uint_as_float(sr[c][j + 1])));
        }
      const float mx = fmaxf(fmaxf(fmaxf(mxp[0], mxp[1]), fmaxf(mxp[2], mxp[3])),
                             fmaxf(fmaxf(mxp[4], mxp[5]), fmaxf(mxp[6], mxp[7])));
      float alpha = 1.f;
      bool rescale = false;
      const float m_new = fmaxf(m_ref, mx * sl2);
      if (m_new > m_ref + 8.f) {
        alpha = exp2f(m_ref - m_new);
        m_ref = m_new;
        rescale = true;
      }
      const float m_use = (m_ref == -INFINITY) ? 0.f : m_ref;
      const float2 negm = make_float2(-m_use, -m_use);
      if (rescale && cnt > 0) {
        mbar_wait(o_full + qt, (cnt - 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < 16; ++c) {
          uint32_t o[8];
          tmem_ld8(tO + 8 * c, o);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 8; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * alpha);
          tmem_st8(tO + 8 * c, o);
        }
      }
      float2 sacc[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) sacc[t] = make_float2(0.f, 0.f);
      auto chunk_exp = [&](int c) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 x2 = __ffma2_rn(
              make_float2(__uint_as_float(sr[c][2 * j]), __uint_as_float(sr[c][2 * j + 1])), sl2v, negm);
          sr[c][2 * j] = __float_as_uint(fast_exp2(x2.x));
          sr[c][2 * j + 1] = __float_as_uint(fast_exp2(x2.y));
        }
      };
      auto chunk_pack = [&](int c) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 p2 = make_float2(__uint_as_float(sr[c][2 * j]), __uint_as_float(sr[c][2 * j + 1]));
          sacc[j & 3] = __fadd2_rn(sacc[j & 3], p2);
          __nv_bfloat162 b = __floats2bfloat162_rn(p2.x, p2.y);
          pk[c][j] = *reinterpret_cast<uint32_t*>(&b);
        }
      };
      // P_t in shared memory, laid out like a TMA-loaded Q tile (two 64-key SW128 boxes; row
      // r's 16-byte chunk j at ((j ^ (r & 7)) << 4)) -- the A operand of the SS PV
      const uint32_t prow = smem_u32(smem + SL::p) + qt * kTileBytes + ((quad * 32 + lane) >> 3) * 1024 +
                            ((lane & 7) << 7);
      auto store_p = [&](int c) {  // keys 32c .. 32c+31
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t a = prow + (c >> 1) * kBoxBytes + (((((c & 1) << 2) + q) ^ (lane & 7)) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(pk[c][4 * q]),
                       "r"(pk[c][4 * q + 1]), "r"(pk[c][4 * q + 2]), "r"(pk[c][4 * q + 3])
                       : "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_leader(p_full + 4 * qt + c);
      };
      chunk_exp(0);
#pragma unroll
      for (int c = 1; c < 4; ++c) {
        chunk_exp(c);
        chunk_pack(c - 1);
        if (c == 1 && cnt > 0 && !rescale) mbar_wait(o_full + qt, (cnt - 1) & 1);  // P buffer free
        store_p(c - 1);
      }
      chunk_pack(3);
      store_p(3);
      const float2 sum2 = __fadd2_rn(__fadd2_rn(sacc[0], sacc[1]), __fadd2_rn(sacc[2], sacc[3]));
      l = l * alpha + (sum2.x + sum2.y);
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
                                 __uint_as_float(o[4 * j + 2]) * inv, __uint_as_float(o[4 * j + 3]) * inv);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(prob.out) + obase + 32 * c);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t wv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              __nv_bfloat162 b = __floats2bfloat162_rn(__uint_as_float(o[8 * j + 2 * e]) * inv,
                                                       __uint_as_float(o[8 * j + 2 * e + 1]) * inv);
              wv[e] = *reinterpret_cast<uint32_t*>(&b);
            }
            dst[j] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
          }
        }
      }
    }
    if (valid_row && prob.lse) {
      const float lse = (l > 0.f) ? (m_ref + __log2f(l)) * 0.69314718055994530942f : -INFINITY;
      prob.lse[static_cast<long long>(split) * prob.split_stride_lse + static_cast<long long>(row) * prob.ld_lse +
               qhead] = lse;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the pair's last MMAs (issued by rank 0) are done with both TMEMs
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc2(tmem, kTmemCols);
#undef TILE_R0
#undef TILE_HEAD
}

#endif  // SPAVA_DEV_VARIANTS

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
                             cudaStream_t stream, std::string* err, const MergeJob* job, const ScoreJob* sj,
                             float scale) {
  if (dh != kHeadDim) {
    if (err) *err = "attention: only dh == 128 is implemented";
    return cudaErrorInvalidValue;
  }
  if (nprob < 1 || nprob > kMaxProbs || hq < 1 || hkv < 1 || hq % hkv) {
    if (err) *err = "attention: bad problem count or head counts";
    return cudaErrorInvalidValue;
  }
  // Per call (reentrant: the reference's operators are called from H host threads at once,
  // simhost.cpp:458-470); the launch copies the parameter block.
  AttnParams P;
  std::memset(&P, 0, sizeof(P));
  P.hq = hq;
  P.hkv = hkv;
  // logit scale: 1/sqrt(dh) (mha_lse, attention.cpp:163-165) unless the caller passes one
  // (attention_lse's explicit scale; heads narrower than 128 zero-padded to 128 columns)
  P.scale_log2 = (scale > 0.f ? scale : 1.0f / sqrtf(static_cast<float>(dh))) * 1.4426950408889634f;
  // kernel variants (spava_debug_attn_variant / SPAVA_ATTN_VARIANT, dev A/B only): all are
  // the ping-pong kernel (2 Q tiles per CTA, 320 threads) with different template switches.
  using KFn = void (*)(AttnParams);
  struct Var { KFn fn; uint32_t smem; int threads = kThreads; };
  // Only the production kernel ships; the A/B variants are compiled into a
  // dev build only (SPAVA_DEV_VARIANTS=1 python -m paper_2601_21444_b200.build --force).
  static const Var variants[] = {
      {attn_fwd_kernel<0, 2, false, true, false, 4, 0, false, false, 1, false>, Smem<2>::bytes},  // 0 production: P in 4 key ranges
#ifdef SPAVA_DEV_VARIANTS
      {attn_fwd_kernel<0, 2, true, true, false, 4, 0, false, false, 1, false>, Smem<2>::bytes},   // 1 0 + cycle counters
      {attn_fwd_kernel<0, 2, false, true, false, 1>, Smem<2>::bytes},  // 2 round-1 kernel (P whole)
      {attn_fwd_kernel<0, 2, false, true, false, 2>, Smem<2>::bytes},  // 3 P in 2 key ranges
      {attn_fwd_kernel<4, 2, false, true, false, 4, 0, false, false, 1, false>, Smem<2>::bytes},  // 4 0 + 25% FMA exp2
      {attn_fwd_kernel<2, 2, false, true, false, 4, 0, false, false, 1, false>, Smem<2>::bytes},  // 5 0 + 12.5% FMA exp2
      {attn_fwd_kernel<0, 3, false, true, false, 4>, Smem<3>::bytes},  // 6 0 + 3-deep K ring
      {attn_fwd_kernel<0, 2, false, true, true, 1>, Smem<2>::bytes},   // 7 speculative stale max
      {attn_fwd_kernel<0, 2, false, true, false, 4, 224, false, false, 1, false>, Smem<2>::bytes, 384},  // 8 0 + setmaxnreg
      {attn_fwd_kernel<4, 2, false, true, false, 4, 224, false, false, 1, false>, Smem<2>::bytes, 384},  // 9 8 + 25% FMA exp2
      {attn_fwd_kernel<2, 2, false, true, false, 4, 224, false, false, 1, false>, Smem<2>::bytes, 384},  // 10 8 + 12.5% FMA exp2
      {attn_fwd_kernel<0, 2, false, true, false, 4, 0, true>, Smem<2>::bytes},    // 11 0 + exp phases alternate
      {attn_fwd_kernel<0, 2, false, true, false, 4, 0, false, true>, Smem<2>::bytes},  // 12 0 + split S load
      {attn_fwd_kernel<0, 2, false, true, false, 4, 0, true, true>, Smem<2>::bytes},   // 13 11 + 12
      {attn_fwd_kernel<4, 2, false, true, false, 4, 224, true, true>, Smem<2>::bytes, 384},  // 14 13 + setmaxnreg + 25% FMA exp2
      {attn_fwd_kernel<0, 2, false, true, false, 4, 0, false, false, 1, false, true>, Smem<2>::bytes},  // 15 split QK (keys 64..127 under the softmax)
      {attn_fwd_kernel<0, 2, true, true, false, 4, 0, false, false, 1, false, true>, Smem<2>::bytes},   // 16 15 + cycle counters
      {attn_fwd_kernel<0, 2, false, true, false, 4, 0, false, false, 2>, Smem<2>::bytes + 10240, 576},  // 17 column-split softmax (4 warpgroups)
      {attn_fwd_kernel<4, 2, false, true, false, 4, 0, false, false, 2>, Smem<2>::bytes + 10240, 576},  // 18 17 + 25% FMA exp2
      {attn_fwd_kernel<2, 2, false, true, false, 4, 0, false, false, 2>, Smem<2>::bytes + 10240, 576},  // 19 17 + 12.5% FMA exp2
#endif
  };
  constexpr int kNumVar = sizeof(variants) / sizeof(variants[0]);
  static_assert(kNumVar <= 32, "attr mask");
  static const int env_sel = [] {
    const char* e = getenv("SPAVA_ATTN_VARIANT");
    const int v = e ? atoi(e) : 0;
    return (v >= 0 && v < kNumVar) ? v : 0;
  }();
  const int forced = g_attn_variant.load();
  const int vsel0 = (forced >= 0 && forced < kNumVar) ? forced : env_sel;
  // trailing merge / column-sum CTAs run with the production block shape
  const bool trailing = (job && job->ctas > 0) || (sj && sj->ctas > 0);
  const int vsel1 = (trailing && variants[vsel0].threads != kThreads) ? 0 : vsel0;
  // the fused-scorer query launch (per-block row statistics) takes the production kernel's
  // instance with the statistics compiled in
  static const Var stats_var = {attn_fwd_kernel<0, 2, false, true, false, 4, 0, false, false, 1, true>,
                                Smem<2>::bytes};
  bool stats = false;
  for (int i = 0; i < nprob; ++i) stats = stats || (probs[i].nq > 0 && probs[i].seg_lse2 != nullptr);
  const bool use_stats = stats && vsel1 == 0;
  const int vsel = use_stats ? 31 : vsel1;  // attr cache slot
  const Var& var = use_stats ? stats_var : variants[vsel1];
  constexpr int rows_per_cta = kTilesPerCta * kBlockM;
  int work = 0;
  int np = 0;
  int src_of[kMaxProbs] = {};
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
    p.head_pair = (v.nq <= kBlockM && (hq / hkv) % 2 == 0) ? 1 : 0;
    p.units = p.head_pair ? 1 : (v.nq + rows_per_cta - 1) / rows_per_cta;
    p.splits = v.splits;
    p.work_begin = work;
    p.out_f32 = v.out_f32;
    p.out = v.out;
    p.ldo = v.ldo;
    p.split_stride_out = v.split_stride_out;
    p.lse = v.lse;
    p.ld_lse = v.ld_lse;
    p.stat_seg[0] = v.stat_seg[0];
    p.stat_seg[1] = v.stat_seg[1];
    p.seg_lse2 = v.seg_lse2;
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
                     static_cast<long long>(hkv) * dh, v.seg[s].ld, err, kBlockN) ||
          !make_tmap(&P.tmap[np][2 + 2 * s], v.seg[s].v, v.seg[s].len,
                     static_cast<long long>(hkv) * dh, v.seg[s].ld, err, kBlockN))
        return cudaErrorInvalidValue;
    }
    work += p.units * (p.head_pair ? hq / 2 : hq) * p.splits;
    src_of[np] = i;
    ++np;
  }
  P.nprob = np;
  P.total_work = work;
  if (job && job->ctas > 0) {
    if (job->nwait < 0 || job->nwait > kMaxPeers || job->mp.nparts < 1 || job->mp.nparts > kMaxMergeParts ||
        job->mp.dh > 1024 || job->ctas > 64) {
      if (err) *err = "attention: bad merge job";
      return cudaErrorInvalidValue;
    }
    P.job = *job;
  }
  uint32_t smem_need = var.smem;
  if (sj && sj->ctas > 0) {
    if (np != 1 || !P.prob[0].seg_lse2 || !sj->counter || !sj->ready || sj->fa.ready != sj->ready ||
        P.prob[0].units != 1 || work / P.prob[0].splits > 32 ||
        sj->ctas != 2 * sj->fa.ntiles || sj->fa.hq != hq || sj->fa.hkv != hkv || sj->fa.n_t != P.prob[0].nq) {
      if (err) *err = "attention: bad fused score job";
      return cudaErrorInvalidValue;
    }
    P.sj = *sj;
    smem_need = std::max(smem_need, FSmem(hkv, hq).bytes());
  }
  const int grid = work + P.job.ctas + P.sj.ctas;
  if (grid == 0) return cudaSuccess;
#ifdef SPAVA_DEV_VARIANTS
  // CTA-pair kernels (dev build, SPAVA_ATTN_PAIR=1: P in TMEM, =2: P in shared memory): two
  // q-heads of one KV group per 2-CTA cluster
  static const int pair_env = [] {
    const char* e = getenv("SPAVA_ATTN_PAIR");
    return e ? atoi(e) : 0;
  }();
  if (pair_env && vsel == 0 && P.job.ctas == 0 && P.sj.ctas == 0) {
    bool ok = true;
    for (int q = 0; q < np; ++q)
      ok = ok && P.prob[q].seg_lse2 == nullptr && ((hq / hkv) % (P.prob[q].head_pair ? 4 : 2)) == 0;
    if (ok) {
      AttnParams P2 = P;
      int pw = 0;
      for (int q = 0; q < np; ++q) {
        AttnProb& p2 = P2.prob[q];
        p2.work_begin = pw;
        pw += p2.units * (p2.head_pair ? hq / 4 : hq / 2) * p2.splits;
        const ProbView& v = probs[src_of[q]];
        for (int sg = 0; sg < v.nseg; ++sg)  // K tiles of a pair: 64-key halves
          if (!make_tmap(&P2.tmap[q][1 + 2 * sg], v.seg[sg].k, v.seg[sg].len, static_cast<long long>(hkv) * dh,
                         v.seg[sg].ld, err, 64))
            return cudaErrorInvalidValue;
      }
      P2.total_work = pw;
      const KFn pf = pair_env == 2 ? attn_pair_ps_kernel<2> : attn_pair_kernel<kPairStages>;
      const uint32_t pbytes = pair_env == 2 ? SmemPS<2>::bytes : SmemP<kPairStages>::bytes;
      static std::atomic<uint32_t> attr_p[kMaxDevices] = {};
      if (cudaError_t e = smem_optin(reinterpret_cast<const void*>(pf), static_cast<int>(pbytes), attr_p, pair_env);
          e != cudaSuccess)
        return e;
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(2 * pw);
      lc.blockDim = dim3(kThreads);
      lc.dynamicSmemBytes = pbytes;
      lc.stream = stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      cudaError_t e = cudaLaunchKernelEx(&lc, pf, P2);
      if (e != cudaSuccess && err) *err = std::string("attention launch (pair): ") + cudaGetErrorString(e);
      return e;
    }
  }
#endif
  static std::atomic<uint32_t> attr_set[kMaxDevices] = {};
  const KFn fn = var.fn;
  const uint32_t smem_bytes = smem_need;
  // opted in at the larger of the kernel's and a fused scorer CTA's need (same for every call)
  if (cudaError_t e = smem_optin(reinterpret_cast<const void*>(fn),
                                 static_cast<int>(std::max(var.smem, kFSmemMaxBytes)), attr_set, vsel);
      e != cudaSuccess)
    return e;
  fn<<<grid, var.threads, smem_bytes, stream>>>(P);
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
#ifdef SPAVA_DEV_VARIANTS
  constexpr int kBuilt = 20;
#else
  constexpr int kBuilt = 1;
#endif
  if (v < -1 || v >= kBuilt) return -1;
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
