// score.cu -- query-aware importance scoring of context blocks ("exact" mode).
//
// Reproduces score_block (simhost.cpp:209-224) -> score_context (approx.cpp:15-69) ->
// matmul_nt (matrix.cpp:73-86) operation by operation:
//   l_hij   = fp32 sum_c q[i,h,c]*k[j,h',c], c ascending        (h' = h / (hq/hkv))
//   x_hij   = double(l_hij) * double(scale)                     (exact in fp64)
//   mx_hi   = max_j x_hij ;  sum_hi = sum_j exp(x_hij - mx_hi)  (fp64, tree order)
//   part_hj = ((0 + p_h0j) + p_h1j) + ...,  p = float(exp(x - mx)/sum)   (fp32, i ascending)
//   score_j = ((0 + part_0j) + part_1j) + ...                   (fp32, h ascending)
// Inputs are bf16, so every q*k product is exact in fp32 and one FFMA per term equals
// the reference's multiply-then-add bit for bit; the logit chains run c-ascending.
// Differences from the CPU reference are confined to (a) the summation order of the
// fp64 normaliser sum_hi (a tree here) and (b) the fp64 exp (table+polynomial, <=1 ulp,
// vs glibc); both
// move p only when it lies within ~1e-15 of an fp32 rounding midpoint.
// p = float(e/sum) is evaluated as e*(1/sum) with a cheaper degree-5 exp and certified:
// accepted only when the result is provably on the same side of the fp32 rounding midpoint
// as the true quotient, else recomputed with the accurate exp and a true division
// (prob_cert), so it equals the correctly rounded quotient.
//
// Kernels (both blocks of a host in one launch each):
//   logits_kernel   : 128x128 CUDA-core SGEMM tile per CTA (8x8 register micro-tiles
//                     as packed FFMA2, c-chunks double-buffered in smem) -> L (fp32).
//   rowstats_kernel : one CTA per (block, head, row): fp64 (mx, sum, 1/sum).
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

// 2^(j/16), j = 0..15, correctly rounded (60-digit decimal arithmetic).  16 doubles fill
// the 32 smem banks exactly once, so the data-dependent table lookup never bank-conflicts
// (a 256-entry table costs ~5 wavefronts per warp lookup and was the scorer's bottleneck).
__device__ __constant__ double c_exp2_16[16] = {
    0x1.0000000000000p+0, 0x1.0b5586cf9890fp+0, 0x1.172b83c7d517bp+0, 0x1.2387a6e756238p+0,
    0x1.306fe0a31b715p+0, 0x1.3dea64c123422p+0, 0x1.4bfdad5362a27p+0, 0x1.5ab07dd485429p+0,
    0x1.6a09e667f3bcdp+0, 0x1.7a11473eb0187p+0, 0x1.8ace5422aa0dbp+0, 0x1.9c49182a3f090p+0,
    0x1.ae89f995ad3adp+0, 0x1.c199bdd85529cp+0, 0x1.d5818dcfba487p+0, 0x1.ea4afa2a490dap+0};

// Polynomial / reduction constants in the constant bank: DFMA takes c[][] operands
// directly, literal 64-bit constants were rematerialised with two IMAD.MOVs per use.
__device__ __constant__ double c_expk[10] = {
    0x1.71547652b82fep+4,   // 16/ln2
    0x1.8p52,               // round-to-integer magic
    -0x1.62e42fefa0000p-5,  // -ln2/16 high (36 bits: kd*hi exact)
    -0x1.cf79abc9e3b3ap-44, // -ln2/16 low
    0x1.a01a01a01a01ap-13,  // 1/7!
    0x1.6c16c16c16c17p-10,  // 1/6!
    0x1.1111111111111p-7,   // 1/5!
    0x1.5555555555555p-5,   // 1/4!
    0x1.5555555555555p-3,   // 1/3!
    0.5};

// exp(x) for -111 <= x <= 0 to ~1 fp64 ulp with no conversion-pipe instructions (cvt/frnd
// issue at 16/clk/SM on sm_100, a quarter of the DFMA rate): x = k ln2/16 + r with k read
// from the low word of x*16/ln2 + 1.5*2^52 (the DFMA itself rounds to nearest),
// Cody-Waite reduction (|r| <= ln2/32), exp(r) by the degree-7 Taylor polynomial
// (truncation < 1.3e-18 relative), 2^(k/16) from the table, 2^(k>>4) added to the
// exponent field.  Callers keep x >= -111 by clamping the fp32 logit at the per-row
// threshold lthr (x(lthr) ~ -110): e^-110 changes neither an fp64 normaliser >= 1 nor any
// fp32 probability (e^-110 < FLT_TRUE_MIN / 2), so the clamp is invisible in every result.
__device__ __forceinline__ double exp_neg(double x, const double* tab) {
  const double t = fma(x, c_expk[0], c_expk[1]);  // low word = k
  const double kd = t - c_expk[1];
  const int k = __double2loint(t);
  double r = fma(kd, c_expk[2], x);
  r = fma(kd, c_expk[3], r);
  double p = fma(c_expk[4], r, c_expk[5]);
  p = fma(p, r, c_expk[6]);
  p = fma(p, r, c_expk[7]);
  p = fma(p, r, c_expk[8]);
  p = fma(p, r, c_expk[9]);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double y = p * tab[k & 15];
  return __hiloint2double(__double2hiint(y) + ((k >> 4) << 20), __double2loint(y));
}

// exp(x) to a relative error below 1.5e-13 for -111 <= x <= 0: exp_neg with the Taylor
// polynomial cut at degree 5 (truncation (ln2/32)^6/720 = 1.4e-13; two DFMAs fewer).  Used
// only where the result is certified afterwards (prob_cert): that window is wide enough
// for this error, so every probability it accepts is the correctly rounded quotient --
// the same bits the accurate path gives.
__device__ __forceinline__ double exp_neg5(double x, const double* tab) {
  const double t = fma(x, c_expk[0], c_expk[1]);
  const double kd = t - c_expk[1];
  const int k = __double2loint(t);
  double r = fma(kd, c_expk[2], x);
  r = fma(kd, c_expk[3], r);
  double p = fma(c_expk[6], r, c_expk[7]);  // 1/120 r + 1/24
  p = fma(p, r, c_expk[8]);
  p = fma(p, r, c_expk[9]);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double y = p * tab[k & 15];
  return __hiloint2double(__double2hiint(y) + ((k >> 4) << 20), __double2loint(y));
}

// x = double(l)*scale - mx for the clamped logit (double(l)*scale is exact, so one fma
// equals the reference's multiply-then-subtract).
__device__ __forceinline__ double xrel(float l, float lthr, double sc, double mx) {
  return fma(static_cast<double>(fmaxf(l, lthr)), sc, -mx);
}

// per-row statistics: mx, sum, 1/sum, lthr (float in the low word of the 4th double)
constexpr int kStat = 4;

__device__ __forceinline__ void load_exp_table(double* tab) {
  const int t = threadIdx.x + threadIdx.y * blockDim.x;
  if (t < 16) tab[t] = c_exp2_16[t];
}

// Raw bf16 chunks are staged by cp.async two chunks ahead (no registers held across the
// FFMA2 loop -- a register prefetch was sunk by ptxas to just before its use, exposing
// the full global latency every chunk).  Thread t copies 16 B (8 c of one row) of Q and
// of K per chunk and later converts exactly those bytes, so cp.async.wait_group alone
// orders copy and conversion (no barrier between them).
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// row / 8-c group of this thread's 16-byte piece (lanes walk rows: conflict-free STS later)
__device__ __forceinline__ void issue_chunk(const ScoreArgs& a, const __nv_bfloat16* k, int h, int hk,
                                            int r0, int j0, int c0, uint4* Rq, uint4* Rk) {
  const int tid = threadIdx.x;
  const int row = tid % kTM, c8 = (tid / kTM) * 8;
  const bool vq = r0 + row < a.n_t, vk = j0 + row < a.l_b;
  const __nv_bfloat16* sq = a.q + static_cast<long long>(vq ? r0 + row : 0) * a.ldq + h * kDh + c0 + c8;
  const __nv_bfloat16* sk = k + static_cast<long long>(vk ? j0 + row : 0) * a.ldk + hk * kDh + c0 + c8;
  cp_async16(Rq + tid, sq, vq);
  cp_async16(Rk + tid, sk, vk);
}

__device__ __forceinline__ void convert_chunk(float* Qs, float* Ks, const uint4* Rq, const uint4* Rk) {
  const int tid = threadIdx.x;
  const int row = tid % kTM, c8 = (tid / kTM) * 8;
  const uint4 q = Rq[tid], kk = Rk[tid];
  const uint32_t qw[4] = {q.x, q.y, q.z, q.w}, kw[4] = {kk.x, kk.y, kk.z, kk.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    Qs[(c8 + 2 * i) * kTM + row] = __uint_as_float(qw[i] << 16);
    Qs[(c8 + 2 * i + 1) * kTM + row] = __uint_as_float(qw[i] & 0xffff0000u);
    Ks[(c8 + 2 * i) * kTN + row] = __uint_as_float(kw[i] << 16);
    Ks[(c8 + 2 * i + 1) * kTN + row] = __uint_as_float(kw[i] & 0xffff0000u);
  }
}

// grid (ntiles, hq, nblk), 256 threads: L tile 128 rows x 128 keys, rows chunked by 128.
__global__ void __launch_bounds__(kThr, 2) logits_kernel(const __grid_constant__ ScoreArgs a) {
  __shared__ __align__(16) float Qs[2][kKC * kTM];
  __shared__ __align__(16) float Ks[2][kKC * kTN];
  __shared__ __align__(16) uint4 Rq[2][kThr];  // raw bf16 chunks (cp.async ring)
  __shared__ __align__(16) uint4 Rk[2][kThr];
  const int tile = blockIdx.x, h = blockIdx.y, blk = blockIdx.z;
  const int hk = h / (a.hq / a.hkv);
  const int j0 = tile * kTN;
  const __nv_bfloat16* k = a.k[blk];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  constexpr int kChunks = kDh / kKC;
  for (int r0 = 0; r0 < a.n_t; r0 += kTM) {
    // accumulators as fp32 pairs over adjacent keys: one packed FFMA2 (fma.rn.f32x2,
    // two independent IEEE fp32 FMAs) per pair -- sm_100's full fp32 rate.
    float2 acc2[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc2[i][j] = make_float2(0.f, 0.f);
    issue_chunk(a, k, h, hk, r0, j0, 0, Rq[0], Rk[0]);
    cp_async_commit();
    issue_chunk(a, k, h, hk, r0, j0, kKC, Rq[1], Rk[1]);
    cp_async_commit();
    cp_async_wait1();
    convert_chunk(Qs[0], Ks[0], Rq[0], Rk[0]);
    __syncthreads();
    for (int ch = 0; ch < kChunks; ++ch) {
      const int cur = ch & 1;
      // chunk ch+2 into the raw slot this thread converted from last (its own bytes only)
      if (ch + 2 < kChunks) issue_chunk(a, k, h, hk, r0, j0, (ch + 2) * kKC, Rq[cur], Rk[cur]);
      cp_async_commit();
#pragma unroll
      for (int c = 0; c < kKC; ++c) {  // ascending c within the chunk, chunks ascending
        const float4 qa = *reinterpret_cast<const float4*>(&Qs[cur][c * kTM + ty * 4]);
        const float4 qb = *reinterpret_cast<const float4*>(&Qs[cur][c * kTM + 64 + ty * 4]);
        const float4 ka = *reinterpret_cast<const float4*>(&Ks[cur][c * kTN + tx * 4]);
        const float4 kb = *reinterpret_cast<const float4*>(&Ks[cur][c * kTN + 64 + tx * 4]);
        const float qv[8] = {qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qb.z, qb.w};
        const float2 k2[4] = {make_float2(ka.x, ka.y), make_float2(ka.z, ka.w),
                              make_float2(kb.x, kb.y), make_float2(kb.z, kb.w)};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float2 q2 = make_float2(qv[i], qv[i]);
#pragma unroll
          for (int j = 0; j < 4; ++j) acc2[i][j] = __ffma2_rn(q2, k2[j], acc2[i][j]);
        }
      }
      if (ch + 1 < kChunks) {
        cp_async_wait1();  // chunk ch+1 landed (ch+2 may still be in flight)
        convert_chunk(Qs[cur ^ 1], Ks[cur ^ 1], Rq[cur ^ 1], Rk[cur ^ 1]);
        __syncthreads();
      }
    }
    // ---- epilogue: L (fp32) straight from the packed accumulators
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = r0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
      if (row < a.n_t) {
        float* Lr = a.L + ((static_cast<long long>(blk) * a.hq + h) * a.n_t + row) * a.ldL + j0;
        *reinterpret_cast<float4*>(Lr + tx * 4) =
            make_float4(acc2[i][0].x, acc2[i][0].y, acc2[i][1].x, acc2[i][1].y);
        *reinterpret_cast<float4*>(Lr + 64 + tx * 4) =
            make_float4(acc2[i][2].x, acc2[i][2].y, acc2[i][3].x, acc2[i][3].y);
      }
    }
    __syncthreads();
  }
}

// One CTA (256 threads) per (blk, h, i) row of L: mx = double(max_j l)*scale (== the max
// of the exact products, monotone), sum = sum_j exp(x_j - mx) over non-pad keys (fp64,
// thread-strided, then butterfly + 8-warp tree).  kPad: an explicit pad mask (the
// partition's pads are a tail, passed as n_valid, so the production path reads no mask).
// kRegF4 > 0: the thread's share of the row (<= kRegF4 float4, l_b <= kRegF4 * 1024) is
// loaded once, all loads in flight together, and kept in registers for the sum pass;
// kRegF4 == 0 streams the row twice (long blocks, e.g. C4 at H = 1).
template <bool kPad, int kRegF4>
__global__ void __launch_bounds__(256) rowstats_kernel(const __grid_constant__ ScoreArgs a) {
  __shared__ double tab[16];
  __shared__ float redf[8];
  __shared__ double redd[8];
  load_exp_table(tab);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const long long r = blockIdx.x;
  const int blk = r >= static_cast<long long>(a.hq) * a.n_t ? 1 : 0;
  const float* L = a.L + r * a.ldL;
  const uint8_t* pad = a.pad[blk];
  const int nv = min(a.n_valid[blk], a.l_b);
  auto vis = [&](int j) { return j < nv && !(kPad && pad[j]); };
  constexpr int kU = kRegF4 > 0 ? kRegF4 : 4;  // float4 loads in flight per thread
  float4 keep[kRegF4 > 0 ? kRegF4 : 1];
  float mxf = -INFINITY;
  for (int j0 = tid * 4; j0 < nv; j0 += kU * 1024) {
    float4 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      v[u] = j0 + u * 1024 < nv ? *reinterpret_cast<const float4*>(L + j0 + u * 1024)
                                : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (kRegF4 > 0) keep[u] = v[u];
      const int j = j0 + u * 1024;
      if (j + 4 <= nv && !kPad) {
        mxf = fmaxf(fmaxf(mxf, fmaxf(v[u].x, v[u].y)), fmaxf(v[u].z, v[u].w));
      } else {
        if (vis(j)) mxf = fmaxf(mxf, v[u].x);
        if (vis(j + 1)) mxf = fmaxf(mxf, v[u].y);
        if (vis(j + 2)) mxf = fmaxf(mxf, v[u].z);
        if (vis(j + 3)) mxf = fmaxf(mxf, v[u].w);
      }
    }
    if (kRegF4 > 0) break;  // the whole share is in registers (l_b <= kRegF4 * 1024)
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mxf = fmaxf(mxf, __shfl_xor_sync(0xffffffffu, mxf, o));
  if (lane == 0) redf[w] = mxf;
  __syncthreads();  // also publishes tab
  mxf = redf[0];
#pragma unroll
  for (int t = 1; t < 8; ++t) mxf = fmaxf(mxf, redf[t]);
  const double sc = static_cast<double>(a.scale);
  const double mx = static_cast<double>(mxf) * sc;
  const float lthr = static_cast<float>((mx - 110.0) / sc);
  double s0 = 0.0, s1 = 0.0;
  auto add4 = [&](const float4& v, int j) {
    double e0 = exp_neg(xrel(v.x, lthr, sc, mx), tab);
    double e1 = exp_neg(xrel(v.y, lthr, sc, mx), tab);
    double e2 = exp_neg(xrel(v.z, lthr, sc, mx), tab);
    double e3 = exp_neg(xrel(v.w, lthr, sc, mx), tab);
    if (kPad || j + 4 > nv) {
      e0 = vis(j) ? e0 : 0.0;
      e1 = vis(j + 1) ? e1 : 0.0;
      e2 = vis(j + 2) ? e2 : 0.0;
      e3 = vis(j + 3) ? e3 : 0.0;
    }
    s0 += e0 + e1;
    s1 += e2 + e3;
  };
  if (mxf != -INFINITY) {
    if (kRegF4 > 0) {
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int j = tid * 4 + u * 1024;
        if (j < nv) add4(keep[u], j);
      }
    } else {
      for (int j0 = tid * 4; j0 < nv; j0 += kU * 1024) {
        float4 v[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u)
          v[u] = j0 + u * 1024 < nv ? *reinterpret_cast<const float4*>(L + j0 + u * 1024)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int j = j0 + u * 1024;
          if (j < nv) add4(v[u], j);
        }
      }
    }
  }
  double sum = s0 + s1;
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) redd[w] = sum;
  __syncthreads();
  if (tid == 0) {
    double tot = 0.0;
#pragma unroll
    for (int t = 0; t < 8; ++t) tot += redd[t];
    a.stats[r * kStat + 0] = mxf == -INFINITY ? -INFINITY : mx;
    a.stats[r * kStat + 1] = tot;
    a.stats[r * kStat + 2] = 1.0 / tot;
    a.stats[r * kStat + 3] = __hiloint2double(0, __float_as_int(lthr));
  }
}

// Short blocks (l_b <= 4096, H >= 4): one WARP per row, 8 rows per CTA -- the same
// statistics with warp-only reductions (the CTA-per-row kernel is dominated by its two
// block reductions there).  Tail pads only (n_valid); two streaming passes over the row
// (the second hits L1/L2).
__global__ void __launch_bounds__(256) rowstats_warp_kernel(const __grid_constant__ ScoreArgs a, int rows) {
  __shared__ double tab[16];
  load_exp_table(tab);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int blk = r >= a.hq * a.n_t ? 1 : 0;
  const float* L = a.L + static_cast<long long>(r) * a.ldL;
  const int nv = min(a.n_valid[blk], a.l_b);
  constexpr int kU = 4;
  float mxf = -INFINITY;
  for (int j0 = lane * 4; j0 < nv; j0 += kU * 128) {
    float4 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      v[u] = j0 + u * 128 < nv ? *reinterpret_cast<const float4*>(L + j0 + u * 128)
                               : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int j = j0 + u * 128;
      if (j + 4 <= nv) {
        mxf = fmaxf(fmaxf(mxf, fmaxf(v[u].x, v[u].y)), fmaxf(v[u].z, v[u].w));
      } else {
        if (j < nv) mxf = fmaxf(mxf, v[u].x);
        if (j + 1 < nv) mxf = fmaxf(mxf, v[u].y);
        if (j + 2 < nv) mxf = fmaxf(mxf, v[u].z);
        if (j + 3 < nv) mxf = fmaxf(mxf, v[u].w);
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mxf = fmaxf(mxf, __shfl_xor_sync(0xffffffffu, mxf, o));
  const double sc = static_cast<double>(a.scale);
  const double mx = static_cast<double>(mxf) * sc;
  const float lthr = static_cast<float>((mx - 110.0) / sc);
  double s0 = 0.0, s1 = 0.0;
  if (mxf != -INFINITY) {
    for (int j0 = lane * 4; j0 < nv; j0 += kU * 128) {
      float4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u)
        v[u] = j0 + u * 128 < nv ? *reinterpret_cast<const float4*>(L + j0 + u * 128)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int j = j0 + u * 128;
        if (j >= nv) continue;
        double e0 = exp_neg(xrel(v[u].x, lthr, sc, mx), tab);
        double e1 = exp_neg(xrel(v[u].y, lthr, sc, mx), tab);
        double e2 = exp_neg(xrel(v[u].z, lthr, sc, mx), tab);
        double e3 = exp_neg(xrel(v[u].w, lthr, sc, mx), tab);
        if (j + 4 > nv) {
          e1 = j + 1 < nv ? e1 : 0.0;
          e2 = j + 2 < nv ? e2 : 0.0;
          e3 = j + 3 < nv ? e3 : 0.0;
        }
        s0 += e0 + e1;
        s1 += e2 + e3;
      }
    }
  }
  double sum = s0 + s1;
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) {
    a.stats[static_cast<long long>(r) * kStat + 0] = mxf == -INFINITY ? -INFINITY : mx;
    a.stats[static_cast<long long>(r) * kStat + 1] = sum;
    a.stats[static_cast<long long>(r) * kStat + 2] = 1.0 / sum;
    a.stats[static_cast<long long>(r) * kStat + 3] = __hiloint2double(0, __float_as_int(lthr));
  }
}

__device__ __forceinline__ float lthr_of(const double* st) {
  return __int_as_float(__double2loint(st[3]));
}

// float(e / sum) from an exp_neg5 value, certified: y = e*(1/sum) is within 1.5e-13 relative
// of the true quotient q = exp(x)/sum, i.e. within ~1.4e3 fp64 ulps of y.  Outside a
// +-2048-ulp window around the fp32 rounding midpoint (29 bits below the fp32 mantissa)
// float(y) == float(q); inside it (probability 2^-17) or below FLT_MIN the caller
// recomputes with the accurate exp and a true division -- exactly what the accurate path
// does there, so accepted and recomputed probabilities are the bits the accurate path gives.
__device__ __forceinline__ float prob_cert(double e, double rinv, bool& redo) {
  const double y = __dmul_rn(e, rinv);
  const unsigned low = static_cast<unsigned>(__double2loint(y)) & ((1u << 29) - 1);
  redo |= (low - ((1u << 28) - 2048)) < 4096u || y < 1.1754943508222875e-38;
  return __double2float_rn(y);
}

// CTA = 32 keys x all heads: warp w owns heads w, w+16, ...; lane owns key j.  Per head the
// column sum runs over query rows i ascending (8-row batches keep 8 loads and 8
// independent exps in flight per lane), then the ordered sum over heads through smem.
// kSmemStats: the per-row statistics (mx, 1/sum, lthr) of every (head, row) are staged in
// shared memory once per CTA (warp-uniform broadcast reads) instead of three global loads
// per element; used whenever hq * n_t rows fit (the C1..C4 shapes).
constexpr int kColWarps = 16;
constexpr int kColStatBytes = 20;  // double mx, double 1/sum, float lthr
template <bool kSmemStats>
__global__ void __launch_bounds__(kColWarps * 32) colsum_kernel(const __grid_constant__ ScoreArgs a) {
  __shared__ float part[32][33];
  __shared__ double tab[16];
  extern __shared__ __align__(16) uint8_t col_smem[];
  double2* sstat = reinterpret_cast<double2*>(col_smem);                       // [hq*n_t] (mx, rinv)
  float* slthr = reinterpret_cast<float*>(col_smem + 16ull * a.hq * a.n_t);    // [hq*n_t]
  load_exp_table(tab);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, blk = blockIdx.y;
  if (kSmemStats && a.softmax) {
    const double* stb = a.stats + static_cast<long long>(blk) * a.hq * a.n_t * kStat;
    for (int r = threadIdx.x; r < a.hq * a.n_t; r += kColWarps * 32) {
      sstat[r] = make_double2(stb[r * kStat], stb[r * kStat + 2]);
      slthr[r] = lthr_of(stb + r * kStat);
    }
  }
  __syncthreads();
  const int j = blockIdx.x * 32 + lane;
  const bool inb = j < a.l_b;  // j < ldL always (ldL is a multiple of 128)
  const double sc = static_cast<double>(a.scale);
  for (int h = w; h < a.hq; h += kColWarps) {
    const long long hb = (static_cast<long long>(blk) * a.hq + h) * a.n_t;
    const float* L = a.L + hb * a.ldL + j;
    const double* st = a.stats + hb * kStat;
    auto mx_of = [&](int i) { return kSmemStats ? sstat[h * a.n_t + i].x : st[i * kStat]; };
    auto rinv_of = [&](int i) { return kSmemStats ? sstat[h * a.n_t + i].y : st[i * kStat + 2]; };
    auto thr_of = [&](int i) { return kSmemStats ? slthr[h * a.n_t + i] : lthr_of(st + i * kStat); };
    float acc = 0.f;
    if (a.softmax) {
      int i = 0;
      float l[8], ln[8];
      if (a.n_t >= 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) ln[u] = L[static_cast<long long>(u) * a.ldL];
      }
      for (; i + 8 <= a.n_t; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) l[u] = ln[u];
        if (i + 16 <= a.n_t) {  // next batch in flight during this one
#pragma unroll
          for (int u = 0; u < 8; ++u) ln[u] = L[static_cast<long long>(i + 8 + u) * a.ldL];
        }
        float p[8];
        bool redo = false;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          p[u] = prob_cert(exp_neg5(xrel(l[u], thr_of(i + u), sc, mx_of(i + u)), tab), rinv_of(i + u), redo);
        if (redo) {
#pragma unroll 1
          for (int u = 0; u < 8; ++u) {
            const double e = exp_neg(xrel(l[u], thr_of(i + u), sc, mx_of(i + u)), tab);
            p[u] = __double2float_rn(__ddiv_rn(e, st[(i + u) * kStat + 1]));
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = __fadd_rn(acc, p[u]);
      }
      for (; i < a.n_t; ++i) {
        const double e = exp_neg(xrel(L[static_cast<long long>(i) * a.ldL], thr_of(i), sc, mx_of(i)), tab);
        acc = __fadd_rn(acc, __double2float_rn(__ddiv_rn(e, st[i * kStat + 1])));
      }
    } else {
      for (int i = 0; i < a.n_t; ++i) acc = __fadd_rn(acc, __fmul_rn(L[static_cast<long long>(i) * a.ldL], a.scale));
    }
    part[h][lane] = acc;
  }
  __syncthreads();
  if (w == 0 && inb) {
    float total = 0.f;
    for (int h = 0; h < a.hq; ++h) total = __fadd_rn(total, part[h][lane]);
    // pad keys -> -inf (approx.cpp:64-66); a block without visible keys is all pads
    a.scores[blk][j] = is_pad(a.pad[blk], a.n_valid[blk], j) ? -INFINITY : total;
  }
}

}  // namespace

size_t score_workspace_bytes(int n_t, int l_b, int hq) {
  // sized for two blocks (lo + hi) scored in one launch
  const size_t L = 2ull * hq * n_t * ld_logits(l_b) * sizeof(float);
  const size_t part = 2ull * hq * n_t * n_ktiles(l_b) * sizeof(double2);
  const size_t st = 2ull * hq * n_t * kStat * sizeof(double);
  return L + part + st + 1024;
}

cudaError_t launch_score_exact2(int nblk, const void* q, long long ldq, int n_t,
                                const void* const* k, long long ldk, int l_b,
                                const uint8_t* const* pad, const int* n_valid, int hq, int hkv,
                                int dh, int softmax, float* const* scores, void* ws,
                                size_t ws_bytes, cudaStream_t stream, float scale) {
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
  a.scale = scale > 0.f ? scale : 1.0f / sqrtf(static_cast<float>(dh));  // score_context's scale
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
    const unsigned grid = static_cast<unsigned>(rows);
    bool any_pad = false;
    for (int b = 0; b < nblk; ++b) any_pad |= a.pad[b] != nullptr;
    if (any_pad)
      rowstats_kernel<true, 0><<<grid, 256, 0, stream>>>(a);
    else if (l_b <= 4 * 1024)
      rowstats_warp_kernel<<<(grid + 7) / 8, 256, 0, stream>>>(a, static_cast<int>(rows));
    else if (l_b <= 8 * 1024)
      rowstats_kernel<false, 8><<<grid, 256, 0, stream>>>(a);
    else if (l_b <= 16 * 1024)
      rowstats_kernel<false, 16><<<grid, 256, 0, stream>>>(a);
    else
      rowstats_kernel<false, 0><<<grid, 256, 0, stream>>>(a);
  }
  const size_t stat_smem = static_cast<size_t>(kColStatBytes) * hq * n_t;
  if (softmax && stat_smem <= 96 * 1024) {
    static std::atomic<uint32_t> attr[kMaxDevices] = {};
    if (cudaError_t e = smem_optin(reinterpret_cast<const void*>(colsum_kernel<true>), 96 * 1024, attr, 0);
        e != cudaSuccess)
      return e;
    colsum_kernel<true><<<dim3((l_b + 31) / 32, nblk), kColWarps * 32, stat_smem, stream>>>(a);
  } else {
    colsum_kernel<false><<<dim3((l_b + 31) / 32, nblk), kColWarps * 32, 0, stream>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_score_exact(const void* q, long long ldq, int n_t, const void* k,
                               long long ldk, int l_b, const uint8_t* pad, int n_valid, int hq,
                               int hkv, int dh, int softmax, float* scores, void* ws,
                               size_t ws_bytes, cudaStream_t stream, float scale) {
  const void* ks[1] = {k};
  const uint8_t* pads[1] = {pad};
  const int nv[1] = {n_valid};
  float* sc[1] = {scores};
  return launch_score_exact2(1, q, ldq, n_t, ks, ldk, l_b, pads, nv, hq, hkv, dh, softmax, sc, ws,
                             ws_bytes, stream, scale);
}

}  // namespace spava
