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
// p = float(e/sum) is evaluated as e*(1/sum) with an exact-division fallback whenever
// the product lands within a few fp64 ulps of an fp32 midpoint (or in fp32 subnormals),
// so it equals the correctly rounded quotient.
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

// 2^(j/256), j = 0..255, correctly rounded (generated with 60-digit decimal arithmetic)
__device__ __constant__ double c_exp2_256[256] = {
    0x1.0000000000000p+0, 0x1.00b1afa5abcbfp+0, 0x1.0163da9fb3335p+0, 0x1.02168143b0281p+0,
    0x1.02c9a3e778061p+0, 0x1.037d42e11bbccp+0, 0x1.04315e86e7f85p+0, 0x1.04e5f72f654b1p+0,
    0x1.059b0d3158574p+0, 0x1.0650a0e3c1f89p+0, 0x1.0706b29ddf6dep+0, 0x1.07bd42b72a836p+0,
    0x1.0874518759bc8p+0, 0x1.092bdf66607e0p+0, 0x1.09e3ecac6f383p+0, 0x1.0a9c79b1f3919p+0,
    0x1.0b5586cf9890fp+0, 0x1.0c0f145e46c85p+0, 0x1.0cc922b7247f7p+0, 0x1.0d83b23395decp+0,
    0x1.0e3ec32d3d1a2p+0, 0x1.0efa55fdfa9c5p+0, 0x1.0fb66affed31bp+0, 0x1.1073028d7233ep+0,
    0x1.11301d0125b51p+0, 0x1.11edbab5e2ab6p+0, 0x1.12abdc06c31ccp+0, 0x1.136a814f204abp+0,
    0x1.1429aaea92de0p+0, 0x1.14e95934f312ep+0, 0x1.15a98c8a58e51p+0, 0x1.166a45471c3c2p+0,
    0x1.172b83c7d517bp+0, 0x1.17ed48695bbc0p+0, 0x1.18af9388c8deap+0, 0x1.1972658375d2fp+0,
    0x1.1a35beb6fcb75p+0, 0x1.1af99f8138a1cp+0, 0x1.1bbe084045cd4p+0, 0x1.1c82f95281c6bp+0,
    0x1.1d4873168b9aap+0, 0x1.1e0e75eb44027p+0, 0x1.1ed5022fcd91dp+0, 0x1.1f9c18438ce4dp+0,
    0x1.2063b88628cd6p+0, 0x1.212be3578a819p+0, 0x1.21f49917ddc96p+0, 0x1.22bdda27912d1p+0,
    0x1.2387a6e756238p+0, 0x1.2451ffb82140ap+0, 0x1.251ce4fb2a63fp+0, 0x1.25e85711ece75p+0,
    0x1.26b4565e27cddp+0, 0x1.2780e341ddf29p+0, 0x1.284dfe1f56381p+0, 0x1.291ba7591bb70p+0,
    0x1.29e9df51fdee1p+0, 0x1.2ab8a66d10f13p+0, 0x1.2b87fd0dad990p+0, 0x1.2c57e39771b2fp+0,
    0x1.2d285a6e4030bp+0, 0x1.2df961f641589p+0, 0x1.2ecafa93e2f56p+0, 0x1.2f9d24abd886bp+0,
    0x1.306fe0a31b715p+0, 0x1.31432edeeb2fdp+0, 0x1.32170fc4cd831p+0, 0x1.32eb83ba8ea32p+0,
    0x1.33c08b26416ffp+0, 0x1.3496266e3fa2dp+0, 0x1.356c55f929ff1p+0, 0x1.36431a2de883bp+0,
    0x1.371a7373aa9cbp+0, 0x1.37f26231e754ap+0, 0x1.38cae6d05d866p+0, 0x1.39a401b7140efp+0,
    0x1.3a7db34e59ff7p+0, 0x1.3b57fbfec6cf4p+0, 0x1.3c32dc313a8e5p+0, 0x1.3d0e544ede173p+0,
    0x1.3dea64c123422p+0, 0x1.3ec70df1c5175p+0, 0x1.3fa4504ac801cp+0, 0x1.40822c367a024p+0,
    0x1.4160a21f72e2ap+0, 0x1.423fb2709468ap+0, 0x1.431f5d950a897p+0, 0x1.43ffa3f84b9d4p+0,
    0x1.44e086061892dp+0, 0x1.45c2042a7d232p+0, 0x1.46a41ed1d0057p+0, 0x1.4786d668b3237p+0,
    0x1.486a2b5c13cd0p+0, 0x1.494e1e192aed2p+0, 0x1.4a32af0d7d3dep+0, 0x1.4b17dea6db7d7p+0,
    0x1.4bfdad5362a27p+0, 0x1.4ce41b817c114p+0, 0x1.4dcb299fddd0dp+0, 0x1.4eb2d81d8abffp+0,
    0x1.4f9b2769d2ca7p+0, 0x1.508417f4531eep+0, 0x1.516daa2cf6642p+0, 0x1.5257de83f4eefp+0,
    0x1.5342b569d4f82p+0, 0x1.542e2f4f6ad27p+0, 0x1.551a4ca5d920fp+0, 0x1.56070dde910d2p+0,
    0x1.56f4736b527dap+0, 0x1.57e27dbe2c4cfp+0, 0x1.58d12d497c7fdp+0, 0x1.59c0827ff07ccp+0,
    0x1.5ab07dd485429p+0, 0x1.5ba11fba87a03p+0, 0x1.5c9268a5946b7p+0, 0x1.5d84590998b93p+0,
    0x1.5e76f15ad2148p+0, 0x1.5f6a320dceb71p+0, 0x1.605e1b976dc09p+0, 0x1.6152ae6cdf6f4p+0,
    0x1.6247eb03a5585p+0, 0x1.633dd1d1929fdp+0, 0x1.6434634ccc320p+0, 0x1.652b9febc8fb7p+0,
    0x1.6623882552225p+0, 0x1.671c1c70833f6p+0, 0x1.68155d44ca973p+0, 0x1.690f4b19e9538p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6b052fa75173ep+0, 0x1.6c012750bdabfp+0, 0x1.6cfdcddd47645p+0,
    0x1.6dfb23c651a2fp+0, 0x1.6ef9298593ae5p+0, 0x1.6ff7df9519484p+0, 0x1.70f7466f42e87p+0,
    0x1.71f75e8ec5f74p+0, 0x1.72f8286ead08ap+0, 0x1.73f9a48a58174p+0, 0x1.74fbd35d7cbfdp+0,
    0x1.75feb564267c9p+0, 0x1.77024b1ab6e09p+0, 0x1.780694fde5d3fp+0, 0x1.790b938ac1cf6p+0,
    0x1.7a11473eb0187p+0, 0x1.7b17b0976cfdbp+0, 0x1.7c1ed0130c132p+0, 0x1.7d26a62ff86f0p+0,
    0x1.7e2f336cf4e62p+0, 0x1.7f3878491c491p+0, 0x1.80427543e1a12p+0, 0x1.814d2add106d9p+0,
    0x1.82589994cce13p+0, 0x1.8364c1eb941f7p+0, 0x1.8471a4623c7adp+0, 0x1.857f4179f5b21p+0,
    0x1.868d99b4492edp+0, 0x1.879cad931a436p+0, 0x1.88ac7d98a6699p+0, 0x1.89bd0a478580fp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8be05bad61778p+0, 0x1.8cf3216b5448cp+0, 0x1.8e06a5e0866d9p+0,
    0x1.8f1ae99157736p+0, 0x1.902fed0282c8ap+0, 0x1.9145b0b91ffc6p+0, 0x1.925c353aa2fe2p+0,
    0x1.93737b0cdc5e5p+0, 0x1.948b82b5f98e5p+0, 0x1.95a44cbc8520fp+0, 0x1.96bdd9a7670b3p+0,
    0x1.97d829fde4e50p+0, 0x1.98f33e47a22a2p+0, 0x1.9a0f170ca07bap+0, 0x1.9b2bb4d53fe0dp+0,
    0x1.9c49182a3f090p+0, 0x1.9d674194bb8d5p+0, 0x1.9e86319e32323p+0, 0x1.9fa5e8d07f29ep+0,
    0x1.a0c667b5de565p+0, 0x1.a1e7aed8eb8bbp+0, 0x1.a309bec4a2d33p+0, 0x1.a42c980460ad8p+0,
    0x1.a5503b23e255dp+0, 0x1.a674a8af46052p+0, 0x1.a799e1330b358p+0, 0x1.a8bfe53c12e59p+0,
    0x1.a9e6b5579fdbfp+0, 0x1.ab0e521356ebap+0, 0x1.ac36bbfd3f37ap+0, 0x1.ad5ff3a3c2774p+0,
    0x1.ae89f995ad3adp+0, 0x1.afb4ce622f2ffp+0, 0x1.b0e07298db666p+0, 0x1.b20ce6c9a8952p+0,
    0x1.b33a2b84f15fbp+0, 0x1.b468415b749b1p+0, 0x1.b59728de5593ap+0, 0x1.b6c6e29f1c52ap+0,
    0x1.b7f76f2fb5e47p+0, 0x1.b928cf22749e4p+0, 0x1.ba5b030a1064ap+0, 0x1.bb8e0b79a6f1fp+0,
    0x1.bcc1e904bc1d2p+0, 0x1.bdf69c3f3a207p+0, 0x1.bf2c25bd71e09p+0, 0x1.c06286141b33dp+0,
    0x1.c199bdd85529cp+0, 0x1.c2d1cd9fa652cp+0, 0x1.c40ab5fffd07ap+0, 0x1.c544778fafb22p+0,
    0x1.c67f12e57d14bp+0, 0x1.c7ba88988c933p+0, 0x1.c8f6d9406e7b5p+0, 0x1.ca3405751c4dbp+0,
    0x1.cb720dcef9069p+0, 0x1.ccb0f2e6d1675p+0, 0x1.cdf0b555dc3fap+0, 0x1.cf3155b5bab74p+0,
    0x1.d072d4a07897cp+0, 0x1.d1b532b08c968p+0, 0x1.d2f87080d89f2p+0, 0x1.d43c8eacaa1d6p+0,
    0x1.d5818dcfba487p+0, 0x1.d6c76e862e6d3p+0, 0x1.d80e316c98398p+0, 0x1.d955d71ff6075p+0,
    0x1.da9e603db3285p+0, 0x1.dbe7cd63a8315p+0, 0x1.dd321f301b460p+0, 0x1.de7d5641c0658p+0,
    0x1.dfc97337b9b5fp+0, 0x1.e11676b197d17p+0, 0x1.e264614f5a129p+0, 0x1.e3b333b16ee12p+0,
    0x1.e502ee78b3ff6p+0, 0x1.e653924676d76p+0, 0x1.e7a51fbc74c83p+0, 0x1.e8f7977cdb740p+0,
    0x1.ea4afa2a490dap+0, 0x1.eb9f4867cca6ep+0, 0x1.ecf482d8e67f1p+0, 0x1.ee4aaa2188510p+0,
    0x1.efa1bee615a27p+0, 0x1.f0f9c1cb6412ap+0, 0x1.f252b376bba97p+0, 0x1.f3ac948dd7274p+0,
    0x1.f50765b6e4540p+0, 0x1.f6632798844f8p+0, 0x1.f7bfdad9cbe14p+0, 0x1.f91d802243c89p+0,
    0x1.fa7c1819e90d8p+0, 0x1.fbdba3692d514p+0, 0x1.fd3c22b8f71f1p+0, 0x1.fe9d96b2a23d9p+0};

// exp(x) for x <= 0 to ~1 fp64 ulp, branch-free: x = k ln2/256 + r (Cody-Waite, |r| <=
// ln2/512), exp(r) by a degree-5 polynomial (remainder < 1e-20), 2^(k/256) from a
// 256-entry smem table.  Returns 0 below -110: such terms change neither an fp64
// normaliser >= 1 nor any fp32 probability (e^-110 < FLT_TRUE_MIN / 2).
__device__ __forceinline__ double exp_neg(double x_in, const double* tab) {
  const bool live = x_in >= -110.0;  // false for -inf
  const double x = live ? x_in : -110.0;
  const double kd = rint(x * 0x1.71547652b82fep+8);  // 256 / ln2
  const int k = static_cast<int>(kd);
  double r = fma(-kd, 0x1.62e42fefa0000p-9, x);       // ln2/256 high (36 bits)
  r = fma(-kd, 0x1.cf79abc9e3b3ap-48, r);              // ln2/256 low
  double p = 0x1.1111111111111p-7;
  p = fma(p, r, 0x1.5555555555555p-5);
  p = fma(p, r, 0x1.5555555555555p-3);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const double y = p * tab[k & 255];
  const double r2 = __hiloint2double(__double2hiint(y) + ((k >> 8) << 20), __double2loint(y));
  return live ? r2 : 0.0;
}

__device__ __forceinline__ void load_exp_table(double* tab) {
  for (int i = threadIdx.x + threadIdx.y * blockDim.x; i < 256; i += blockDim.x * blockDim.y)
    tab[i] = c_exp2_256[i];
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
    // accumulators as fp32 pairs over adjacent keys: one packed FFMA2 (fma.rn.f32x2,
    // two independent IEEE fp32 FMAs) per pair -- sm_100's full fp32 rate.
    float2 acc2[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc2[i][j] = make_float2(0.f, 0.f);
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
        store_chunk(Qs[cur ^ 1], Ks[cur ^ 1], qr, kr);
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

// one CTA (256 threads) per (blk, h, i) row of L: mx = double(max_j l)*scale (== max of
// the exact products, monotone), sum = sum_j exp(x_j - mx) over non-pad keys (fp64 tree).
__global__ void __launch_bounds__(256) rowstats_kernel(const __grid_constant__ ScoreArgs a) {
  __shared__ double tab[256];
  __shared__ float redf[8];
  __shared__ double redd[8];
  load_exp_table(tab);
  const long long r = blockIdx.x;
  const int blk = static_cast<int>(r / (static_cast<long long>(a.hq) * a.n_t));
  const float* L = a.L + r * a.ldL;
  const uint8_t* pad = a.pad[blk];
  const int nv = a.n_valid[blk];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  float mxf = -INFINITY;
  for (int j = tid * 4; j < a.l_b; j += 1024) {
    const float4 v = *reinterpret_cast<const float4*>(L + j);
    const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (j + u < a.l_b && !is_pad(pad, nv, j + u)) mxf = fmaxf(mxf, e[u]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mxf = fmaxf(mxf, __shfl_xor_sync(0xffffffffu, mxf, o));
  if (lane == 0) redf[w] = mxf;
  __syncthreads();
  mxf = redf[0];
#pragma unroll
  for (int t = 1; t < 8; ++t) mxf = fmaxf(mxf, redf[t]);
  const double sc = static_cast<double>(a.scale);
  const double mx = static_cast<double>(mxf) * sc;
  double s0 = 0.0, s1 = 0.0;
  if (mxf != -INFINITY) {
    for (int j = tid * 4; j < a.l_b; j += 1024) {
      const float4 v = *reinterpret_cast<const float4*>(L + j);
      const float e[4] = {v.x, v.y, v.z, v.w};
      double t[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        t[u] = (j + u < a.l_b && !is_pad(pad, nv, j + u))
                   ? exp_neg(__dsub_rn(__dmul_rn(static_cast<double>(e[u]), sc), mx), tab)
                   : 0.0;
      s0 += t[0] + t[1];
      s1 += t[2] + t[3];
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
    a.stats[r * 3 + 0] = mxf == -INFINITY ? -INFINITY : mx;
    a.stats[r * 3 + 1] = tot;
    a.stats[r * 3 + 2] = 1.0 / tot;
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

// block (32, 8): thread (x, y) owns keys j, j+1 (j = blockIdx.x*64 + 2x) of block blockIdx.y
// for heads y, y+8, ...; rows i ascending per head (8-row batches keep 8 loads and 16
// independent exps in flight), heads ascending for the total.
__global__ void __launch_bounds__(256) colsum_kernel(const __grid_constant__ ScoreArgs a) {
  __shared__ float part[32][65];
  __shared__ double tab[256];
  load_exp_table(tab);
  __syncthreads();
  const int x = threadIdx.x, y = threadIdx.y, blk = blockIdx.y;
  const int j = blockIdx.x * 64 + 2 * x;
  const bool inb = j < a.l_b;  // j+1 < ldL always (ldL is a multiple of 128)
  const double sc = static_cast<double>(a.scale);
  for (int h = y; h < a.hq; h += 8) {
    float acc0 = 0.f, acc1 = 0.f;
    if (inb) {
      const long long hb = (static_cast<long long>(blk) * a.hq + h) * a.n_t;
      const float* L = a.L + hb * a.ldL + j;
      const double* st = a.stats + hb * 3;
      if (a.softmax) {
        int i = 0;
        for (; i + 8 <= a.n_t; i += 8) {
          float2 l[8];
          double m[8], sm[8], ri[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            l[u] = *reinterpret_cast<const float2*>(L + (i + u) * a.ldL);
            m[u] = st[(i + u) * 3];
            sm[u] = st[(i + u) * 3 + 1];
            ri[u] = st[(i + u) * 3 + 2];
          }
          float p0[8], p1[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            p0[u] = prob_f32(exp_neg(__dsub_rn(__dmul_rn(static_cast<double>(l[u].x), sc), m[u]), tab), sm[u], ri[u]);
            p1[u] = prob_f32(exp_neg(__dsub_rn(__dmul_rn(static_cast<double>(l[u].y), sc), m[u]), tab), sm[u], ri[u]);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            acc0 = __fadd_rn(acc0, p0[u]);
            acc1 = __fadd_rn(acc1, p1[u]);
          }
        }
        for (; i < a.n_t; ++i) {
          const float2 l = *reinterpret_cast<const float2*>(L + i * a.ldL);
          acc0 = __fadd_rn(acc0, prob_f32(exp_neg(__dsub_rn(__dmul_rn(static_cast<double>(l.x), sc), st[i * 3]), tab),
                                          st[i * 3 + 1], st[i * 3 + 2]));
          acc1 = __fadd_rn(acc1, prob_f32(exp_neg(__dsub_rn(__dmul_rn(static_cast<double>(l.y), sc), st[i * 3]), tab),
                                          st[i * 3 + 1], st[i * 3 + 2]));
        }
      } else {
        for (int i = 0; i < a.n_t; ++i) {
          const float2 l = *reinterpret_cast<const float2*>(L + i * a.ldL);
          acc0 = __fadd_rn(acc0, __fmul_rn(l.x, a.scale));
          acc1 = __fadd_rn(acc1, __fmul_rn(l.y, a.scale));
        }
      }
    }
    part[h][2 * x] = acc0;
    part[h][2 * x + 1] = acc1;
  }
  __syncthreads();
  const int t = y * 32 + x;
  const int jj = blockIdx.x * 64 + t;
  if (t < 64 && jj < a.l_b) {
    float total = 0.f;
    for (int h = 0; h < a.hq; ++h) total = __fadd_rn(total, part[h][t]);
    // pad keys -> -inf (approx.cpp:64-66); a block without visible keys is all pads
    a.scores[blk][jj] = is_pad(a.pad[blk], a.n_valid[blk], jj) ? -INFINITY : total;
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
    rowstats_kernel<<<static_cast<unsigned>(rows), 256, 0, stream>>>(a);
  }
  colsum_kernel<<<dim3((l_b + 63) / 64, nblk), dim3(32, 8), 0, stream>>>(a);
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
