// select.cu -- essential-KV selection and packing (the compressor's back half).
//
// select_essential (approx.cpp:71-102): stable descending sort of the block's scores
// (ties -> lower index), take at most l_p stopping at the first non-finite, return the
// chosen indices ascending (+ global offset) and gather their K/V rows.
// GPU form, no sort at all (one CTA per block -- 1024 threads, or 256 for l_b <= 4096 --
// each thread owning 16 consecutive keys of a chunk):
//   1. count finite scores (k = min(l_p, #finite); any +inf sorts first and ends the
//      selection immediately; NaN is rejected),
//   2. 3-pass MSB radix select (11/11/10-bit digits, warp-aggregated smem histograms,
//      parallel bucket scan) over order-preserving uint32 keys finds the k-th largest
//      key T and how many keys equal to T are taken,
//   3. one index-ordered block scan emits key > T plus the lowest-index keys == T
//      (exactly the stable-sort tie rule), already ascending,
// then a multi-CTA gather copies the selected K/V rows (16 B per lane, coalesced)
// straight into this host's slot of the exchange buffer.
#include <cuda_bf16.h>

#include "fabric_dev.cuh"
#include "spava_internal.h"

namespace spava {

namespace {

constexpr int kItems = 16;
// 1024 threads for long blocks; 256 for l_b <= 4096 (H >= 4 shapes), where the selection
// is latency-bound and a smaller CTA halves the barrier / scan depth
constexpr int kSelBig = 1024, kSelSmall = 256;

__device__ __forceinline__ uint32_t order_key(float s) {
  const uint32_t u = __float_as_uint(s);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// inclusive warp scan
__device__ __forceinline__ int warp_incl(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += n;
  }
  return v;
}

// exclusive block scan of v (thread order); *total = block sum.  Uses red[NW + 1].
template <int NW>
__device__ __forceinline__ int block_excl(int v, int* red, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int inc = warp_incl(v);
  __syncthreads();
  if (lane == 31) red[w] = inc;
  __syncthreads();
  if (w == 0) {
    const int x = lane < NW ? red[lane] : 0;
    const int xi = warp_incl(x);
    if (lane < NW) red[lane] = xi - x;
    if (lane == 31) red[NW] = xi;
  }
  __syncthreads();
  *total = red[NW];
  return red[w] + inc - v;
}

__device__ __forceinline__ void load_items(const float* s, int l_b, int base, float (&v)[kItems]) {
  // thread t owns keys [base + t*kItems, +kItems)
  const int j0 = base + threadIdx.x * kItems;
  if (j0 + kItems <= l_b && ((reinterpret_cast<uintptr_t>(s + j0) & 15) == 0)) {
#pragma unroll
    for (int q = 0; q < kItems / 4; ++q) {
      const float4 f = reinterpret_cast<const float4*>(s + j0)[q];
      v[4 * q] = f.x;
      v[4 * q + 1] = f.y;
      v[4 * q + 2] = f.z;
      v[4 * q + 3] = f.w;
    }
  } else {
#pragma unroll
    for (int t = 0; t < kItems; ++t) v[t] = (j0 + t < l_b) ? s[j0 + t] : -INFINITY;
  }
}

// one job per block (lo, hi): selection and gather of both blocks in one launch each
struct SelJob {
  const float* scores;
  int global_offset;
  int32_t* idx;
  int32_t* count;
  const uint4* k;
  const uint4* v;
  uint4* k_out;
  uint4* v_out;
  PeerSlots peers;
  FlagRaise fr;
  int require_full;  // a passing source: fewer than l_p keys is reported (status bit 2)
};
struct SelJobs {
  SelJob j[2];
  int l_b, l_p, w16;
  long long ld16, ld_out16;
  int32_t* status;
};

// kOne: the whole block fits one chunk (l_b <= kSelThreads * kItems, every C1..C4 shape):
// each thread loads its 16 scores once and keeps them in registers for all five passes
// (count, three radix digits, emission) instead of re-reading them from L2 every pass.
template <int kSelThreads, bool kOne>
__global__ void __launch_bounds__(kSelThreads) select_kernel(const __grid_constant__ SelJobs J) {
  constexpr int kChunk = kSelThreads * kItems;
  constexpr int kWarps = kSelThreads / 32;
  const SelJob& jb = J.j[blockIdx.x];
  const float* __restrict__ scores = jb.scores;
  const int l_b = J.l_b, l_p = J.l_p, global_offset = jb.global_offset;
  int32_t* __restrict__ idx = jb.idx;
  int32_t* __restrict__ count = jb.count;
  int32_t* __restrict__ status = J.status;
  __shared__ int hist[2048];
  __shared__ int red[kWarps + 1];
  __shared__ uint32_t sh_prefix;
  __shared__ int sh_need;
  const int tid = threadIdx.x;
  float vk[kItems];  // kOne: this thread's scores for every pass
  if (kOne) load_items(scores, l_b, 0, vk);
  auto items = [&](int base, float (&v)[kItems]) {
    if (kOne) {
#pragma unroll
      for (int t = 0; t < kItems; ++t) v[t] = vk[t];
    } else {
      load_items(scores, l_b, base, v);
    }
  };
  // ---- 1. counts
  int fin = 0, bad = 0;
  for (int base = 0; base < l_b; base += kChunk) {
    float v[kItems];
    items(base, v);
#pragma unroll
    for (int t = 0; t < kItems; ++t) {
      fin += isfinite(v[t]) ? 1 : 0;
      bad += (isnan(v[t]) || (isinf(v[t]) && v[t] > 0.f)) ? 1 : 0;
    }
  }
  int tot_fin, tot_bad;
  block_excl<kWarps>(fin, red, &tot_fin);
  block_excl<kWarps>(bad, red, &tot_bad);
  const int k = tot_bad > 0 ? 0 : min(l_p, tot_fin);
  if (tot_bad > 0 && tid == 0 && status) {
    // NaN is invalid input; +inf sorts first and stops the selection at once
    bool nan = false;
    for (int j = 0; j < l_b && !nan; ++j) nan = isnan(scores[j]);
    if (nan) atomicOr(status, 1);
  }
  if (k == 0) {
    for (int r = tid; r < l_p; r += kSelThreads) idx[r] = -1;
    if (tid == 0) {
      *count = 0;
      if (jb.require_full && l_p > 0 && status) atomicOr(status, 2);
    }
    return;
  }
  // ---- 2. radix select: digits [31:21], [20:10], [9:0]
  uint32_t prefix = 0, mask = 0;
  int need = k;
  const int shifts[3] = {21, 10, 0};
  const int bits[3] = {11, 11, 10};
#pragma unroll 1
  for (int pass = 0; pass < 3; ++pass) {
    const int shift = shifts[pass], nb = 1 << bits[pass];
    for (int b = tid; b < nb; b += kSelThreads) hist[b] = 0;
    __syncthreads();
    for (int base = 0; base < l_b; base += kChunk) {
      float v[kItems];
      items(base, v);
#pragma unroll
      for (int t = 0; t < kItems; ++t) {
        const uint32_t key = order_key(v[t]);
        const bool ok = isfinite(v[t]) && ((key & mask) == prefix);
        const unsigned digit = (key >> shift) & static_cast<unsigned>(nb - 1);
        const unsigned active = __ballot_sync(0xffffffffu, ok);
        if (ok) {
          const unsigned peers = __match_any_sync(active, digit);
          if ((__ffs(peers) - 1) == (tid & 31)) atomicAdd(&hist[digit], __popc(peers));
        }
      }
    }
    __syncthreads();
    // bucket holding the need-th largest: descending suffix scan (2 buckets / thread)
    const int per = nb / kSelThreads;  // buckets per thread
    int c = 0;
    for (int u = 0; u < per; ++u) c += hist[nb - 1 - (tid * per + u)];
    int tot;
    const int before = block_excl<kWarps>(c, red, &tot);  // keys in buckets above this thread's
    if (before < need && before + c >= need) {
      int cum = before;
      for (int u = 0; u < per; ++u) {
        const int b = nb - 1 - (tid * per + u);
        if (cum + hist[b] >= need) {
          sh_prefix = prefix | (static_cast<uint32_t>(b) << shift);
          sh_need = need - cum;
          break;
        }
        cum += hist[b];
      }
    }
    __syncthreads();
    prefix = sh_prefix;
    need = sh_need;
    mask |= static_cast<uint32_t>(nb - 1) << shift;
  }
  const uint32_t T = prefix;  // key of the k-th largest; `need` keys == T are taken
  // ---- 3. index-ordered emission
  int eq_base = 0, out_base = 0;
  for (int base = 0; base < l_b; base += kChunk) {
    float v[kItems];
    items(base, v);
    int n_eq = 0;
#pragma unroll
    for (int t = 0; t < kItems; ++t) n_eq += (isfinite(v[t]) && order_key(v[t]) == T) ? 1 : 0;
    int eq_tot;
    int eq_rank = eq_base + block_excl<kWarps>(n_eq, red, &eq_tot);
    int flags = 0, n_sel = 0;
#pragma unroll
    for (int t = 0; t < kItems; ++t) {
      const bool f = isfinite(v[t]);
      const uint32_t key = order_key(v[t]);
      bool sel = f && key > T;
      if (f && key == T) {
        sel = eq_rank < need;
        ++eq_rank;
      }
      if (sel) {
        flags |= 1 << t;
        ++n_sel;
      }
    }
    int sel_tot;
    int pos = out_base + block_excl<kWarps>(n_sel, red, &sel_tot);
    const int j0 = base + tid * kItems;
#pragma unroll
    for (int t = 0; t < kItems; ++t)
      if (flags & (1 << t)) idx[pos++] = global_offset + j0 + t;
    eq_base += eq_tot;
    out_base += sel_tot;
  }
  for (int r = out_base + tid; r < l_p; r += kSelThreads) idx[r] = -1;  // defined tail
  if (tid == 0) {
    *count = out_base;
    // the exchange slot is fixed-size (l_p rows): a short selection would be attended as
    // zero rows where the reference drops them (approx.cpp:83-90), so it is an error here
    if (jb.require_full && out_base < l_p && status) atomicOr(status, 2);
  }
}

// warp per selected row; rows >= count are zero-filled so the slot is well defined.
// Peer fabric: the same rows (and the slot's index list / count) are also stored straight
// into every peer GPU's exchange slot over NVLink -- the pass round is this kernel's
// epilogue, no separate collective.
__global__ void gather_kernel(const __grid_constant__ SelJobs J) {
  const SelJob& jb = J.j[blockIdx.y];
  const int r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r < J.l_p) {  // (no early exit: the peer flag raise below synchronises the CTA)
    const int n = *jb.count;
    const int32_t* idx = jb.idx;
    const PeerSlots& peers = jb.peers;
    const long long o = r * J.ld_out16;
    if (lane == 0)
      for (int q = 0; q < peers.n; ++q) {
        static_cast<int32_t*>(peers.idx[q])[r] = idx[r];
        if (r == 0) *static_cast<int32_t*>(peers.cnt[q]) = n;
      }
    const long long src = r < n ? static_cast<long long>(idx[r] - jb.global_offset) * J.ld16 : 0;
    for (int c = lane; c < J.w16; c += 32) {
      const uint4 kx = r < n ? jb.k[src + c] : make_uint4(0, 0, 0, 0);
      const uint4 vx = r < n ? jb.v[src + c] : make_uint4(0, 0, 0, 0);
      jb.k_out[o + c] = kx;
      jb.v_out[o + c] = vx;
      for (int q = 0; q < peers.n; ++q) {
        static_cast<uint4*>(peers.k[q])[o + c] = kx;
        static_cast<uint4*>(peers.v[q])[o + c] = vx;
      }
    }
  }
  // peer fabric: the last CTA of this block's round raises arrive[round][me] in every peer
  raise_when_done(jb.fr, gridDim.x);
}

}  // namespace

cudaError_t launch_select_pack_n(const SelectPackJob* jobs, int n, int l_b, int l_p, long long ld, int width,
                                 long long ld_out, int32_t* status, cudaStream_t stream) {
  if (n < 1 || n > 2 || l_p < 0 || l_p > l_b || (width % 8) || (ld % 8) || (ld_out % 8))
    return cudaErrorInvalidValue;
  SelJobs J{};
  J.l_b = l_b;
  J.l_p = l_p;
  J.w16 = width / 8;
  J.ld16 = ld / 8;
  J.ld_out16 = ld_out / 8;
  J.status = status;
  bool gather = l_p > 0;
  for (int i = 0; i < n; ++i) {
    const SelectPackJob& s = jobs[i];
    if (s.peers && (s.peers->n < 0 || s.peers->n > kMaxPeers)) return cudaErrorInvalidValue;
    SelJob& j = J.j[i];
    j.scores = s.scores;
    j.global_offset = s.global_offset;
    j.idx = s.idx;
    j.count = s.count;
    j.k = static_cast<const uint4*>(s.k);
    j.v = static_cast<const uint4*>(s.v);
    j.k_out = static_cast<uint4*>(s.k_out);
    j.v_out = static_cast<uint4*>(s.v_out);
    if (s.peers) j.peers = *s.peers;
    j.fr = s.fr;
    j.require_full = s.require_full;
    gather = gather && s.k_out && s.v_out;
    if (!(l_p > 0 && s.k_out && s.v_out) && (j.peers.n > 0 || j.fr.n > 0))
      return cudaErrorInvalidValue;  // a peer slot is only published through the gather
    if (j.fr.n < 0 || j.fr.n > kMaxPeers || (j.fr.n > 0 && !j.fr.counter)) return cudaErrorInvalidValue;
  }
  if (l_b <= kSelSmall * kItems)
    select_kernel<kSelSmall, true><<<n, kSelSmall, 0, stream>>>(J);
  else if (l_b <= kSelBig * kItems)
    select_kernel<kSelBig, true><<<n, kSelBig, 0, stream>>>(J);
  else
    select_kernel<kSelBig, false><<<n, kSelBig, 0, stream>>>(J);
  if (gather) gather_kernel<<<dim3((l_p + 7) / 8, n), 256, 0, stream>>>(J);
  return cudaGetLastError();
}

cudaError_t launch_select_pack(const float* scores, int l_b, int l_p, int global_offset,
                               const void* k, const void* v, long long ld, int width, int32_t* idx,
                               void* k_out, void* v_out, long long ld_out, int32_t* count,
                               int32_t* status, cudaStream_t stream, const PeerSlots* peers) {
  const SelectPackJob job{scores, global_offset, k, v, idx, k_out, v_out, count, peers};
  return launch_select_pack_n(&job, 1, l_b, l_p, ld, width, ld_out, status, stream);
}

}  // namespace spava
