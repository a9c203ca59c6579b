// select.cu -- essential-KV selection and packing (the compressor's back half).
//
// select_essential (approx.cpp:71-102): stable descending sort of the block's scores
// (ties -> lower index), take at most l_p stopping at the first non-finite, return the
// chosen indices ascending (+ global offset) and gather their K/V rows.
// GPU form, no sort at all:
//   1. one CTA counts finite scores (k = min(l_p, #finite); any +inf sorts first and
//      ends the selection immediately, NaN is rejected),
//   2. 4-pass MSB radix select over order-preserving uint32 keys finds the k-th largest
//      key T and how many of the keys equal to T are taken,
//   3. an index-ordered block scan emits key > T, plus the lowest-index keys == T
//      (exactly the stable-sort tie rule), already ascending,
// then a multi-CTA gather copies the selected K/V rows (16 B per lane, coalesced)
// straight into the exchange buffer slot of this host.
#include <cuda_bf16.h>

#include "spava_internal.h"

namespace spava {

namespace {

constexpr int kSelThreads = 1024;

__device__ __forceinline__ uint32_t order_key(float s) {
  const uint32_t u = __float_as_uint(s);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ int block_sum(int v, int* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  int t = 0;
  for (int i = 0; i < kSelThreads / 32; ++i) t += red[i];
  return t;
}

// exclusive prefix of a per-thread flag across the block (index order = thread order);
// returns the prefix, *total receives the block total.
__device__ __forceinline__ int block_excl_scan(int flag, int* red, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(0xffffffffu, flag);
  const int in_warp = __popc(b & ((1u << lane) - 1u));
  __syncthreads();
  if (lane == 0) red[w] = __popc(b);
  __syncthreads();
  int before = 0, tot = 0;
  for (int i = 0; i < kSelThreads / 32; ++i) {
    const int c = red[i];
    if (i < w) before += c;
    tot += c;
  }
  *total = tot;
  return before + in_warp;
}

__global__ void __launch_bounds__(kSelThreads) select_kernel(const float* __restrict__ scores,
                                                             int l_b, int l_p, int global_offset,
                                                             int32_t* __restrict__ idx,
                                                             int32_t* __restrict__ count,
                                                             int32_t* __restrict__ status) {
  __shared__ int hist[256];
  __shared__ int red[kSelThreads / 32];
  __shared__ uint32_t sh_prefix;
  __shared__ int sh_take;
  const int tid = threadIdx.x;
  int fin = 0, pinf = 0, nan = 0;
  for (int j = tid; j < l_b; j += kSelThreads) {
    const float s = scores[j];
    fin += isfinite(s) ? 1 : 0;
    pinf += (isinf(s) && s > 0.f) ? 1 : 0;
    nan += isnan(s) ? 1 : 0;
  }
  fin = block_sum(fin, red);
  pinf = block_sum(pinf, red);
  nan = block_sum(nan, red);
  int k = (pinf > 0 || nan > 0) ? 0 : min(l_p, fin);
  if (nan > 0 && tid == 0 && status) atomicExch(status, 1);
  if (k == 0) {
    if (tid == 0) *count = 0;
    return;
  }
  // ---- radix select: the k-th largest key
  uint32_t prefix = 0, mask = 0;
  int need = k;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int b = tid; b < 256; b += kSelThreads) hist[b] = 0;
    __syncthreads();
    for (int base = 0; base < l_b; base += kSelThreads) {  // warp-uniform trip count
      const int j = base + tid;
      const float s = j < l_b ? scores[j] : -INFINITY;
      bool ok = isfinite(s);
      const uint32_t key = order_key(s);
      ok = ok && ((key & mask) == prefix);
      const unsigned digit = (key >> shift) & 255u;
      // warp-aggregated histogram update (scores cluster in few buckets)
      const unsigned active = __ballot_sync(0xffffffffu, ok);
      if (ok) {
        const unsigned peers = __match_any_sync(active, digit);
        if ((__ffs(peers) - 1) == static_cast<int>(threadIdx.x & 31))
          atomicAdd(&hist[digit], __popc(peers));
      }
    }
    __syncthreads();
    if (tid == 0) {
      int cum = 0;
      for (int b = 255; b >= 0; --b) {
        if (cum + hist[b] >= need) {
          sh_prefix = prefix | (static_cast<uint32_t>(b) << shift);
          sh_take = need - cum;
          break;
        }
        cum += hist[b];
      }
    }
    __syncthreads();
    prefix = sh_prefix;
    need = sh_take;
    mask |= 255u << shift;
  }
  const uint32_t T = prefix;  // key of the k-th largest; `need` keys == T are taken
  // ---- index-ordered emission
  int eq_base = 0, out_base = 0;
  for (int base = 0; base < l_b; base += kSelThreads) {
    const int j = base + tid;
    bool fin_j = false;
    uint32_t key = 0;
    if (j < l_b) {
      const float s = scores[j];
      fin_j = isfinite(s);
      key = order_key(s);
    }
    const int is_eq = (fin_j && key == T) ? 1 : 0;
    int eq_tot;
    const int eq_rank = block_excl_scan(is_eq, red, &eq_tot);
    const int sel = (fin_j && (key > T || (is_eq && eq_base + eq_rank < need))) ? 1 : 0;
    int sel_tot;
    const int pos = block_excl_scan(sel, red, &sel_tot);
    if (sel) idx[out_base + pos] = global_offset + j;
    eq_base += eq_tot;
    out_base += sel_tot;
  }
  if (tid == 0) *count = out_base;
}

// warp per selected row; rows >= count are zero-filled so the slot is well defined.
__global__ void gather_kernel(const int32_t* __restrict__ idx, const int32_t* __restrict__ count,
                              int global_offset, int l_p, const uint4* __restrict__ k,
                              const uint4* __restrict__ v, long long ld16, int w16,
                              uint4* __restrict__ k_out, uint4* __restrict__ v_out,
                              long long ld_out16) {
  const int r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= l_p) return;
  const int n = *count;
  uint4* ko = k_out + r * ld_out16;
  uint4* vo = v_out + r * ld_out16;
  if (r < n) {
    const long long src = static_cast<long long>(idx[r] - global_offset) * ld16;
    for (int c = lane; c < w16; c += 32) {
      ko[c] = k[src + c];
      vo[c] = v[src + c];
    }
  } else {
    for (int c = lane; c < w16; c += 32) {
      ko[c] = make_uint4(0, 0, 0, 0);
      vo[c] = make_uint4(0, 0, 0, 0);
    }
  }
}

}  // namespace

cudaError_t launch_select_pack(const float* scores, int l_b, int l_p, int global_offset,
                               const void* k, const void* v, long long ld, int width, int32_t* idx,
                               void* k_out, void* v_out, long long ld_out, int32_t* count,
                               int32_t* status, cudaStream_t stream) {
  if (l_p < 0 || l_p > l_b || (width % 8) || (ld % 8) || (ld_out % 8)) return cudaErrorInvalidValue;
  select_kernel<<<1, kSelThreads, 0, stream>>>(scores, l_b, l_p, global_offset, idx, count, status);
  if (l_p > 0 && k_out && v_out) {
    gather_kernel<<<(l_p + 7) / 8, 256, 0, stream>>>(
        idx, count, global_offset, l_p, static_cast<const uint4*>(k), static_cast<const uint4*>(v),
        ld / 8, width / 8, static_cast<uint4*>(k_out), static_cast<uint4*>(v_out), ld_out / 8);
  }
  return cudaGetLastError();
}

}  // namespace spava
