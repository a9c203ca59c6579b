// merge.cu -- exact lse merge of attention partials over disjoint key sets.
//
// merge_partials / mha_merge (attention.cpp:88-119, 180-197), same arithmetic order:
// per (row, head): mx = max over valid parts of double(lse_p); denom = sum_p
// exp(lse_p - mx) (fp64, part order); w_p = float(exp(lse_p - mx)/denom);
// out = sum_p w_p * out_p (fp32, part order).  A part is valid where its lse is finite;
// a row invalid in every part is an error in the reference -> zero row + status flag.
// Used twice per layer: to combine the split-KV partials of one host's query attention
// (also emitting the merged lse, mx + log(denom)), and to merge the H hosts' query
// partials in host order after the qpartial exchange.
// One CTA per (row, head): warp 0 computes the part weights once into smem, then every
// thread produces one output column.
#include <cuda_bf16.h>

#include "fabric_dev.cuh"
#include "spava_internal.h"

namespace spava {

namespace {

// kMinB: blocks per SM the register budget must allow.  The dh = 128 instance asks for 16
// so a (128 rows x 16 heads) query merge -- 2048 CTAs -- runs in one wave (at the default
// 38 registers only 12 CTAs fit per SM: 1.15 waves, the second one nearly empty).
template <int kMaxT, int kMinB>
__global__ void __launch_bounds__(kMaxT, kMinB) merge_kernel(const __grid_constant__ MergeParams p) {
  __shared__ float w[kMaxMergeParts];
  __shared__ int ok_sh;
  __shared__ float lse_sh;
  const int i = blockIdx.x, h = blockIdx.y, c = threadIdx.x;
  if (threadIdx.x < 32) {
    merge_weights_warp(p, i, h, w, &ok_sh, &lse_sh);
    __syncwarp();  // lane 0 wrote ok_sh
    if (threadIdx.x == 0 && !ok_sh && p.status) atomicOr(p.status, 4);
  }
  __syncthreads();
  const long long col = static_cast<long long>(h) * p.dh + c;
  const float acc = ok_sh ? merge_column(p, w, i, col) : 0.f;
  merge_store(p, i, col, acc);
  if (p.dst_lse && c == 0) p.dst_lse[static_cast<long long>(i) * p.hq + h] = lse_sh;
  // peer fabric: the qpartial round is this kernel's epilogue (NVLink stores into every
  // peer's slot, then the last CTA raises the round's arrive flags); only the f32 slot
  // layout is ever published
  const long long d = static_cast<long long>(i) * p.ld_dst + col;
  for (int q = 0; q < p.npeer; ++q) {
    static_cast<float*>(p.peer_dst[q])[d] = acc;
    if (c == 0) p.peer_lse[q][static_cast<long long>(i) * p.hq + h] = lse_sh;
  }
  raise_when_done(p.fr, gridDim.x * gridDim.y);
}

}  // namespace

cudaError_t launch_merge(const MergeParams& p, cudaStream_t stream) {
  if (p.nparts < 1 || p.nparts > kMaxMergeParts || p.dh < 32 || p.dh > 1024) return cudaErrorInvalidValue;
  if (p.npeer < 0 || p.npeer > kMaxPeers || (p.npeer > 0 && (!p.dst_f32 || !p.dst_lse)))
    return cudaErrorInvalidValue;
  if (p.fr.n < 0 || p.fr.n > kMaxPeers || (p.fr.n > 0 && (!p.fr.counter || p.rows == 0)))
    return cudaErrorInvalidValue;
  if (p.rows == 0) return cudaSuccess;
  if (p.dh == 128)
    merge_kernel<128, 16><<<dim3(p.rows, p.hq), p.dh, 0, stream>>>(p);
  else
    merge_kernel<1024, 1><<<dim3(p.rows, p.hq), p.dh, 0, stream>>>(p);
  return cudaGetLastError();
}

// DelayInjection analogue (simhost.hpp:51-55, simhost.cpp:139-147): one thread spins on
// %globaltimer so a stream reaches its next operation late (schedule-independence tests).
__global__ void delay_kernel(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

cudaError_t launch_delay(unsigned long long ns, cudaStream_t stream) {
  if (ns == 0) return cudaSuccess;
  delay_kernel<<<1, 1, 0, stream>>>(ns);
  return cudaGetLastError();
}

}  // namespace spava
