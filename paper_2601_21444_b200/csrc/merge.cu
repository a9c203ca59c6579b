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

#include "spava_internal.h"

namespace spava {

namespace {

__global__ void merge_kernel(const __grid_constant__ MergeParams p) {
  __shared__ float w[kMaxMergeParts];
  __shared__ int ok_sh;
  __shared__ float lse_sh;
  const int i = blockIdx.x, h = blockIdx.y, c = threadIdx.x;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    // lanes own parts lane, lane+32 (kMaxMergeParts = 64)
    float l0 = -INFINITY, l1 = -INFINITY;
    if (lane < p.nparts) l0 = p.lse[lane][static_cast<long long>(i) * p.ld_lse + h];
    if (lane + 32 < p.nparts) l1 = p.lse[lane + 32][static_cast<long long>(i) * p.ld_lse + h];
    double mx = -INFINITY;
    if (isfinite(l0)) mx = static_cast<double>(l0);
    if (isfinite(l1)) mx = fmax(mx, static_cast<double>(l1));
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const bool ok = isfinite(mx);
    double e0 = 0.0, e1 = 0.0;
    if (ok) {
      if (isfinite(l0)) e0 = exp(__dsub_rn(static_cast<double>(l0), mx));
      if (isfinite(l1)) e1 = exp(__dsub_rn(static_cast<double>(l1), mx));
    }
    // denominator in part order (reference adds parts sequentially)
    double denom = 0.0;
    for (int q = 0; q < p.nparts; ++q) {
      const double eq = __shfl_sync(0xffffffffu, q < 32 ? e0 : e1, q & 31);
      denom = __dadd_rn(denom, eq);
    }
    if (lane < p.nparts) w[lane] = ok && isfinite(l0) ? __double2float_rn(__ddiv_rn(e0, denom)) : 0.f;
    if (lane + 32 < p.nparts) w[lane + 32] = ok && isfinite(l1) ? __double2float_rn(__ddiv_rn(e1, denom)) : 0.f;
    if (lane == 0) {
      ok_sh = ok;
      lse_sh = ok ? __double2float_rn(mx + log(denom)) : -INFINITY;
      if (!ok && p.status) atomicOr(p.status, 4);
    }
  }
  __syncthreads();
  const long long col = static_cast<long long>(h) * p.dh + c;
  float acc = 0.f;
  if (ok_sh) {
    for (int q = 0; q < p.nparts; ++q) {
      const float wq = w[q];
      if (wq == 0.f) continue;  // invalid part (weights of valid parts are > 0 or underflow)
      acc = __fadd_rn(acc, __fmul_rn(wq, p.out[q][static_cast<long long>(i) * p.ld_part + col]));
    }
  }
  const long long d = static_cast<long long>(i) * p.ld_dst + col;
  if (p.dst_f32)
    static_cast<float*>(p.dst)[d] = acc;
  else
    static_cast<__nv_bfloat16*>(p.dst)[d] = __float2bfloat16_rn(acc);
  if (p.dst_lse && c == 0) p.dst_lse[static_cast<long long>(i) * p.hq + h] = lse_sh;
  // peer fabric: the qpartial round is this kernel's epilogue (NVLink stores into every
  // peer's slot); only the f32 slot layout is ever published
  for (int q = 0; q < p.npeer; ++q) {
    static_cast<float*>(p.peer_dst[q])[d] = acc;
    if (c == 0) p.peer_lse[q][static_cast<long long>(i) * p.hq + h] = lse_sh;
  }
}

}  // namespace

cudaError_t launch_merge(const MergeParams& p, cudaStream_t stream) {
  if (p.nparts < 1 || p.nparts > kMaxMergeParts || p.dh < 32 || p.dh > 1024) return cudaErrorInvalidValue;
  if (p.npeer < 0 || p.npeer > kMaxPeers || (p.npeer > 0 && (!p.dst_f32 || !p.dst_lse)))
    return cudaErrorInvalidValue;
  if (p.rows == 0) return cudaSuccess;
  merge_kernel<<<dim3(p.rows, p.hq), p.dh, 0, stream>>>(p);
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
