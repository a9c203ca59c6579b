// merge.cu -- exact lse merge of attention partials over disjoint key sets.
//
// merge_partials / mha_merge (attention.cpp:88-119, 180-197), same arithmetic order:
// per (row, head): mx = max over valid parts of double(lse_p); denom = sum_p
// exp(lse_p - mx) (fp64); w_p = float(exp(lse_p - mx)/denom); out = sum_p w_p * out_p
// (fp32, part order).  A part is valid where its lse is finite; a row invalid in every
// part is an error in the reference -> zero row + status flag here.
// Used twice per layer: to combine the split-KV partials of one host's query attention
// (also emitting the merged lse, mx + log(denom)), and to merge the H hosts' query
// partials in host order after the qpartial exchange.
#include <cuda_bf16.h>

#include "spava_internal.h"

namespace spava {

namespace {

// grid (rows, hq), block dh threads (one output column each)
__global__ void merge_kernel(const __grid_constant__ MergeParams p) {
  const int i = blockIdx.x, h = blockIdx.y, c = threadIdx.x;
  double mx = -INFINITY;
  for (int q = 0; q < p.nparts; ++q) {
    const float l = p.lse[q][static_cast<long long>(i) * p.ld_lse + h];
    if (isfinite(l)) mx = fmax(mx, static_cast<double>(l));
  }
  const long long col = static_cast<long long>(h) * p.dh + c;
  float acc = 0.f;
  double denom = 0.0;
  const bool ok = isfinite(mx);
  if (ok) {
    for (int q = 0; q < p.nparts; ++q) {
      const float l = p.lse[q][static_cast<long long>(i) * p.ld_lse + h];
      if (isfinite(l)) denom = __dadd_rn(denom, exp(__dsub_rn(static_cast<double>(l), mx)));
    }
    for (int q = 0; q < p.nparts; ++q) {
      const float l = p.lse[q][static_cast<long long>(i) * p.ld_lse + h];
      if (!isfinite(l)) continue;
      const float w = __double2float_rn(__ddiv_rn(exp(__dsub_rn(static_cast<double>(l), mx)), denom));
      acc = __fadd_rn(acc, __fmul_rn(w, p.out[q][static_cast<long long>(i) * p.ld_part + col]));
    }
  } else if (p.status && c == 0) {
    atomicExch(p.status, 1);
  }
  const long long d = static_cast<long long>(i) * p.ld_dst + col;
  if (p.dst_f32)
    static_cast<float*>(p.dst)[d] = acc;
  else
    static_cast<__nv_bfloat16*>(p.dst)[d] = __float2bfloat16_rn(acc);
  if (p.dst_lse && c == 0)
    p.dst_lse[static_cast<long long>(i) * p.hq + h] =
        ok ? __double2float_rn(mx + log(denom)) : -INFINITY;
}

}  // namespace

cudaError_t launch_merge(const MergeParams& p, cudaStream_t stream) {
  if (p.nparts < 1 || p.nparts > kMaxMergeParts || p.dh < 1 || p.dh > 1024) return cudaErrorInvalidValue;
  if (p.rows == 0) return cudaSuccess;
  merge_kernel<<<dim3(p.rows, p.hq), p.dh, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace spava
