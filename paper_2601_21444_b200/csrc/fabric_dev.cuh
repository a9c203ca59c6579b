// fabric_dev.cuh -- device side of the peer (NVLink P2P) exchange, shared by the kernels
// that produce or consume a round in their own epilogue / prologue.
//
//   raise_when_done  producer epilogue: after every CTA of a group has stored its part of a
//                    slot into the peers' buffers, the last CTA raises arrive[round][me] in
//                    every peer (system-scope release) -- no separate flag kernel.
//   wait_flags_geq   consumer prologue: spin (acquire, system scope) until every listed
//                    flag reached the epoch; 8 s %globaltimer watchdog traps instead of
//                    hanging.
//   merge_*          mha_merge / merge_partials (attention.cpp:88-119, 180-197) for one
//                    (row, head), same arithmetic order as merge_kernel (one code path, so
//                    the receive-side merge inside the stage launch is bit-identical).
#pragma once

#include <cuda_bf16.h>

#include "spava_internal.h"

namespace spava {

__device__ __forceinline__ void raise_when_done(const FlagRaise& f, unsigned group_ctas) {
  if (f.n == 0) return;
  __threadfence_system();  // this thread's peer stores, before the CTA's arrival
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(f.counter, 1u) == group_ctas - 1) {
    __threadfence_system();  // every CTA's stores (observed through the counter) first
    for (int q = 0; q < f.n; ++q)
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f.addr[q]), "r"(f.value) : "memory");
    atomicExch(f.counter, 0u);  // ready for the next launch (stream order)
  }
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// one thread spins; the caller synchronises the CTA afterwards
__device__ __forceinline__ void wait_flags_geq(const uint32_t* const* flags, int n, uint32_t epoch) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int q = 0; q < n; ++q) {
    while (static_cast<int32_t>(ld_acquire_sys(flags[q]) - epoch) < 0) {
      __nanosleep(200);
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 8000000000ull) __trap();
    }
  }
}

// Part weights of (row i, head h), computed by one full warp: lanes own parts lane, lane+32.
// w[q] = float(exp(lse_q - mx) / denom) (0 for an invalid part), denominator in part order.
__device__ __forceinline__ void merge_weights_warp(const MergeParams& p, int i, int h, float* w, int* ok_out,
                                                   float* lse_out) {
  const int lane = threadIdx.x & 31;
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
  double denom = 0.0;  // part order (the reference adds parts sequentially)
  for (int q = 0; q < p.nparts; ++q) {
    const double eq = __shfl_sync(0xffffffffu, q < 32 ? e0 : e1, q & 31);
    denom = __dadd_rn(denom, eq);
  }
  if (lane < p.nparts) w[lane] = ok && isfinite(l0) ? __double2float_rn(__ddiv_rn(e0, denom)) : 0.f;
  if (lane + 32 < p.nparts) w[lane + 32] = ok && isfinite(l1) ? __double2float_rn(__ddiv_rn(e1, denom)) : 0.f;
  if (lane == 0) {
    *ok_out = ok;
    *lse_out = ok ? __double2float_rn(mx + log(denom)) : -INFINITY;
  }
}

// out[i, col] = sum_q w_q * out_q[i, col], fp32, part order (invalid parts skipped)
__device__ __forceinline__ float merge_column(const MergeParams& p, const float* w, int i, long long col) {
  float acc = 0.f;
  for (int q = 0; q < p.nparts; ++q) {
    const float wq = w[q];
    if (wq == 0.f) continue;  // invalid part (weights of valid parts are > 0 or underflow)
    acc = __fadd_rn(acc, __fmul_rn(wq, p.out[q][static_cast<long long>(i) * p.ld_part + col]));
  }
  return acc;
}

__device__ __forceinline__ void merge_store(const MergeParams& p, int i, long long col, float acc) {
  const long long d = static_cast<long long>(i) * p.ld_dst + col;
  if (p.dst_f32)
    static_cast<float*>(p.dst)[d] = acc;
  else
    static_cast<__nv_bfloat16*>(p.dst)[d] = __float2bfloat16_rn(acc);
}

// Receive-side merge inside another launch (the stage attention grid's trailing CTAs):
// CTA `c` of `ctas` waits for every peer's qpartial, then merges its share of the (row,
// head) pairs, one warp per pair.  `w` = nwarps * kMaxMergeParts floats of shared memory.
__device__ __forceinline__ void merge_job(const MergeJob& J, int c, float* w_smem) {
  if (threadIdx.x == 0) wait_flags_geq(J.wait, J.nwait, J.epoch);
  __syncthreads();
  const MergeParams& p = J.mp;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  float* w = w_smem + warp * kMaxMergeParts;
  __shared__ int ok_sh[32];
  __shared__ float lse_sh[32];
  for (int pair = c * nw + warp; pair < p.rows * p.hq; pair += J.ctas * nw) {
    const int i = pair / p.hq, h = pair % p.hq;
    merge_weights_warp(p, i, h, w, &ok_sh[warp], &lse_sh[warp]);
    __syncwarp();
    const bool ok = ok_sh[warp];
    if (!ok && lane == 0 && p.status) atomicOr(p.status, 4);
    for (int cc = lane; cc < p.dh; cc += 32) {
      const long long col = static_cast<long long>(h) * p.dh + cc;
      merge_store(p, i, col, ok ? merge_column(p, w, i, col) : 0.f);
    }
    if (p.dst_lse && lane == 0) p.dst_lse[static_cast<long long>(i) * p.hq + h] = lse_sh[warp];
    __syncwarp();
  }
}

}  // namespace spava
