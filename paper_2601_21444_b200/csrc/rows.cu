// rows.cu -- split_context on the device (partition.cpp:40-85) and its inverse.
//
// The global sequence is [E_v (n_v rows) | E_Q (n_t rows)], token-major, row_bytes per row.
// Physical host h owns the virtual pair (lo, hi) (zigzag_map / naive_map, partition.cpp:
// 21-29); its host-local buffer is [anchor E_v[0,l_a) | block lo | block hi | E_Q], where
// block v = E_v rows [l_a + v*l_b, l_a + (v+1)*l_b) zero-padded at the tail
// (partition.cpp:64-79).  split_rows gathers that buffer from the global rows; merge_rows
// writes a host's block outputs back to their global positions (non-pad rows only) and,
// for the host that owns the shared rows, the anchor and query rows.  Pure HBM copies:
// one CTA per 8 destination rows, 16-byte vectors, coalesced.
#include "spava_internal.h"

namespace spava {

namespace {

struct RowMap {
  int l_a, l_b, n_t, n_v, lo, hi;
};

// host-local row r -> global row, or -1 for a pad row
__device__ __forceinline__ long long global_row(const RowMap& m, int r) {
  if (r < m.l_a) return r;
  r -= m.l_a;
  if (r < 2 * m.l_b) {
    const int v = r < m.l_b ? m.lo : m.hi;
    const long long g = static_cast<long long>(m.l_a) + static_cast<long long>(v) * m.l_b + (r % m.l_b);
    return g < m.n_v ? g : -1;
  }
  return static_cast<long long>(m.n_v) + (r - 2 * m.l_b);
}

__global__ void split_rows_kernel(RowMap m, const uint8_t* src, long long ld_src, uint8_t* dst,
                                  long long ld_dst, int vec16, int rows) {
  const int r = blockIdx.x * 8 + threadIdx.y;
  if (r >= rows) return;
  const long long g = global_row(m, r);
  uint4* d = reinterpret_cast<uint4*>(dst + r * ld_dst);
  const uint4* s = g >= 0 ? reinterpret_cast<const uint4*>(src + g * ld_src) : nullptr;
  for (int i = threadIdx.x; i < vec16; i += 32) d[i] = s ? s[i] : make_uint4(0u, 0u, 0u, 0u);
}

__global__ void merge_rows_kernel(RowMap m, const uint8_t* src, long long ld_src, uint8_t* dst,
                                  long long ld_dst, int vec16, int rows, int shared) {
  const int r = blockIdx.x * 8 + threadIdx.y;
  if (r >= rows) return;
  const bool block_row = r >= m.l_a && r < m.l_a + 2 * m.l_b;
  if (!block_row && !shared) return;
  const long long g = global_row(m, r);
  if (g < 0) return;
  const uint4* s = reinterpret_cast<const uint4*>(src + r * ld_src);
  uint4* d = reinterpret_cast<uint4*>(dst + g * ld_dst);
  for (int i = threadIdx.x; i < vec16; i += 32) d[i] = s[i];
}

// Frame-parallel encode gather fused with split_context (simhost.cpp:280-302 then
// partition.cpp:40-85): E_v is not materialised on any GPU -- rank q holds global E_v rows
// [off[q], off[q+1]) (its frame_partition share, in frame order) and each destination row
// is read straight from the owning rank's buffer (an NVLink peer load for the peer
// fabric).  Every host moves only its l_a + 2*l_b rows instead of the n_v-row AllGather.
__global__ void gather_split_kernel(RowMap m, const __grid_constant__ GatherParts parts,
                                    const uint8_t* eq, long long ld_q, uint8_t* dst, long long ld_dst,
                                    int vec16, int rows) {
  const int r = blockIdx.x * 8 + threadIdx.y;
  if (r >= rows) return;
  const long long g = global_row(m, r);
  const uint4* s = nullptr;
  if (g >= m.n_v) {
    s = reinterpret_cast<const uint4*>(eq + (g - m.n_v) * ld_q);
  } else if (g >= 0) {
    int q = 0;
    while (q + 1 < parts.n && g >= parts.off[q + 1]) ++q;
    s = reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(parts.base[q]) + (g - parts.off[q]) * parts.ld);
  }
  uint4* d = reinterpret_cast<uint4*>(dst + r * ld_dst);
  for (int i = threadIdx.x; i < vec16; i += 32) d[i] = s ? s[i] : make_uint4(0u, 0u, 0u, 0u);
}

}  // namespace

cudaError_t launch_gather_split(int l_a, int l_b, int n_t, int n_v, int lo, int hi, const GatherParts& parts,
                                const void* eq, long long ld_q, void* dst, long long ld_dst, int row_bytes,
                                cudaStream_t stream) {
  if (row_bytes % 16 || ld_q % 16 || ld_dst % 16 || parts.ld % 16 || parts.n < 1 || parts.n > kMaxPeers + 1 ||
      (reinterpret_cast<uintptr_t>(eq) | reinterpret_cast<uintptr_t>(dst)) % 16)
    return cudaErrorInvalidValue;
  for (int q = 0; q < parts.n; ++q)
    if (reinterpret_cast<uintptr_t>(parts.base[q]) % 16) return cudaErrorInvalidValue;
  const RowMap m{l_a, l_b, n_t, n_v, lo, hi};
  const int rows = l_a + 2 * l_b + n_t;
  if (rows <= 0) return cudaSuccess;
  gather_split_kernel<<<dim3((rows + 7) / 8), dim3(32, 8), 0, stream>>>(
      m, parts, static_cast<const uint8_t*>(eq), ld_q, static_cast<uint8_t*>(dst), ld_dst, row_bytes / 16, rows);
  return cudaGetLastError();
}

cudaError_t launch_split_rows(int l_a, int l_b, int n_t, int n_v, int lo, int hi, const void* src,
                              long long ld_src, void* dst, long long ld_dst, int row_bytes,
                              bool merge, bool shared, cudaStream_t stream) {
  if (row_bytes % 16 || ld_src % 16 || ld_dst % 16 ||
      (reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) % 16)
    return cudaErrorInvalidValue;
  const RowMap m{l_a, l_b, n_t, n_v, lo, hi};
  const int rows = l_a + 2 * l_b + n_t;
  if (rows <= 0) return cudaSuccess;
  const dim3 grid((rows + 7) / 8), block(32, 8);
  if (merge)
    merge_rows_kernel<<<grid, block, 0, stream>>>(m, static_cast<const uint8_t*>(src), ld_src,
                                                  static_cast<uint8_t*>(dst), ld_dst, row_bytes / 16, rows,
                                                  shared ? 1 : 0);
  else
    split_rows_kernel<<<grid, block, 0, stream>>>(m, static_cast<const uint8_t*>(src), ld_src,
                                                  static_cast<uint8_t*>(dst), ld_dst, row_bytes / 16, rows);
  return cudaGetLastError();
}

}  // namespace spava
