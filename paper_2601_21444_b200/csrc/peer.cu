// peer.cu -- flag stores and stream waits for the peer (NVLink P2P) fabric.
//
// The peer fabric replaces the GatherFabric's ordered AllGather rounds
// (simhost.cpp:73-124, rounds pass1 / pass2 / qpartial at :343-365, :404-414) with
// stores from the producing kernels straight into every peer GPU's exchange slot (the
// select gather and the query split-merge take the peers' IPC-mapped slot pointers).
// Ordering between GPUs is carried by 32-bit epoch flags in each GPU's exchange buffer:
//   * producer stream, after the storing kernel: a one-warp kernel raises arrive[round][me]
//     in every peer with a system-scope release store (the storing kernel completed
//     earlier in stream order, so its peer stores happen-before the flag -- a kernel,
//     not cuStreamWriteValue32, because peer device addresses are always valid kernel
//     operands);
//   * consumer stream, before the first reader: cuStreamWaitValue32(arrive[round][q] >=
//     epoch) for every peer q -- the wait sits in the stream's hardware queue, no spinning
//     kernel occupies an SM.
// The driver entry points are resolved once; no CPU fallback exists (an error is returned).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>
#include <mutex>

#include "spava_internal.h"

namespace spava {

namespace {

struct MemOps {
  PFN_cuStreamWaitValue32_v11070 wait = nullptr;
  PFN_cuStreamBatchMemOp_v11070 batch = nullptr;
  unsigned wait_flags = CU_STREAM_WAIT_VALUE_GEQ;
};

const MemOps& memops() {
  static MemOps m;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      m.wait = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(p);
    p = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamBatchMemOp", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      m.batch = reinterpret_cast<PFN_cuStreamBatchMemOp_v11070>(p);
    int dev = 0, flush = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&flush, static_cast<cudaDeviceAttr>(CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES),
                               dev) == cudaSuccess &&
        flush)
      m.wait_flags |= CU_STREAM_WAIT_VALUE_FLUSH;
  });
  return m;
}

}  // namespace

namespace {
struct FlagAddrs {
  uint32_t* p[kMaxPeers];
  int n;
};
__global__ void flag_store_kernel(const __grid_constant__ FlagAddrs f, uint32_t value) {
  if (threadIdx.x < f.n) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f.p[threadIdx.x]), "r"(value) : "memory");
  }
}
}  // namespace

cudaError_t peer_flags_store(cudaStream_t s, uint32_t* const* addrs, int n, uint32_t value) {
  if (n <= 0) return cudaSuccess;
  if (n > kMaxPeers) return cudaErrorInvalidValue;
  FlagAddrs f{};
  for (int i = 0; i < n; ++i) f.p[i] = addrs[i];
  f.n = n;
  flag_store_kernel<<<1, 32, 0, s>>>(f, value);
  return cudaGetLastError();
}

cudaError_t stream_wait_geq_u32(cudaStream_t s, const uint32_t* addr, uint32_t value) {
  const MemOps& m = memops();
  if (!m.wait) return cudaErrorNotSupported;
  return m.wait(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), value, m.wait_flags) ==
                 CUDA_SUCCESS
             ? cudaSuccess
             : cudaErrorUnknown;
}

// every address >= value, as one batched stream memory operation (one host call for all
// peers' flags of a round instead of one per peer)
cudaError_t stream_wait_all_geq_u32(cudaStream_t s, const uint32_t* const* addrs, int n, uint32_t value) {
  if (n <= 0) return cudaSuccess;
  const MemOps& m = memops();
  if (!m.batch || n > kMaxPeers) {
    for (int i = 0; i < n; ++i) {
      const cudaError_t e = stream_wait_geq_u32(s, addrs[i], value);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  CUstreamBatchMemOpParams ops[kMaxPeers];
  std::memset(ops, 0, sizeof(ops));
  for (int i = 0; i < n; ++i) {
    ops[i].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_32;
    ops[i].waitValue.address = reinterpret_cast<CUdeviceptr>(addrs[i]);
    ops[i].waitValue.value = value;
    ops[i].waitValue.flags = m.wait_flags;
  }
  return m.batch(reinterpret_cast<CUstream>(s), static_cast<unsigned>(n), ops, 0) == CUDA_SUCCESS
             ? cudaSuccess
             : cudaErrorUnknown;
}

}  // namespace spava
