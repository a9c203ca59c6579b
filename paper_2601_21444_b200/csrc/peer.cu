// peer.cu -- stream memory operations for the peer (NVLink P2P) fabric.
//
// The peer fabric replaces the GatherFabric's ordered AllGather rounds
// (simhost.cpp:73-124, rounds pass1 / pass2 / qpartial at :343-365, :404-414) with
// stores from the producing kernels straight into every peer GPU's exchange slot (the
// select gather and the query split-merge take the peers' IPC-mapped slot pointers).
// Ordering between GPUs is carried by 32-bit epoch flags in each GPU's exchange buffer:
//   * producer stream, after the storing kernel: cuStreamWriteValue32 into each peer's
//     arrive[round][me] (the default write carries a system-scope memory fence, so the
//     kernel's peer stores are visible before the flag);
//   * consumer stream, before the first reader: cuStreamWaitValue32(arrive[round][q] >=
//     epoch) for every peer q -- the wait sits in the stream's hardware queue, no spinning
//     kernel occupies an SM.
// The driver entry points are resolved once; no CPU fallback exists (an error is returned).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "spava_internal.h"

namespace spava {

namespace {

struct MemOps {
  PFN_cuStreamWaitValue32_v11070 wait = nullptr;
  PFN_cuStreamWriteValue32_v11070 write = nullptr;
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
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      m.write = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(p);
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

cudaError_t stream_write_u32(cudaStream_t s, uint32_t* addr, uint32_t value) {
  const MemOps& m = memops();
  if (!m.write) return cudaErrorNotSupported;
  return m.write(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), value,
                 CU_STREAM_WRITE_VALUE_DEFAULT) == CUDA_SUCCESS
             ? cudaSuccess
             : cudaErrorUnknown;
}

cudaError_t stream_wait_geq_u32(cudaStream_t s, const uint32_t* addr, uint32_t value) {
  const MemOps& m = memops();
  if (!m.wait) return cudaErrorNotSupported;
  return m.wait(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), value, m.wait_flags) ==
                 CUDA_SUCCESS
             ? cudaSuccess
             : cudaErrorUnknown;
}

}  // namespace spava
