// PCIe microbenchmark for the host-buffer (e2e) path: copy-engine H2D / D2H alone and
// together, and kernel zero-copy reads / writes of pinned host memory (UVA) alone and
// together with a copy in the other direction.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void zc_read(const uint4* __restrict__ src, size_t n, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = src[i];
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x12345678u) sink[0] = acc;
}
__global__ void zc_write(uint4* dst, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = make_uint4((unsigned)i, 1, 2, 3);
}
int main() {
  const size_t H = 168ull << 20, D = 134ull << 20;
  void *hh, *hd, *dh, *dd, *sink;
  cudaMallocHost(&hh, H); cudaMallocHost(&hd, D); cudaMalloc(&dh, H); cudaMalloc(&dd, D); cudaMalloc(&sink, 64);
  cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t a, b, c; cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&c);
  auto time = [&](auto fn, const char* name, double bytes) {
    for (int w = 0; w < 2; ++w) fn();
    cudaDeviceSynchronize();
    cudaEventRecord(a, s1); cudaStreamWaitEvent(s2, a, 0);
    for (int r = 0; r < 5; ++r) fn();
    cudaEventRecord(c, s2); cudaStreamWaitEvent(s1, c, 0); cudaEventRecord(b, s1);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    printf("%-44s %8.3f ms  %7.1f GB/s\n", name, ms, bytes / ms / 1e6);
  };
  int sms = 148;
  time([&] { cudaMemcpyAsync(dh, hh, H, cudaMemcpyHostToDevice, s1); }, "copy H2D 168MB", H);
  time([&] { cudaMemcpyAsync(hd, dd, D, cudaMemcpyDeviceToHost, s1); }, "copy D2H 134MB", D);
  time([&] { cudaMemcpyAsync(dh, hh, H, cudaMemcpyHostToDevice, s1); cudaMemcpyAsync(hd, dd, D, cudaMemcpyDeviceToHost, s2); },
       "copy H2D + D2H concurrent (302MB)", H + D);
  for (int blocks : {sms, 2 * sms, 4 * sms}) {
    char nm[64];
    snprintf(nm, 64, "kernel zero-copy read 168MB (%d CTAs)", blocks);
    time([&] { zc_read<<<blocks, 512, 0, s1>>>((const uint4*)hh, H / 16, (uint4*)sink); }, nm, H);
    snprintf(nm, 64, "kernel zero-copy write 134MB (%d CTAs)", blocks);
    time([&] { zc_write<<<blocks, 512, 0, s1>>>((uint4*)hd, D / 16); }, nm, D);
  }
  time([&] { zc_read<<<2 * sms, 512, 0, s1>>>((const uint4*)hh, H / 16, (uint4*)sink); zc_write<<<2 * sms, 512, 0, s2>>>((uint4*)hd, D / 16); },
       "zero-copy read 168 + write 134 concurrent", H + D);
  time([&] { zc_read<<<2 * sms, 512, 0, s1>>>((const uint4*)hh, H / 16, (uint4*)sink); cudaMemcpyAsync(hd, dd, D, cudaMemcpyDeviceToHost, s2); },
       "zero-copy read 168 + copy D2H 134", H + D);
  time([&] { cudaMemcpyAsync(dh, hh, H, cudaMemcpyHostToDevice, s1); zc_write<<<2 * sms, 512, 0, s2>>>((uint4*)hd, D / 16); },
       "copy H2D 168 + zero-copy write 134", H + D);
  return 0;
}
