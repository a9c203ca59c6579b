// decoder.cu -- the step on either side of the Spava attention:
// the reference decoder layer (simhost.cpp:196-207 project, :431-436 finish_group,
// model.cpp:60-75, matrix.cpp:128-150 layer_norm) around spava_host_layer:
//   xn = norm ? layer_norm(x, g1) : x
//   q, k, v = xn Wq, xn Wk, xn Wv                 (one GEMM against [Wq | Wk | Wv])
//   a = Spava attention layer (q, k, v)           (spava_host_layer, this library)
//   x += a Wo
//   f = norm ? layer_norm(x, g2) : x
//   x += relu(f W1) W2
// Rows are the host-local rows [anchor | lo | hi | query]; every operation is row-wise or
// a GEMM over rows, so applying it to the whole buffer equals the reference's per-part
// project / finish_group calls.  GEMMs are plain bf16 library GEMMs (cuBLASLt, fp32
// accumulation, ReLU and residual folded into the GEMM epilogue / beta); layer_norm is a
// one-warp-per-row kernel.
#include <cublasLt.h>
#include <cuda_bf16.h>

#include "spava_internal.h"

namespace spava {

namespace {

// one warp per row: mean / variance in fp32 over the row, out = (x - mean) * rsqrt(var +
// 1e-5) * g  (matrix.cpp:128-150 with the reference's eps)
__global__ void layer_norm_kernel(const __nv_bfloat16* x, long long ldx, const float* g, int d,
                                  __nv_bfloat16* y, long long ldy, int rows) {
  const int r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const __nv_bfloat16* xr = x + r * ldx;
  float s = 0.f, s2 = 0.f;
  for (int j = lane * 2; j < d; j += 64) {
    const float2 v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(xr + j));
    s += v.x + v.y;
    s2 += v.x * v.x + v.y * v.y;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  const float mean = s / d;
  const float var = fmaxf(s2 / d - mean * mean, 0.f);
  const float inv = rsqrtf(var + 1e-5f);
  __nv_bfloat16* yr = y + r * ldy;
  for (int j = lane * 2; j < d; j += 64) {
    const float2 v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(xr + j));
    const float g0 = g ? g[j] : 1.f, g1 = g ? g[j + 1] : 1.f;
    *reinterpret_cast<__nv_bfloat162*>(yr + j) =
        __floats2bfloat162_rn((v.x - mean) * inv * g0, (v.y - mean) * inv * g1);
  }
}

// row-major C[M x N] (ldc) = A[M x K] (lda) * B[K x N] (ldb) + beta * C, optional ReLU:
// column-major view D^T = B^T A^T, i.e. cuBLASLt m = N, n = M, k = K with A <-> B swapped.
cudaError_t gemm_rm(cublasLtHandle_t lt, int M, int N, int K, const __nv_bfloat16* A, long long lda,
                    const __nv_bfloat16* B, long long ldb, __nv_bfloat16* C, long long ldc, float beta,
                    bool relu, void* ws, size_t ws_bytes, cudaStream_t stream, std::string* err) {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
  cublasLtMatmulPreference_t pref = nullptr;
  cublasStatus_t st = CUBLAS_STATUS_SUCCESS;
  auto chk = [&](cublasStatus_t s) {
    if (s != CUBLAS_STATUS_SUCCESS && st == CUBLAS_STATUS_SUCCESS) st = s;
  };
  chk(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
  if (relu) {
    const cublasLtEpilogue_t epi = CUBLASLT_EPILOGUE_RELU;
    chk(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_EPILOGUE, &epi, sizeof(epi)));
  }
  chk(cublasLtMatrixLayoutCreate(&la, CUDA_R_16BF, N, K, ldb));  // B^T: N x K, ld = ldb
  chk(cublasLtMatrixLayoutCreate(&lb, CUDA_R_16BF, K, M, lda));  // A^T: K x M, ld = lda
  chk(cublasLtMatrixLayoutCreate(&lc, CUDA_R_16BF, N, M, ldc));  // C^T: N x M, ld = ldc
  chk(cublasLtMatmulPreferenceCreate(&pref));
  chk(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws_bytes,
                                           sizeof(ws_bytes)));
  cublasLtMatmulHeuristicResult_t heur{};
  int found = 0;
  if (st == CUBLAS_STATUS_SUCCESS)
    chk(cublasLtMatmulAlgoGetHeuristic(lt, op, la, lb, lc, lc, pref, 1, &heur, &found));
  const float alpha = 1.f;
  if (st == CUBLAS_STATUS_SUCCESS && found == 0) st = CUBLAS_STATUS_NOT_SUPPORTED;
  if (st == CUBLAS_STATUS_SUCCESS)
    chk(cublasLtMatmul(lt, op, &alpha, B, la, A, lb, &beta, C, lc, C, lc, &heur.algo, ws, ws_bytes, stream));
  if (pref) cublasLtMatmulPreferenceDestroy(pref);
  if (lc) cublasLtMatrixLayoutDestroy(lc);
  if (lb) cublasLtMatrixLayoutDestroy(lb);
  if (la) cublasLtMatrixLayoutDestroy(la);
  if (op) cublasLtMatmulDescDestroy(op);
  if (st != CUBLAS_STATUS_SUCCESS) {
    if (err) *err = "cublasLt matmul failed (" + std::to_string(static_cast<int>(st)) + ")";
    return cudaErrorUnknown;
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_layer_norm(const void* x, long long ldx, const float* g, int d, void* y,
                              long long ldy, int rows, cudaStream_t stream) {
  if (d % 2 || rows <= 0) return rows <= 0 ? cudaSuccess : cudaErrorInvalidValue;
  layer_norm_kernel<<<(rows + 7) / 8, 256, 0, stream>>>(static_cast<const __nv_bfloat16*>(x), ldx, g, d,
                                                        static_cast<__nv_bfloat16*>(y), ldy, rows);
  return cudaGetLastError();
}

cudaError_t gemm_bf16_rm(void* lt, int M, int N, int K, const void* A, long long lda, const void* B,
                         long long ldb, void* C, long long ldc, float beta, bool relu, void* ws,
                         size_t ws_bytes, cudaStream_t stream, std::string* err) {
  return gemm_rm(static_cast<cublasLtHandle_t>(lt), M, N, K, static_cast<const __nv_bfloat16*>(A), lda,
                 static_cast<const __nv_bfloat16*>(B), ldb, static_cast<__nv_bfloat16*>(C), ldc, beta, relu,
                 ws, ws_bytes, stream, err);
}

void* gemm_handle_create() {
  cublasLtHandle_t h = nullptr;
  return cublasLtCreate(&h) == CUBLAS_STATUS_SUCCESS ? h : nullptr;
}

void gemm_handle_destroy(void* h) {
  if (h) cublasLtDestroy(static_cast<cublasLtHandle_t>(h));
}

}  // namespace spava
