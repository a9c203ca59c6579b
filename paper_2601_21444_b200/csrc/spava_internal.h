// spava_internal.h -- device-side descriptors shared by the Spava kernels and the
// host runtime (never part of the public C ABI, see include/spava_b200.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <string>

namespace spava {

// ---------------------------------------------------------------- attention
constexpr int kHeadDim = 128;       // dh (Qwen2.5-VL 3B/7B)
constexpr int kBlockM = 128;        // query rows per Q tile (TMEM lanes)
constexpr int kBlockN = 128;        // keys per KV tile
constexpr int kTilesPerCta = 2;     // two Q tiles share every K/V tile (ping-pong softmax)
constexpr int kMaxDevices = 64;    // per-device caches of kernel attributes
constexpr int kMaxSegs = 5;         // [anchor | passing lo-round | passing hi-round | own]
                                     // (+1: a row chunk splits own into visible prefix + causal)
constexpr int kMaxProbs = 3;        // attention problems fused into one launch

struct AttnSeg {
  int len;     // keys in the segment; key j of row i is visible iff j < len (&& j <= i if causal)
  int causal;  // MaskKind::CausalWithin (attention.hpp:14)
};

struct AttnProb {
  int nq;                    // query rows
  int nseg;
  AttnSeg seg[kMaxSegs];
  int units;                 // ceil(nq / 256), or 1 with head pairing
  int head_pair;             // nq <= 128: the CTA's two Q tiles are q-heads h, h+1
  int splits;                // split-KV factor; >1 writes per-split partials
  int work_begin;            // first work index of this problem
  int out_f32;               // 0: bf16 output, 1: f32 output
  void* out;                 // [splits][nq][ldo]
  long long ldo;             // row stride (elements)
  long long split_stride_out;
  float* lse;                // nullable; [splits][nq][ld_lse] natural-log lse per head
  int stat_seg[2];           // fused fast scorer: segment index of block lo / hi (-1: none)
  float* seg_lse2;           // nullable; [2][splits][nq][hq] log2-domain lse of those segments
  int ld_lse;
  long long split_stride_lse;
};

// ---------------------------------------------------------------- peer fabric / merge
constexpr int kMaxPeers = 7;  // peers of one rank (8 GPUs per box)
// Producer epilogue (peer fabric): once every CTA of a group has stored its part of a slot
// into the peers' buffers, the last one raises these flags (fabric_dev.cuh).
struct FlagRaise {
  uint32_t* addr[kMaxPeers];
  int n;  // 0 = nothing to raise
  uint32_t value;
  unsigned* counter;  // zeroed device counter, reset by the last CTA
};

constexpr int kMaxMergeParts = 64;
struct MergeParams {
  const float* out[kMaxMergeParts];  // [rows][ld_part]
  const float* lse[kMaxMergeParts];  // [rows][ld_lse]
  int nparts;
  int rows, hq, dh;
  long long ld_part;
  int ld_lse;
  void* dst;
  long long ld_dst;
  int dst_f32;
  float* dst_lse;  // nullable [rows][hq]
  int32_t* status; // nullable; set to 1 if a row is invalid in every part
  // peer fabric: the merged rows / lse are also stored into these peers' slots (same layout)
  int npeer;
  void* peer_dst[kMaxPeers];
  float* peer_lse[kMaxPeers];
  FlagRaise fr;  // peer fabric: raise the qpartial arrive flags once every CTA has stored
};
// Receive-side merge run by the trailing CTAs of a stage attention launch (peer fabric):
// wait until every peer's qpartial flag reached `epoch`, then merge into mp.dst.
struct MergeJob {
  MergeParams mp;
  const uint32_t* wait[kMaxPeers];
  int nwait;
  uint32_t epoch;
  int ctas;  // 0 = no job
};

// tensor-core scorer arguments (score_fast.cu / score_fast_dev.cuh)
struct FastArgs {
  CUtensorMap tq;        // Q_qr [n_t x hq*128]
  CUtensorMap tk[2];     // K block [l_b x hkv*128], per block
  int n_valid[2];
  const uint8_t* pad[2];
  float* scores[2];
  float2* part;          // [blk][hq][n_t][ntiles] (tile max, tile sum), log2 domain
  float* lse2;           // [blk][hq][n_t]
  int n_t, l_b, hq, hkv, ntiles;
  float sl2;             // (1/sqrt(dh)) * log2(e)
  const uint32_t* ready; // pass 1 inside another launch: wait for *ready >= epoch first
  uint32_t epoch;
};

// Fast-mode scorer fused into the query attention launch: the attention CTAs of the (single)
// query problem emit per-split log2 row statistics of the lo / hi segments (AttnProb
// seg_lse2); the last split of each head group combines them into fa.lse2, the last group
// releases *fa.ready = epoch; then
// `ctas` trailing CTAs (one per (block, 128-key tile)) run the column-sum pass.
struct ScoreJob {
  FastArgs fa;
  int ctas;            // 0 = no job
  unsigned* counter;   // [ngroups + 1] zeroed: finished splits per head group, groups done
  uint32_t* ready;     // = fa.ready
};

struct __align__(64) AttnParams {
  // per problem: [0] = Q, [1+2s] = K of segment s, [2+2s] = V of segment s
  CUtensorMap tmap[kMaxProbs][1 + 2 * kMaxSegs];
  AttnProb prob[kMaxProbs];
  int nprob;
  int hq, hkv;
  int total_work;
  float scale_log2;  // (1/sqrt(dh)) * log2(e)
  MergeJob job;      // job.ctas trailing CTAs run the receive-side query merge
  ScoreJob sj;       // sj.ctas trailing CTAs run the fast scorer's column sums
};

// Opt kernel `fn` into `bytes` of dynamic shared memory on the current device, once per
// (device, bit of `mask`): the attribute is per device context.  Thread-safe (a race only
// repeats the idempotent call).
inline cudaError_t smem_optin(const void* fn, int bytes, std::atomic<uint32_t>* mask, uint32_t bit) {
  int dev = 0;
  cudaGetDevice(&dev);
  const bool cached = dev >= 0 && dev < kMaxDevices;
  if (cached && (mask[dev].load(std::memory_order_acquire) & (1u << bit))) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && cached) mask[dev].fetch_or(1u << bit, std::memory_order_release);
  return e;
}

// Host launch helpers (attention.cu)
struct SegView {
  const void* k;
  const void* v;
  long long ld;  // row stride in elements (bf16)
  int len;
  int causal;
};
struct ProbView {
  const void* q;
  long long ldq;
  int nq;
  int nseg;
  SegView seg[kMaxSegs];
  void* out;
  long long ldo;
  int out_f32;
  float* lse;
  int ld_lse;
  int splits;
  long long split_stride_out;
  long long split_stride_lse;
  int stat_seg[2] = {-1, -1};  // fused fast scorer (see AttnProb)
  float* seg_lse2 = nullptr;
};
void attn_prof_read(unsigned long long* out16);  // dev: cycle counters of variant 2
int attn_set_variant(int v);                     // dev: -1 = env/default, else variant id
cudaError_t launch_attention(const ProbView* probs, int nprob, int hq, int hkv, int dh,
                             cudaStream_t stream, std::string* err, const MergeJob* job = nullptr,
                             const ScoreJob* sj = nullptr, float scale = 0.f);

// 2D bf16 [rows x cols] tensor map, box 64 cols x box_rows rows, 128B swizzle
bool make_tmap_bf16(CUtensorMap* m, const void* base, long long rows, long long cols, long long ld,
                    int box_rows, std::string* err);

// ---------------------------------------------------------------- scoring
size_t score_workspace_bytes(int n_t, int l_b, int hq);  // sized for 2 blocks
cudaError_t launch_score_exact2(int nblk, const void* q, long long ldq, int n_t,
                                const void* const* k, long long ldk, int l_b,
                                const uint8_t* const* pad, const int* n_valid, int hq, int hkv,
                                int dh, int softmax, float* const* scores, void* ws,
                                size_t ws_bytes, cudaStream_t stream, float scale = 0.f);
cudaError_t launch_score_exact(const void* q, long long ldq, int n_t, const void* k,
                               long long ldk, int l_b, const uint8_t* pad, int n_valid, int hq,
                               int hkv, int dh, int softmax, float* scores, void* ws,
                               size_t ws_bytes, cudaStream_t stream, float scale = 0.f);

// fast (tensor-core) scoring: same definition as score_block, logits from tcgen05 bf16
// MMAs with fp32 accumulation (not bit-faithful; see score_fast.cu)
size_t score_fast_workspace_bytes(int n_t, int l_b, int hq);  // sized for 2 blocks
cudaError_t launch_score_fast2(int nblk, const void* q, long long ldq, int n_t,
                               const void* const* k, long long ldk, int l_b,
                               const uint8_t* const* pad, const int* n_valid, int hq, int hkv,
                               int dh, float* const* scores, void* ws, size_t ws_bytes,
                               cudaStream_t stream, std::string* err);

// ---------------------------------------------------------------- selection
// peer fabric: the same slot in up to kMaxPeers other GPUs' exchange buffers (IPC-mapped)
struct PeerSlots {
  void* k[kMaxPeers];
  void* v[kMaxPeers];
  void* idx[kMaxPeers];
  void* cnt[kMaxPeers];
  int n;
};
struct SelectPackJob {
  const float* scores;
  int global_offset;
  const void* k;
  const void* v;
  int32_t* idx;
  void* k_out;
  void* v_out;
  int32_t* count;
  const PeerSlots* peers;  // nullable
  int require_full = 0;    // passing source: count < l_p sets status bit 2
  FlagRaise fr = {};       // peer fabric: this round's arrive flags, raised by the gather
};
// select + pack of 1 or 2 blocks (same l_b / l_p / widths) in one select and one gather launch
cudaError_t launch_select_pack_n(const SelectPackJob* jobs, int n, int l_b, int l_p, long long ld, int width,
                                 long long ld_out, int32_t* status, cudaStream_t stream);
cudaError_t launch_select_pack(const float* scores, int l_b, int l_p, int global_offset,
                               const void* k, const void* v, long long ld, int width, int32_t* idx,
                               void* k_out, void* v_out, long long ld_out, int32_t* count,
                               int32_t* status, cudaStream_t stream, const PeerSlots* peers = nullptr);
// encode gather: rank q's share of E_v rows [off[q], off[q+1]) at base[q] (row stride ld)
struct GatherParts {
  const void* base[kMaxPeers + 1];
  long long off[kMaxPeers + 2];
  long long ld;
  int n;
};
cudaError_t launch_gather_split(int l_a, int l_b, int n_t, int n_v, int lo, int hi, const GatherParts& parts,
                                const void* eq, long long ld_q, void* dst, long long ld_dst, int row_bytes,
                                cudaStream_t stream);
// stream memory operations (driver API): the peer fabric's arrival / release flags
// one kernel: system-scope release store of `value` to every address (peer flags)
cudaError_t peer_flags_store(cudaStream_t s, uint32_t* const* addrs, int n, uint32_t value);
cudaError_t stream_wait_geq_u32(cudaStream_t s, const uint32_t* addr, uint32_t value);
cudaError_t stream_wait_all_geq_u32(cudaStream_t s, const uint32_t* const* addrs, int n, uint32_t value);

// ---------------------------------------------------------------- split_context rows
cudaError_t launch_split_rows(int l_a, int l_b, int n_t, int n_v, int lo, int hi, const void* src,
                              long long ld_src, void* dst, long long ld_dst, int row_bytes,
                              bool merge, bool shared, cudaStream_t stream);

// ---------------------------------------------------------------- decoder layer (f2)
cudaError_t launch_layer_norm(const void* x, long long ldx, const float* g, int d, void* y,
                              long long ldy, int rows, cudaStream_t stream);
// tcgen05 GEMM (gemm.cu): C (+)= A B row-major bf16, fp32 accumulation; C's column ranges
// [col0[r], col0[r+1]) go to out[r] (stride ldo[r]); beta * C residual and ReLU epilogue
cudaError_t launch_gemm_bf16(int M, int N, int K, const void* A, long long lda, const void* B, long long ldb,
                             int nout, const int* col0, void* const* out, const long long* ldo, float beta,
                             bool relu, cudaStream_t stream, std::string* err);

// ---------------------------------------------------------------- merge
cudaError_t launch_merge(const MergeParams& p, cudaStream_t stream);
cudaError_t launch_delay(unsigned long long ns, cudaStream_t stream);  // test: stream delay

}  // namespace spava
