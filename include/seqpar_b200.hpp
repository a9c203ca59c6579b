// seqpar_b200.hpp -- C++ drop-in mirror of the reference's hot-path operator API
// (namespace seqpar, /root/reference/proj/core/include/seqpar/{partition,approx,attention}.hpp)
// implemented on the B200 C ABI (spava_b200.h).
//
// Same names, argument meaning and error behaviour (std::invalid_argument /
// std::out_of_range) as the reference, on host fp32 matrices: each call uploads its
// operands as bf16, runs the sm_100a kernels, and returns host results.  Differences:
//   * the GPU path computes in bf16 with fp32 accumulation (dh = 128 only); inputs that
//     are not bf16-representable are rounded to nearest-even on upload;
//   * every attention/score entry point takes an optional kv_heads (GQA) that defaults
//     to `heads`, which is the reference's (MHA) behaviour;
//   * pad masks passed to attention must be tail masks (the only kind split_context
//     produces, partition.cpp:71-79).
// The per-layer fast path (no host round trips) is spava_host_layer in spava_b200.h.
#pragma once

#include <cstdint>
#include <span>
#include <utility>
#include <vector>

namespace seqpar_b200 {

// Dense row-major fp32 matrix (layout-compatible with seqpar::Matrix, matrix.hpp:12-32).
struct Matrix {
  int rows = 0;
  int cols = 0;
  std::vector<float> data;
  Matrix() = default;
  Matrix(int r, int c) : rows(r), cols(c), data(static_cast<size_t>(r) * c, 0.0f) {}
  float& at(int r, int c) { return data[static_cast<size_t>(r) * cols + c]; }
  float at(int r, int c) const { return data[static_cast<size_t>(r) * cols + c]; }
  const float* row(int r) const { return data.data() + static_cast<size_t>(r) * cols; }
  float* row(int r) { return data.data() + static_cast<size_t>(r) * cols; }
};

// ---- partition.hpp:13-63
struct HostTopology {
  int physical = 0;
  bool zigzag = true;
  int virtual_hosts() const { return 2 * physical; }
  std::pair<int, int> virtual_pair(int h) const;
  int physical_of(int v) const;
};
HostTopology zigzag_map(int hosts);
HostTopology naive_map(int hosts);

struct BlockPlan {
  int n_v = 0, n_t = 0, l_a = 0, l_b = 0, l_p = 0, pad = 0, virtual_hosts = 0;
  int block_offset(int v) const { return l_a + v * l_b; }
  int query_offset() const { return l_a + virtual_hosts * l_b; }
};
struct ContextSplit {
  Matrix anchor;
  std::vector<Matrix> blocks;
  Matrix query;
  std::vector<int> global_offsets;
  std::vector<std::vector<uint8_t>> pad_mask;
};
std::pair<BlockPlan, ContextSplit> split_context(const Matrix& e_v, const Matrix& e_q, int hosts,
                                                 int l_a, int l_p);
std::pair<int, int> slice_anchor(int l_a, int hosts, int h);
BlockPlan default_plan(int n, int hosts);

// ---- attention.hpp:14-63
enum class MaskKind { CausalWithin, FullyVisible };
struct KeySegment {
  const Matrix* k = nullptr;
  const Matrix* v = nullptr;
  MaskKind mask = MaskKind::FullyVisible;
  const std::vector<uint8_t>* pad = nullptr;  // tail pads only
};
struct MultiHeadPartial {
  Matrix out;  // n_q x heads*dh
  Matrix lse;  // n_q x heads
};
MultiHeadPartial mha_lse(const Matrix& q, std::span<const KeySegment> segments, int heads,
                         bool allow_invalid_rows = false, int kv_heads = 0);
Matrix mha_merge(std::span<const MultiHeadPartial> parts, int heads);

// ---- approx.hpp:13-81
struct ScoreVector {
  std::vector<float> scores;
  int source = 0;
};
struct PassingBlock {
  int source = 0;
  std::vector<int> indices;
  Matrix k, v;
};
struct PassingAssembly {
  Matrix k, v;
  std::vector<int> indices;
};
struct BlockQkv {
  int vhost = 0;
  Matrix q, k, v;
  const std::vector<uint8_t>* pad = nullptr;
  int global_offset = 0;
};

// score_block (simhost.cpp:209-224): per-head score_context summed over heads.
ScoreVector score_block(const Matrix& q_qr, const Matrix& k_block, int heads,
                        const std::vector<uint8_t>* pad, int source = 0,
                        bool softmax_scores = true, int kv_heads = 0);
PassingBlock select_essential(const Matrix& k_block, const Matrix& v_block,
                              const ScoreVector& scores, int l_p, int global_offset);
PassingAssembly assemble_passing(int v, std::span<const PassingBlock> all_compressed);
Matrix anchor_attention(const Matrix& q_a, const Matrix& k_a, const Matrix& v_a, int heads,
                        int kv_heads = 0);
Matrix block_attention(const BlockQkv& block, const Matrix& k_a, const Matrix& v_a,
                       const PassingAssembly& passing, int heads, int kv_heads = 0);
MultiHeadPartial query_attention(const Matrix& q_qr, const Matrix& anchor_k,
                                 const Matrix& anchor_v, std::pair<int, int> anchor_slice,
                                 const BlockQkv& block_lo, const BlockQkv& block_hi,
                                 const Matrix* query_k, const Matrix* query_v,
                                 bool include_query_self, int heads, int query_offset,
                                 std::vector<int>* key_indices, int kv_heads = 0);

}  // namespace seqpar_b200
