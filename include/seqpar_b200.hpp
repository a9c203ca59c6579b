// seqpar_b200.hpp -- C++ drop-in mirror of the reference's hot-path operator API
// (namespace seqpar, /root/reference/proj/core/include/seqpar/{partition,approx,attention}.hpp)
// implemented on the B200 C ABI (spava_b200.h).
//
// Same names, argument meaning and error behaviour (std::invalid_argument /
// std::out_of_range) as the reference, on host fp32 matrices: each call uploads its
// operands as bf16, runs the sm_100a kernels, and returns host results.  Reference call
// sites compile unchanged (CostCounters* in the reference's position).  Differences:
//   * the GPU path computes in bf16 with fp32 accumulation; inputs that are not
//     bf16-representable are rounded to nearest-even on upload; head widths up to 128
//     (narrower heads, e.g. the acceptance suite's d = 64 / 4 heads, are zero-padded to
//     the kernels' 128 columns -- exact for the scores, see spava_score_block_ex);
//   * every attention/score entry point takes an optional trailing kv_heads (GQA) that
//     defaults to `heads`, which is the reference's (MHA) behaviour;
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
// partition.hpp:45: floor(F/H) frames per host, one extra for the first F mod H hosts
std::vector<int> frame_partition(int frames, int hosts);

// ---- costs.hpp:9-54 (algorithmic FLOP tallies, same convention and buckets)
enum class AttnSite { AnchorSelf, BlockAnchor, BlockPassing, BlockOwn, QueryAttn, EncodeAttn, Score, Other };
struct CostCounters {
  uint64_t anchor_self = 0, block_anchor = 0, block_passing = 0, block_own = 0, query_attn = 0,
           encode_attn = 0, score = 0, other = 0;
  void add(AttnSite site, uint64_t flops) {
    switch (site) {
      case AttnSite::AnchorSelf: anchor_self += flops; break;
      case AttnSite::BlockAnchor: block_anchor += flops; break;
      case AttnSite::BlockPassing: block_passing += flops; break;
      case AttnSite::BlockOwn: block_own += flops; break;
      case AttnSite::QueryAttn: query_attn += flops; break;
      case AttnSite::EncodeAttn: encode_attn += flops; break;
      case AttnSite::Score: score += flops; break;
      case AttnSite::Other: other += flops; break;
    }
  }
  uint64_t balanced_total() const { return anchor_self + block_passing + block_own; }
  uint64_t attention_total() const {
    return anchor_self + block_anchor + block_passing + block_own + query_attn;
  }
};

// ---- attention.hpp:14-63
enum class MaskKind { CausalWithin, FullyVisible };
struct KeySegment {
  const Matrix* k = nullptr;
  const Matrix* v = nullptr;
  MaskKind mask = MaskKind::FullyVisible;
  const std::vector<uint8_t>* pad = nullptr;  // tail pads only
  AttnSite site = AttnSite::Other;
};
// single-head attention output + per-row lse (-inf and a zero row: no visible key)
struct AttnPartial {
  Matrix out;
  std::vector<float> lse;
  bool row_valid(int r) const;
};
float invalid_lse();
AttnPartial attention_lse(const Matrix& q, std::span<const KeySegment> segments, float scale,
                          bool allow_invalid_rows = false, CostCounters* counters = nullptr);
Matrix merge_partials(std::span<const AttnPartial> parts);
struct MultiHeadPartial {
  Matrix out;  // n_q x heads*dh
  Matrix lse;  // n_q x heads
};
MultiHeadPartial mha_lse(const Matrix& q, std::span<const KeySegment> segments, int heads,
                         bool allow_invalid_rows = false, CostCounters* counters = nullptr,
                         int kv_heads = 0);
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

// score_context (approx.hpp:38-41): one head, explicit scale
ScoreVector score_context(const Matrix& q_qr, const Matrix& k_block, float scale,
                          const std::vector<uint8_t>* pad_mask, int source = 0,
                          bool softmax_aggregation = true, CostCounters* counters = nullptr);
// score_block (simhost.cpp:209-224): per-head score_context summed over heads.
ScoreVector score_block(const Matrix& q_qr, const Matrix& k_block, int heads,
                        const std::vector<uint8_t>* pad, int source = 0,
                        bool softmax_scores = true, CostCounters* counters = nullptr, int kv_heads = 0);
PassingBlock select_essential(const Matrix& k_block, const Matrix& v_block,
                              const ScoreVector& scores, int l_p, int global_offset);
PassingAssembly assemble_passing(int v, std::span<const PassingBlock> all_compressed);
Matrix anchor_attention(const Matrix& q_a, const Matrix& k_a, const Matrix& v_a, int heads,
                        CostCounters* counters = nullptr, int kv_heads = 0);
Matrix block_attention(const BlockQkv& block, const Matrix& k_a, const Matrix& v_a,
                       const PassingAssembly& passing, int heads, CostCounters* counters = nullptr,
                       int kv_heads = 0);
MultiHeadPartial query_attention(const Matrix& q_qr, const Matrix& anchor_k,
                                 const Matrix& anchor_v, std::pair<int, int> anchor_slice,
                                 const BlockQkv& block_lo, const BlockQkv& block_hi,
                                 const Matrix* query_k, const Matrix* query_v,
                                 bool include_query_self, int heads, int query_offset,
                                 std::vector<int>* key_indices, CostCounters* counters = nullptr,
                                 int kv_heads = 0);

}  // namespace seqpar_b200
