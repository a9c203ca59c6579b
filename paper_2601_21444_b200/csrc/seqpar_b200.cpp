// seqpar_b200.cu -- host implementation of include/seqpar_b200.hpp: the reference's
// operator API (seqpar::, partition/approx/attention.hpp) on top of the C ABI.
// Host-only code (compiled by nvcc with the rest of the library); every compute call
// goes through spava_* and therefore through the sm_100a kernels -- no CPU math here
// beyond the reference's own host-side bookkeeping (split_context row copies,
// assemble_passing concatenation, key-index audit lists).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>

#include "../../include/seqpar_b200.hpp"
#include "../../include/spava_b200.h"

namespace seqpar_b200 {

namespace {

constexpr int kDh = 128;

void check(int rc, const char* what) {
  if (rc == SPAVA_OK) return;
  const std::string msg = std::string(what) + ": " + spava_last_error();
  if (rc == SPAVA_EINVAL) throw std::invalid_argument(msg);
  if (rc == SPAVA_ERANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

struct Dev {
  void* p = nullptr;
  explicit Dev(size_t bytes) { cuda_check(cudaMalloc(&p, std::max<size_t>(bytes, 16)), "cudaMalloc"); }
  ~Dev() { cudaFree(p); }
  Dev(Dev&& o) noexcept : p(o.p) { o.p = nullptr; }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

// fp32 -> bf16 (round to nearest even) upload of a whole matrix
Dev upload_bf16(const Matrix& m) {
  std::vector<__nv_bfloat16> h(m.data.size());
  for (size_t i = 0; i < h.size(); ++i) h[i] = __float2bfloat16_rn(m.data[i]);
  Dev d(h.size() * sizeof(__nv_bfloat16));
  cuda_check(cudaMemcpy(d.p, h.data(), h.size() * sizeof(__nv_bfloat16), cudaMemcpyHostToDevice), "H2D");
  return d;
}

Dev upload_f32(const float* p, size_t n) {
  Dev d(n * sizeof(float));
  if (n) cuda_check(cudaMemcpy(d.p, p, n * sizeof(float), cudaMemcpyHostToDevice), "H2D");
  return d;
}

Matrix download_f32(const void* d, int rows, int cols) {
  Matrix m(rows, cols);
  if (m.data.size())
    cuda_check(cudaMemcpy(m.data.data(), d, m.data.size() * sizeof(float), cudaMemcpyDeviceToHost), "D2H");
  return m;
}

Matrix download_bf16(const void* d, int rows, int cols) {
  std::vector<__nv_bfloat16> h(static_cast<size_t>(rows) * cols);
  if (h.size())
    cuda_check(cudaMemcpy(h.data(), d, h.size() * sizeof(__nv_bfloat16), cudaMemcpyDeviceToHost), "D2H");
  Matrix m(rows, cols);
  for (size_t i = 0; i < h.size(); ++i) m.data[i] = __bfloat162float(h[i]);
  return m;
}

int head_dim(int width, int heads, const char* what) {
  if (heads < 1 || width % heads)
    throw std::invalid_argument(std::string(what) + ": model width not divisible by head count");
  if (width / heads < 1 || width / heads > kDh)
    throw std::invalid_argument(std::string(what) + ": the B200 path implements head widths 1..128");
  return width / heads;
}

// [rows x heads*dh] -> device bf16 [rows x heads*128]: each head zero-padded to the
// kernels' 128 columns (zero products are exact, so narrow heads compute as themselves)
Dev upload_heads_bf16(const Matrix& m, int heads, int dh) {
  if (dh == kDh) return upload_bf16(m);
  const size_t W = static_cast<size_t>(heads) * kDh;
  std::vector<__nv_bfloat16> h(static_cast<size_t>(m.rows) * W, __float2bfloat16_rn(0.f));
  for (int r = 0; r < m.rows; ++r)
    for (int g = 0; g < heads; ++g)
      for (int c = 0; c < dh; ++c) h[r * W + g * kDh + c] = __float2bfloat16_rn(m.at(r, g * dh + c));
  Dev d(h.size() * sizeof(__nv_bfloat16));
  cuda_check(cudaMemcpy(d.p, h.data(), h.size() * sizeof(__nv_bfloat16), cudaMemcpyHostToDevice), "H2D");
  return d;
}

// device f32 [rows x heads*wp] -> [rows x heads*dh] (drops each head's padding columns)
Matrix download_heads_f32(const void* d, int rows, int heads, int dh, int wp) {
  if (dh == wp) return download_f32(d, rows, heads * dh);
  Matrix full = download_f32(d, rows, heads * wp), m(rows, heads * dh);
  for (int r = 0; r < rows; ++r)
    for (int g = 0; g < heads; ++g)
      for (int c = 0; c < dh; ++c) m.at(r, g * dh + c) = full.at(r, g * wp + c);
  return m;
}

// host f32 [rows x heads*dh] -> device f32 [rows x heads*wp] (zero columns past dh)
Dev upload_heads_f32(const Matrix& m, int heads, int dh, int wp) {
  if (dh == wp) return upload_f32(m.data.data(), m.data.size());
  std::vector<float> h(static_cast<size_t>(m.rows) * heads * wp, 0.f);
  for (int r = 0; r < m.rows; ++r)
    for (int g = 0; g < heads; ++g)
      for (int c = 0; c < dh; ++c) h[(static_cast<size_t>(r) * heads + g) * wp + c] = m.at(r, g * dh + c);
  return upload_f32(h.data(), h.size());
}

// reference FLOP convention (attention.cpp:33-36): per key segment 2 (causal) or 4 x
// n_q x n_k x dh, per head
void count_attention(CostCounters* counters, std::span<const KeySegment> segs, int n_q, int dh, int heads) {
  if (!counters) return;
  for (const KeySegment& s : segs) {
    const uint64_t pair_cost = s.mask == MaskKind::CausalWithin ? 2u : 4u;
    counters->add(s.site, pair_cost * static_cast<uint64_t>(n_q) * s.k->rows * dh * heads);
  }
}

// tail pad mask -> number of valid keys; a non-tail mask is unsupported on the device path
int valid_len(const std::vector<uint8_t>* pad, int rows, const char* what) {
  if (!pad) return rows;
  if (static_cast<int>(pad->size()) != rows) throw std::invalid_argument(std::string(what) + ": pad mask length mismatch");
  int n = rows;
  while (n > 0 && (*pad)[n - 1]) --n;
  for (int j = 0; j < n; ++j)
    if ((*pad)[j]) throw std::invalid_argument(std::string(what) + ": only tail pad masks are supported");
  return n;
}

}  // namespace

// ------------------------------------------------------------------ partition
std::pair<int, int> HostTopology::virtual_pair(int h) const {
  spava_plan p{};
  p.hosts = physical;
  p.virtual_hosts = 2 * physical;
  p.zigzag = zigzag ? 1 : 0;
  int lo, hi;
  check(spava_virtual_pair(&p, h, &lo, &hi), "virtual_pair");
  return {lo, hi};
}

int HostTopology::physical_of(int v) const {
  spava_plan p{};
  p.hosts = physical;
  p.virtual_hosts = 2 * physical;
  p.zigzag = zigzag ? 1 : 0;
  int h;
  check(spava_physical_of(&p, v, &h), "physical_of");
  return h;
}

HostTopology zigzag_map(int hosts) {
  if (hosts < 1) throw std::invalid_argument("zigzag_map: need at least one host");
  return {hosts, true};
}

HostTopology naive_map(int hosts) {
  if (hosts < 1) throw std::invalid_argument("naive_map: need at least one host");
  return {hosts, false};
}

std::pair<BlockPlan, ContextSplit> split_context(const Matrix& e_v, const Matrix& e_q, int hosts,
                                                 int l_a, int l_p) {
  spava_plan p{};
  check(spava_make_plan(e_v.rows, e_q.rows, hosts, l_a, l_p, 1, &p), "split_context");
  BlockPlan plan{p.n_v, p.n_t, p.l_a, p.l_b, p.l_p, p.pad, p.virtual_hosts};
  ContextSplit split;
  split.anchor = Matrix(l_a, e_v.cols);
  std::memcpy(split.anchor.data.data(), e_v.data.data(), sizeof(float) * split.anchor.data.size());
  split.query = e_q;
  for (int v = 0; v < p.virtual_hosts; ++v) {
    Matrix block(p.l_b, e_v.cols);
    std::vector<uint8_t> mask(p.l_b);
    check(spava_pad_mask(&p, v, mask.data()), "split_context");
    for (int r = 0; r < p.l_b; ++r)
      if (!mask[r])
        std::memcpy(block.row(r), e_v.row(plan.block_offset(v) + r), sizeof(float) * e_v.cols);
    split.blocks.push_back(std::move(block));
    split.global_offsets.push_back(plan.block_offset(v));
    split.pad_mask.push_back(std::move(mask));
  }
  return {plan, split};
}

std::pair<int, int> slice_anchor(int l_a, int hosts, int h) {
  int b, e;
  check(spava_slice_anchor(l_a, hosts, h, &b, &e), "slice_anchor");
  return {b, e};
}

std::vector<int> frame_partition(int frames, int hosts) {
  if (hosts < 1) throw std::invalid_argument("frame_partition: need at least one host");
  if (frames < 0) throw std::invalid_argument("frame_partition: negative frame count");
  std::vector<int> counts(hosts);
  check(spava_frame_partition(frames, hosts, counts.data()), "frame_partition");
  return counts;
}

BlockPlan default_plan(int n, int hosts) {
  spava_plan p{};
  check(spava_default_plan(n, hosts, &p), "default_plan");
  return BlockPlan{p.n_v, p.n_t, p.l_a, p.l_b, p.l_p, p.pad, p.virtual_hosts};
}

// ------------------------------------------------------------------- scoring
namespace {
ScoreVector score_impl(const Matrix& q_qr, const Matrix& k_block, int heads, int kv_heads, float scale,
                       const std::vector<uint8_t>* pad, int source, bool softmax, CostCounters* counters,
                       const char* what) {
  if (q_qr.rows == 0) throw std::invalid_argument("score_context: empty query");
  const int dh = head_dim(q_qr.cols, heads, what);
  if (k_block.cols != kv_heads * dh) throw std::invalid_argument("score_context: width mismatch");
  if (pad && static_cast<int>(pad->size()) != k_block.rows)
    throw std::invalid_argument("score_context: pad mask length mismatch");
  if (counters) counters->add(AttnSite::Score, 2ull * q_qr.rows * k_block.rows * dh * heads);
  Dev q = upload_heads_bf16(q_qr, heads, dh), k = upload_heads_bf16(k_block, kv_heads, dh);
  Dev pd(pad ? pad->size() : 1);
  if (pad) cuda_check(cudaMemcpy(pd.p, pad->data(), pad->size(), cudaMemcpyHostToDevice), "H2D");
  Dev sc(sizeof(float) * std::max(k_block.rows, 1));
  const size_t wsb = spava_score_workspace(q_qr.rows, k_block.rows, heads);
  Dev ws(wsb);
  check(spava_score_block_ex(q.p, heads * kDh, q_qr.rows, k.p, kv_heads * kDh, k_block.rows,
                             pad ? pd.as<uint8_t>() : nullptr, k_block.rows, heads, kv_heads, kDh,
                             softmax ? 1 : 0, sc.as<float>(), ws.p, wsb, nullptr, scale),
        what);
  ScoreVector out;
  out.source = source;
  out.scores.resize(k_block.rows);
  cuda_check(cudaMemcpy(out.scores.data(), sc.p, sizeof(float) * k_block.rows, cudaMemcpyDeviceToHost), "D2H");
  return out;
}
}  // namespace

ScoreVector score_context(const Matrix& q_qr, const Matrix& k_block, float scale,
                          const std::vector<uint8_t>* pad_mask, int source, bool softmax_aggregation,
                          CostCounters* counters) {
  if (q_qr.rows == 0) throw std::invalid_argument("score_context: empty query");
  if (q_qr.cols != k_block.cols) throw std::invalid_argument("score_context: width mismatch");
  if (!(scale > 0.f) || !std::isfinite(scale)) throw std::invalid_argument("score_context: scale must be > 0");
  return score_impl(q_qr, k_block, 1, 1, scale, pad_mask, source, softmax_aggregation, counters, "score_context");
}

ScoreVector score_block(const Matrix& q_qr, const Matrix& k_block, int heads,
                        const std::vector<uint8_t>* pad, int source, bool softmax_scores,
                        CostCounters* counters, int kv_heads) {
  if (kv_heads <= 0) kv_heads = heads;
  const int dh = head_dim(q_qr.cols, heads, "score_block");
  return score_impl(q_qr, k_block, heads, kv_heads, 1.0f / std::sqrt(static_cast<float>(dh)), pad, source,
                    softmax_scores, counters, "score_block");
}

PassingBlock select_essential(const Matrix& k_block, const Matrix& v_block,
                              const ScoreVector& scores, int l_p, int global_offset) {
  if (l_p < 0 || l_p > k_block.rows) throw std::invalid_argument("select_essential: l_p out of range");
  if (static_cast<int>(scores.scores.size()) != k_block.rows)
    throw std::invalid_argument("select_essential: score length mismatch");
  const int l_b = k_block.rows, w = k_block.cols;
  Dev s = upload_f32(scores.scores.data(), scores.scores.size());
  Dev idx(sizeof(int32_t) * std::max(l_p, 1)), cnt(4), st(4);
  cuda_check(cudaMemset(st.p, 0, 4), "memset");
  const bool gather = (w % 8) == 0 && w > 0;
  Dev k = upload_bf16(k_block), v = upload_bf16(v_block);
  Dev ko(sizeof(__nv_bfloat16) * std::max<size_t>(static_cast<size_t>(l_p) * w, 1));
  Dev vo(sizeof(__nv_bfloat16) * std::max<size_t>(static_cast<size_t>(l_p) * w, 1));
  check(spava_select_pack(s.as<float>(), l_b, l_p, global_offset, gather ? k.p : nullptr,
                          gather ? v.p : nullptr, gather ? w : 8, gather ? w : 8, idx.as<int32_t>(),
                          gather ? ko.p : nullptr, gather ? vo.p : nullptr, gather ? w : 8,
                          cnt.as<int32_t>(), st.as<int32_t>(), nullptr),
        "select_essential");
  int n = 0, status = 0;
  cuda_check(cudaMemcpy(&n, cnt.p, 4, cudaMemcpyDeviceToHost), "D2H");
  cuda_check(cudaMemcpy(&status, st.p, 4, cudaMemcpyDeviceToHost), "D2H");
  if (status) throw std::invalid_argument("select_essential: NaN score");
  PassingBlock pb;
  pb.source = scores.source;
  pb.indices.resize(n);
  if (n) cuda_check(cudaMemcpy(pb.indices.data(), idx.p, sizeof(int) * n, cudaMemcpyDeviceToHost), "D2H");
  if (gather) {
    pb.k = download_bf16(ko.p, n, w);
    pb.v = download_bf16(vo.p, n, w);
  } else {  // widths the 16-byte gather cannot move: host row copy of the selection
    pb.k = Matrix(n, w);
    pb.v = Matrix(n, v_block.cols);
    for (int i = 0; i < n; ++i) {
      std::memcpy(pb.k.row(i), k_block.row(pb.indices[i] - global_offset), sizeof(float) * w);
      std::memcpy(pb.v.row(i), v_block.row(pb.indices[i] - global_offset), sizeof(float) * v_block.cols);
    }
  }
  return pb;
}

PassingAssembly assemble_passing(int v, std::span<const PassingBlock> all) {
  std::vector<const PassingBlock*> src(std::max(v, 0), nullptr);
  for (const PassingBlock& pb : all)
    if (pb.source < v && pb.source >= 0) src[pb.source] = &pb;
  int rows = 0, kc = 0, vc = 0;
  for (int s = 0; s < v; ++s) {
    if (!src[s]) throw std::invalid_argument("assemble_passing: missing source block " + std::to_string(s));
    rows += src[s]->k.rows;
    kc = src[s]->k.cols;
    vc = src[s]->v.cols;
  }
  PassingAssembly out;
  out.k = Matrix(rows, kc);
  out.v = Matrix(rows, vc);
  int r = 0;
  for (int s = 0; s < v; ++s) {
    std::memcpy(out.k.row(r), src[s]->k.data.data(), sizeof(float) * src[s]->k.data.size());
    std::memcpy(out.v.row(r), src[s]->v.data.data(), sizeof(float) * src[s]->v.data.size());
    out.indices.insert(out.indices.end(), src[s]->indices.begin(), src[s]->indices.end());
    r += src[s]->k.rows;
  }
  return out;
}

// ------------------------------------------------------------------ attention
namespace {
MultiHeadPartial mha_impl(const Matrix& q, std::span<const KeySegment> segments, int heads, int kv_heads,
                          float scale, bool allow_invalid_rows, CostCounters* counters, const char* what) {
  const int dh = head_dim(q.cols, heads, what);
  if (segments.size() > 4) throw std::invalid_argument(std::string(what) + ": at most 4 key segments");
  std::vector<std::unique_ptr<Dev>> keep;
  std::vector<spava_segment> segs;
  for (const KeySegment& s : segments) {
    if (s.k->cols != kv_heads * dh) throw std::invalid_argument("attention_lse: key width != query width");
    if (s.k->rows != s.v->rows) throw std::invalid_argument("attention_lse: K/V row mismatch");
    if (s.v->cols != s.k->cols) throw std::invalid_argument("attention_lse: V width mismatch");
    if (s.mask == MaskKind::CausalWithin && s.k->rows != q.rows)
      throw std::invalid_argument("attention_lse: causal segment must match query rows");
    const int n = valid_len(s.pad, s.k->rows, "attention_lse");
    keep.push_back(std::make_unique<Dev>(upload_heads_bf16(*s.k, kv_heads, dh)));
    keep.push_back(std::make_unique<Dev>(upload_heads_bf16(*s.v, kv_heads, dh)));
    segs.push_back(spava_segment{keep[keep.size() - 2]->p, keep.back()->p, static_cast<int64_t>(kv_heads) * kDh, n,
                                 s.mask == MaskKind::CausalWithin ? 1 : 0});
  }
  count_attention(counters, segments, q.rows, dh, heads);
  MultiHeadPartial out;
  {
    const int64_t W = static_cast<int64_t>(heads) * kDh;
    Dev dq = upload_heads_bf16(q, heads, dh);
    Dev o(sizeof(float) * std::max<size_t>(static_cast<size_t>(q.rows) * W, 1));
    Dev l(sizeof(float) * std::max<size_t>(static_cast<size_t>(q.rows) * heads, 1));
    check(spava_attention_ex(dq.p, W, q.rows, segs.data(), static_cast<int>(segs.size()), heads, kv_heads, kDh,
                             o.p, W, 1, l.as<float>(), 1, nullptr, 0, nullptr, scale),
          what);
    out.out = download_heads_f32(o.p, q.rows, heads, dh, kDh);
    out.lse = download_f32(l.p, q.rows, heads);
  }
  if (!allow_invalid_rows)
    for (int i = 0; i < q.rows; ++i)
      for (int h = 0; h < heads; ++h)
        if (!std::isfinite(out.lse.at(i, h)))
          throw std::invalid_argument("attention_lse: query row " + std::to_string(i) + " has no visible keys");
  return out;
}

// merge over parts given as device f32 [rows x heads*wp] / [rows x heads] (wp >= 32)
Matrix merge_impl(const std::vector<const float*>& po, const std::vector<const float*>& pl, int rows, int heads,
                  int dh, int wp) {
  Matrix out;
  int status = 0;
  {
    const int64_t W = static_cast<int64_t>(heads) * wp;
    Dev o(sizeof(float) * std::max<size_t>(static_cast<size_t>(rows) * W, 1)), st(4);
    cuda_check(cudaMemset(st.p, 0, 4), "memset");
    check(spava_mha_merge(static_cast<int>(po.size()), po.data(), pl.data(), rows, W, heads, wp, o.p, W, 1,
                          nullptr, st.as<int32_t>(), nullptr),
          "merge_partials");
    out = download_heads_f32(o.p, rows, heads, dh, wp);
    cuda_check(cudaMemcpy(&status, st.p, 4, cudaMemcpyDeviceToHost), "D2H");
  }
  if (status) throw std::invalid_argument("merge_partials: a row is invalid in every part");
  return out;
}
}  // namespace

float invalid_lse() { return -std::numeric_limits<float>::infinity(); }
bool AttnPartial::row_valid(int r) const { return std::isfinite(lse[r]); }

AttnPartial attention_lse(const Matrix& q, std::span<const KeySegment> segments, float scale,
                          bool allow_invalid_rows, CostCounters* counters) {
  if (!(scale > 0.f) || !std::isfinite(scale)) throw std::invalid_argument("attention_lse: scale must be > 0");
  MultiHeadPartial m = mha_impl(q, segments, 1, 1, scale, allow_invalid_rows, counters, "attention_lse");
  AttnPartial p;
  p.out = std::move(m.out);
  p.lse.assign(m.lse.data.begin(), m.lse.data.end());
  return p;
}

Matrix merge_partials(std::span<const AttnPartial> parts) {
  if (parts.empty()) throw std::invalid_argument("merge_partials: empty part list");
  const int rows = parts.front().out.rows, d = parts.front().out.cols;
  if (d < 1 || d > 1024) throw std::invalid_argument("merge_partials: width 1..1024");
  const int wp = std::max(d, 32);  // the merge kernel's minimum row width
  std::vector<std::unique_ptr<Dev>> keep;
  std::vector<const float*> po, pl;
  for (const AttnPartial& p : parts) {
    if (p.out.rows != rows || p.out.cols != d || static_cast<int>(p.lse.size()) != rows)
      throw std::invalid_argument("merge_partials: part shape mismatch");
    keep.push_back(std::make_unique<Dev>(upload_heads_f32(p.out, 1, d, wp)));
    po.push_back(keep.back()->as<float>());
    keep.push_back(std::make_unique<Dev>(upload_f32(p.lse.data(), p.lse.size())));
    pl.push_back(keep.back()->as<float>());
  }
  return merge_impl(po, pl, rows, 1, d, wp);
}

MultiHeadPartial mha_lse(const Matrix& q, std::span<const KeySegment> segments, int heads,
                         bool allow_invalid_rows, CostCounters* counters, int kv_heads) {
  if (kv_heads <= 0) kv_heads = heads;
  const int dh = head_dim(q.cols, heads, "mha_lse");
  return mha_impl(q, segments, heads, kv_heads, 1.0f / std::sqrt(static_cast<float>(dh)), allow_invalid_rows,
                  counters, "mha_lse");
}

Matrix mha_merge(std::span<const MultiHeadPartial> parts, int heads) {
  if (parts.empty()) throw std::invalid_argument("mha_merge: empty part list");
  const int rows = parts.front().out.rows, d = parts.front().out.cols;
  const int dh = head_dim(d, heads, "mha_merge");
  const int wp = std::max(dh, 32);
  std::vector<std::unique_ptr<Dev>> keep;
  std::vector<const float*> po, pl;
  for (const MultiHeadPartial& p : parts) {
    if (p.out.rows != rows || p.out.cols != d || p.lse.rows != rows || p.lse.cols != heads)
      throw std::invalid_argument("merge_partials: part shape mismatch");
    keep.push_back(std::make_unique<Dev>(upload_heads_f32(p.out, heads, dh, wp)));
    po.push_back(keep.back()->as<float>());
    keep.push_back(std::make_unique<Dev>(upload_f32(p.lse.data.data(), p.lse.data.size())));
    pl.push_back(keep.back()->as<float>());
  }
  return merge_impl(po, pl, rows, heads, dh, wp);
}

Matrix anchor_attention(const Matrix& q_a, const Matrix& k_a, const Matrix& v_a, int heads,
                        CostCounters* counters, int kv_heads) {
  const KeySegment seg{&k_a, &v_a, MaskKind::CausalWithin, nullptr, AttnSite::AnchorSelf};
  return mha_lse(q_a, std::span<const KeySegment>(&seg, 1), heads, false, counters, kv_heads).out;
}

Matrix block_attention(const BlockQkv& block, const Matrix& k_a, const Matrix& v_a,
                       const PassingAssembly& passing, int heads, CostCounters* counters, int kv_heads) {
  std::vector<KeySegment> segs;
  if (k_a.rows > 0) segs.push_back({&k_a, &v_a, MaskKind::FullyVisible, nullptr, AttnSite::BlockAnchor});
  if (passing.k.rows > 0)
    segs.push_back({&passing.k, &passing.v, MaskKind::FullyVisible, nullptr, AttnSite::BlockPassing});
  segs.push_back({&block.k, &block.v, MaskKind::CausalWithin, block.pad, AttnSite::BlockOwn});
  return mha_lse(block.q, segs, heads, /*allow_invalid_rows=*/true, counters, kv_heads).out;
}

MultiHeadPartial query_attention(const Matrix& q_qr, const Matrix& anchor_k,
                                 const Matrix& anchor_v, std::pair<int, int> anchor_slice,
                                 const BlockQkv& lo, const BlockQkv& hi, const Matrix* query_k,
                                 const Matrix* query_v, bool include_query_self, int heads,
                                 int query_offset, std::vector<int>* key_indices, CostCounters* counters,
                                 int kv_heads) {
  const int a0 = anchor_slice.first, a1 = anchor_slice.second;
  if (a0 < 0 || a1 < a0 || a1 > anchor_k.rows) throw std::invalid_argument("slice_rows out of range");
  Matrix ka(a1 - a0, anchor_k.cols), va(a1 - a0, anchor_v.cols);
  if (a1 > a0) {
    std::memcpy(ka.data.data(), anchor_k.row(a0), sizeof(float) * ka.data.size());
    std::memcpy(va.data.data(), anchor_v.row(a0), sizeof(float) * va.data.size());
  }
  std::vector<KeySegment> segs;
  if (ka.rows > 0) segs.push_back({&ka, &va, MaskKind::FullyVisible, nullptr, AttnSite::QueryAttn});
  segs.push_back({&lo.k, &lo.v, MaskKind::FullyVisible, lo.pad, AttnSite::QueryAttn});
  segs.push_back({&hi.k, &hi.v, MaskKind::FullyVisible, hi.pad, AttnSite::QueryAttn});
  if (include_query_self) segs.push_back({query_k, query_v, MaskKind::CausalWithin, nullptr, AttnSite::QueryAttn});
  if (key_indices) {  // approx.cpp:174-185
    for (int i = a0; i < a1; ++i) key_indices->push_back(i);
    for (const BlockQkv* b : {&lo, &hi})
      for (int i = 0; i < b->k.rows; ++i)
        if (!b->pad || !(*b->pad)[i]) key_indices->push_back(b->global_offset + i);
    if (include_query_self)
      for (int i = 0; i < q_qr.rows; ++i) key_indices->push_back(query_offset + i);
  }
  return mha_lse(q_qr, segs, heads, /*allow_invalid_rows=*/true, counters, kv_heads);
}

}  // namespace seqpar_b200
