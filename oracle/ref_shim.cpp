// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (parity checker / CPU baseline).
//
// A C-ABI veneer over the UNMODIFIED reference operators of the Spava hot path,
// compiled together with the reference sources where they lie under
// /root/reference/proj/core/src (matrix.cpp, attention.cpp, approx.cpp,
// partition.cpp) by oracle/Makefile into oracle/_ref/libseqpar_ref.so.
// No reference source is copied into this repository; this file only
// marshals flat fp32 host arrays into seqpar::Matrix and calls:
//   seqpar::score_context     approx.cpp:15-69
//   seqpar::select_essential  approx.cpp:71-102
//   seqpar::assemble_passing  approx.cpp:104-132
//   seqpar::anchor_attention  approx.cpp:134-138
//   seqpar::block_attention   approx.cpp:140-154
//   seqpar::query_attention   approx.cpp:156-188
//   seqpar::attention_lse / mha_lse / merge_partials / mha_merge
//                             attention.cpp:18-119, 158-197
//   seqpar::split_context / slice_anchor / zigzag_map / naive_map / default_plan
//                             partition.cpp:9-113
// score_block (simhost.cpp:209-224) is file-local in the reference; it is
// restated here verbatim in behaviour (per-head column slice, score_context,
// float accumulation over heads in ascending order).
//
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
// reference) may load this library.

#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "seqpar/approx.hpp"
#include "seqpar/attention.hpp"
#include "seqpar/matrix.hpp"
#include "seqpar/partition.hpp"

using namespace seqpar;

namespace {
thread_local std::string g_err;

Matrix mk(const float* p, int r, int c) {
  Matrix m(r, c);
  if (p && static_cast<size_t>(r) * c) std::memcpy(m.data.data(), p, sizeof(float) * r * c);
  return m;
}

void put(float* dst, const Matrix& m) {
  if (dst && !m.data.empty()) std::memcpy(dst, m.data.data(), sizeof(float) * m.data.size());
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = std::string("out_of_range: ") + e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = std::string("error: ") + e.what();
    return 3;
  }
}
}  // namespace

extern "C" {

struct ref_seg {
  const float* k;
  const float* v;
  int rows;
  int causal;          // 1 = MaskKind::CausalWithin, 0 = FullyVisible
  const uint8_t* pad;  // nullable, length rows
};

const char* ref_last_error() { return g_err.c_str(); }

// score_context for one head slice (q: n_q x d, k: n_k x d).
int ref_score_context(const float* q, int n_q, const float* k, int n_k, int d, float scale,
                      const uint8_t* pad, int softmax, float* out) {
  return guard([&] {
    Matrix mq = mk(q, n_q, d), mk_ = mk(k, n_k, d);
    std::vector<uint8_t> pm;
    if (pad) pm.assign(pad, pad + n_k);
    ScoreVector sv = score_context(mq, mk_, scale, pad ? &pm : nullptr, 0, softmax != 0);
    std::memcpy(out, sv.scores.data(), sizeof(float) * n_k);
  });
}

// score_block (simhost.cpp:209-224): q: n_t x heads*dh, k: l_b x heads*dh.
int ref_score_block(const float* q, int n_t, const float* k, int l_b, int heads, int dh,
                    const uint8_t* pad, int softmax, float* out) {
  return guard([&] {
    Matrix mq = mk(q, n_t, heads * dh), mkb = mk(k, l_b, heads * dh);
    std::vector<uint8_t> pm;
    if (pad) pm.assign(pad, pad + l_b);
    const float scale = 1.0f / std::sqrt(static_cast<float>(dh));
    std::vector<float> total(l_b, 0.0f);
    for (int h = 0; h < heads; ++h) {
      Matrix qh = mq.slice_cols(h * dh, (h + 1) * dh);
      Matrix kh = mkb.slice_cols(h * dh, (h + 1) * dh);
      ScoreVector part = score_context(qh, kh, scale, pad ? &pm : nullptr, 0, softmax != 0);
      for (int j = 0; j < l_b; ++j) total[j] += part.scores[j];
    }
    std::memcpy(out, total.data(), sizeof(float) * l_b);
  });
}

// select_essential: returns the number of selected rows in *count; idx_out is
// global_offset + local index, ascending; k_out/v_out (nullable) the gathered rows.
int ref_select_essential(const float* k, const float* v, int l_b, int width, const float* scores,
                         int l_p, int global_offset, int* idx_out, float* k_out, float* v_out,
                         int* count) {
  return guard([&] {
    Matrix mkb = k ? mk(k, l_b, width) : Matrix(l_b, width);
    Matrix mvb = v ? mk(v, l_b, width) : Matrix(l_b, width);
    ScoreVector sv;
    sv.scores.assign(scores, scores + l_b);
    PassingBlock pb = select_essential(mkb, mvb, sv, l_p, global_offset);
    *count = static_cast<int>(pb.indices.size());
    if (idx_out) std::memcpy(idx_out, pb.indices.data(), sizeof(int) * pb.indices.size());
    put(k_out, pb.k);
    put(v_out, pb.v);
  });
}

static std::vector<KeySegment> build_segs(const ref_seg* segs, int nseg, int width,
                                          std::vector<Matrix>& store,
                                          std::vector<std::vector<uint8_t>>& pads) {
  store.reserve(2 * nseg);
  pads.reserve(nseg);
  std::vector<KeySegment> out;
  for (int s = 0; s < nseg; ++s) {
    store.push_back(mk(segs[s].k, segs[s].rows, width));
    store.push_back(mk(segs[s].v, segs[s].rows, width));
    const std::vector<uint8_t>* pp = nullptr;
    if (segs[s].pad) {
      pads.emplace_back(segs[s].pad, segs[s].pad + segs[s].rows);
      pp = &pads.back();
    }
    out.push_back({&store[store.size() - 2], &store.back(),
                   segs[s].causal ? MaskKind::CausalWithin : MaskKind::FullyVisible, pp,
                   AttnSite::Other});
  }
  return out;
}

// attention_lse (single head; q: nq x d; every seg k,v: rows x d).
int ref_attention_lse(const float* q, int nq, int d, const ref_seg* segs, int nseg, float scale,
                      int allow_invalid, float* out, float* lse) {
  return guard([&] {
    std::vector<Matrix> store;
    std::vector<std::vector<uint8_t>> pads;
    std::vector<KeySegment> ks = build_segs(segs, nseg, d, store, pads);
    Matrix mq = mk(q, nq, d);
    AttnPartial p = attention_lse(mq, ks, scale, allow_invalid != 0);
    put(out, p.out);
    if (lse) std::memcpy(lse, p.lse.data(), sizeof(float) * nq);
  });
}

// mha_lse: q nq x d (d = heads*dh), segs k/v rows x d.  out nq x d, lse nq x heads.
int ref_mha_lse(const float* q, int nq, int d, int heads, const ref_seg* segs, int nseg,
                int allow_invalid, float* out, float* lse) {
  return guard([&] {
    std::vector<Matrix> store;
    std::vector<std::vector<uint8_t>> pads;
    std::vector<KeySegment> ks = build_segs(segs, nseg, d, store, pads);
    Matrix mq = mk(q, nq, d);
    MultiHeadPartial p = mha_lse(mq, ks, heads, allow_invalid != 0);
    put(out, p.out);
    put(lse, p.lse);
  });
}

int ref_anchor_attention(const float* q, const float* k, const float* v, int l_a, int d,
                         int heads, float* out) {
  return guard([&] {
    put(out, anchor_attention(mk(q, l_a, d), mk(k, l_a, d), mk(v, l_a, d), heads));
  });
}

// block_attention with a pre-assembled passing set (k_p/v_p: n_p x d; n_p may be 0).
int ref_block_attention(const float* q, const float* k, const float* v, int l_b,
                        const uint8_t* pad, const float* k_a, const float* v_a, int l_a,
                        const float* k_p, const float* v_p, int n_p, int d, int heads,
                        float* out) {
  return guard([&] {
    std::vector<uint8_t> pm;
    if (pad) pm.assign(pad, pad + l_b);
    BlockQkv blk;
    blk.q = mk(q, l_b, d);
    blk.k = mk(k, l_b, d);
    blk.v = mk(v, l_b, d);
    blk.pad = pad ? &pm : nullptr;
    PassingAssembly pa;
    pa.k = mk(k_p, n_p, d);
    pa.v = mk(v_p, n_p, d);
    put(out, block_attention(blk, mk(k_a, l_a, d), mk(v_a, l_a, d), pa, heads));
  });
}

// query_attention: anchor (l_a rows) sliced [a0,a1); blocks lo/hi (l_b rows each, pads
// nullable); query self keys (n_t rows) included iff include_self.  key_idx (nullable)
// receives the attended key indices; *n_keys their count.
int ref_query_attention(const float* q, int n_t, const float* k_a, const float* v_a, int l_a,
                        int a0, int a1, const float* k_lo, const float* v_lo,
                        const uint8_t* pad_lo, int off_lo, const float* k_hi,
                        const float* v_hi, const uint8_t* pad_hi, int off_hi, int l_b,
                        const float* k_q, const float* v_q, int include_self, int d, int heads,
                        int query_offset, float* out, float* lse, int* key_idx, int* n_keys) {
  return guard([&] {
    std::vector<uint8_t> plo, phi;
    if (pad_lo) plo.assign(pad_lo, pad_lo + l_b);
    if (pad_hi) phi.assign(pad_hi, pad_hi + l_b);
    BlockQkv lo, hi;
    lo.k = mk(k_lo, l_b, d);
    lo.v = mk(v_lo, l_b, d);
    lo.pad = pad_lo ? &plo : nullptr;
    lo.global_offset = off_lo;
    hi.k = mk(k_hi, l_b, d);
    hi.v = mk(v_hi, l_b, d);
    hi.pad = pad_hi ? &phi : nullptr;
    hi.global_offset = off_hi;
    Matrix kq = mk(k_q, n_t, d), vq = mk(v_q, n_t, d);
    std::vector<int> keys;
    MultiHeadPartial p = query_attention(mk(q, n_t, d), mk(k_a, l_a, d), mk(v_a, l_a, d),
                                         {a0, a1}, lo, hi, &kq, &vq, include_self != 0, heads,
                                         query_offset, &keys);
    put(out, p.out);
    put(lse, p.lse);
    if (n_keys) *n_keys = static_cast<int>(keys.size());
    if (key_idx) std::memcpy(key_idx, keys.data(), sizeof(int) * keys.size());
  });
}

// mha_merge over nparts partials (outs[p]: rows x d, lses[p]: rows x heads).
int ref_mha_merge(int nparts, const float* const* outs, const float* const* lses, int rows,
                  int d, int heads, float* out) {
  return guard([&] {
    std::vector<MultiHeadPartial> parts(nparts);
    for (int p = 0; p < nparts; ++p) {
      parts[p].out = mk(outs[p], rows, d);
      parts[p].lse = mk(lses[p], rows, heads);
    }
    put(out, mha_merge(parts, heads));
  });
}

// merge_partials (single head): outs[p] rows x d, lses[p] rows.
int ref_merge_partials(int nparts, const float* const* outs, const float* const* lses, int rows,
                       int d, float* out) {
  return guard([&] {
    std::vector<AttnPartial> parts(nparts);
    for (int p = 0; p < nparts; ++p) {
      parts[p].out = mk(outs[p], rows, d);
      parts[p].lse.assign(lses[p], lses[p] + rows);
    }
    put(out, merge_partials(parts));
  });
}

// assemble_passing: given nblk blocks (sources, idx arrays of counts[b]), returns the
// indices of the assembly for virtual host v (idx_out) and its row count.
int ref_assemble_indices(int v, int nblk, const int* sources, const int* counts,
                         const int* const* idx, int* idx_out, int* n_out) {
  return guard([&] {
    std::vector<PassingBlock> blocks(nblk);
    for (int b = 0; b < nblk; ++b) {
      blocks[b].source = sources[b];
      blocks[b].indices.assign(idx[b], idx[b] + counts[b]);
      blocks[b].k = Matrix(counts[b], 1);
      blocks[b].v = Matrix(counts[b], 1);
    }
    PassingAssembly pa = assemble_passing(v, blocks);
    *n_out = static_cast<int>(pa.indices.size());
    if (idx_out) std::memcpy(idx_out, pa.indices.data(), sizeof(int) * pa.indices.size());
  });
}

// Partition geometry via split_context on an index matrix: returns l_b, pad, the
// per-virtual-block offsets (2H) and pad masks (2H x l_b, u8) when non-null.
int ref_split_geometry(int n_v, int n_t, int hosts, int l_a, int l_p, int* l_b, int* pad,
                       int* offsets, uint8_t* pad_masks, int* query_offset) {
  return guard([&] {
    Matrix ev(n_v, 1), eq(n_t, 1);
    for (int r = 0; r < n_v; ++r) ev.at(r, 0) = static_cast<float>(r);
    auto [plan, split] = split_context(ev, eq, hosts, l_a, l_p);
    *l_b = plan.l_b;
    *pad = plan.pad;
    if (query_offset) *query_offset = plan.query_offset();
    for (int v = 0; v < plan.virtual_hosts; ++v) {
      if (offsets) offsets[v] = split.global_offsets[v];
      if (pad_masks)
        std::memcpy(pad_masks + static_cast<size_t>(v) * plan.l_b, split.pad_mask[v].data(),
                    plan.l_b);
    }
  });
}

int ref_virtual_pair(int hosts, int zigzag, int h, int* lo, int* hi) {
  return guard([&] {
    HostTopology t = zigzag ? zigzag_map(hosts) : naive_map(hosts);
    auto p = t.virtual_pair(h);
    *lo = p.first;
    *hi = p.second;
  });
}

int ref_physical_of(int hosts, int zigzag, int v, int* h) {
  return guard([&] {
    HostTopology t = zigzag ? zigzag_map(hosts) : naive_map(hosts);
    *h = t.physical_of(v);
  });
}

int ref_slice_anchor(int l_a, int hosts, int h, int* b, int* e) {
  return guard([&] {
    auto p = slice_anchor(l_a, hosts, h);
    *b = p.first;
    *e = p.second;
  });
}

int ref_default_plan(int n, int hosts, int* l_a, int* l_b, int* l_p, int* pad) {
  return guard([&] {
    BlockPlan p = default_plan(n, hosts);
    *l_a = p.l_a;
    *l_b = p.l_b;
    *l_p = p.l_p;
    *pad = p.pad;
  });
}

}  // extern "C"
