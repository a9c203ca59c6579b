// The reference's own hot-path unit tests (proj/tests/test_approx.cpp, test_tensor.cpp,
// test_partition.cpp, acceptance.cpp criteria 2/6), restated against the drop-in C++
// mirror seqpar_b200:: (include/seqpar_b200.hpp) -- i.e. run through the B200 kernels.
// Widths are heads*128 (the device path's dh); fp64 brute-force oracles as in the
// reference tests; tolerances are the bf16 ones of DESIGN.md.  Exit code = #failures.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <random>
#include <stdexcept>
#include <vector>

#include "seqpar_b200.hpp"

using namespace seqpar_b200;

static int failures = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);      \
      ++failures;                                                  \
    }                                                              \
  } while (0)

static float bf(float x) {  // round to bf16 (what the device stores)
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000u;
  std::memcpy(&x, &u, 4);
  return x;
}

static Matrix rnd(int r, int c, std::mt19937_64& g) {
  std::normal_distribution<float> d(0.f, 1.f);
  Matrix m(r, c);
  for (float& v : m.data) v = bf(d(g));
  return m;
}

// per-head dense attention in fp64 over an explicit visible-key list (test_tensor.cpp:24-45)
static Matrix naive(const Matrix& q, const Matrix& k, const Matrix& v, int heads, int kv_heads,
                    const std::vector<std::vector<int>>& vis, double scale = 0.0) {
  const int dh = q.cols / heads, g = heads / kv_heads;
  Matrix out(q.rows, q.cols);
  const double sc = scale > 0 ? scale : 1.0 / std::sqrt(double(float(dh)));
  for (int h = 0; h < heads; ++h)
    for (int i = 0; i < q.rows; ++i) {
      std::vector<double> l;
      double mx = -1e300;
      for (int j : vis[i]) {
        double d = 0;
        for (int c = 0; c < dh; ++c) d += double(q.at(i, h * dh + c)) * k.at(j, (h / g) * dh + c);
        l.push_back(d * sc);
        mx = std::max(mx, l.back());
      }
      double den = 0;
      for (double x : l) den += std::exp(x - mx);
      for (size_t t = 0; t < vis[i].size(); ++t) {
        const double w = std::exp(l[t] - mx) / den;
        for (int c = 0; c < dh; ++c) out.at(i, h * dh + c) += float(w * v.at(vis[i][t], (h / g) * dh + c));
      }
    }
  return out;
}

static float max_abs(const Matrix& a, const Matrix& b) {
  float m = 0;
  for (size_t i = 0; i < a.data.size(); ++i) m = std::max(m, std::fabs(a.data[i] - b.data[i]));
  return m;
}

int main() {
  std::mt19937_64 gen(2601);
  // ---- test_partition.cpp:42-52, 71-87, 122-159
  CHECK(zigzag_map(4).virtual_pair(0) == std::make_pair(0, 7));
  CHECK(zigzag_map(4).virtual_pair(3) == std::make_pair(3, 4));
  CHECK(naive_map(2).virtual_pair(1) == std::make_pair(2, 3));
  {
    Matrix ev(21, 2), eq(3, 2);
    auto [plan, split] = split_context(ev, eq, 2, 4, 0);
    CHECK(plan.pad == 3 && plan.l_b == 5);
    CHECK((split.pad_mask[3] == std::vector<uint8_t>{0, 0, 1, 1, 1}));
  }
  CHECK(slice_anchor(5, 2, 0) == std::make_pair(0, 3));
  bool threw = false;
  try { slice_anchor(8, 4, 4); } catch (const std::out_of_range&) { threw = true; }
  CHECK(threw);
  CHECK(default_plan(8192, 4).l_a == 128 && default_plan(8192, 4).l_p == 64);

  // ---- test_approx.cpp:90-105 select_essential pins
  {
    Matrix k = rnd(4, 128, gen), v = rnd(4, 128, gen);
    ScoreVector sv{{0.1f, 0.9f, 0.5f, 0.9f}, 0};
    CHECK((select_essential(k, v, sv, 2, 0).indices == std::vector<int>{1, 3}));
    ScoreVector ties{{0.5f, 0.5f, 0.5f, 0.5f}, 0};
    CHECK((select_essential(k, v, ties, 2, 0).indices == std::vector<int>{0, 1}));
    PassingBlock all = select_essential(k, v, sv, 4, 10);
    CHECK((all.indices == std::vector<int>{10, 11, 12, 13}));
    CHECK(all.k.data == k.data && all.v.data == v.data);
  }
  // ---- test_approx.cpp:107-128 / acceptance criterion 6: vs stable sort, ties
  {
    std::uniform_int_distribution<int> lv(0, 4), nd(1, 40);
    Matrix kk(40, 8), vv(40, 8);
    int bad = 0;
    for (int it = 0; it < 200; ++it) {
      const int n = nd(gen);
      ScoreVector sv;
      for (int j = 0; j < n; ++j) sv.scores.push_back(lv(gen) / 4.0f);
      std::uniform_int_distribution<int> lp(0, n);
      const int l_p = lp(gen);
      std::vector<int> order(n);
      std::iota(order.begin(), order.end(), 0);
      std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return sv.scores[a] > sv.scores[b]; });
      std::vector<int> want(order.begin(), order.begin() + l_p);
      std::sort(want.begin(), want.end());
      Matrix k(n, 8), v(n, 8);
      if (select_essential(k, v, sv, l_p, 0).indices != want) ++bad;
    }
    CHECK(bad == 0);
  }
  // ---- test_approx.cpp:26-44 score closed form (one head, dh = 128)
  {
    Matrix q(1, 128), k(2, 128);
    q.at(0, 0) = 1.f;
    k.at(1, 0) = bf(std::log(3.0f) * std::sqrt(128.f));
    ScoreVector s = score_block(q, k, 1, nullptr);
    CHECK(std::fabs(s.scores[0] - 0.25f) < 2e-3f && std::fabs(s.scores[1] - 0.75f) < 2e-3f);
    std::vector<uint8_t> pad = {0, 1};
    ScoreVector sp = score_block(q, k, 1, &pad);
    CHECK(std::isinf(sp.scores[1]) && std::fabs(sp.scores[0] - 1.f) < 1e-6f);
  }
  // ---- test_tensor.cpp:116-128 single visible key; :163-174 invalid rows
  {
    Matrix q = rnd(3, 128, gen), k = rnd(1, 128, gen), v = rnd(1, 128, gen);
    KeySegment seg{&k, &v, MaskKind::FullyVisible, nullptr};
    MultiHeadPartial p = mha_lse(q, std::span<const KeySegment>(&seg, 1), 1);
    float err = 0;
    for (int i = 0; i < 3; ++i)
      for (int c = 0; c < 128; ++c) err = std::max(err, std::fabs(p.out.at(i, c) - v.at(0, c)));
    CHECK(err < 4e-3f);
    std::vector<uint8_t> pad = {1};
    KeySegment ps{&k, &v, MaskKind::FullyVisible, &pad};
    bool t2 = false;
    try { mha_lse(q, std::span<const KeySegment>(&ps, 1), 1); } catch (const std::invalid_argument&) { t2 = true; }
    CHECK(t2);
    MultiHeadPartial pi = mha_lse(q, std::span<const KeySegment>(&ps, 1), 1, true);
    CHECK(!std::isfinite(pi.lse.at(0, 0)) && pi.out.at(0, 0) == 0.f);
  }
  // ---- test_tensor.cpp:148-161 causal vs brute force (GQA 4/2)
  {
    const int n = 200, heads = 4, kvh = 2;
    Matrix q = rnd(n, heads * 128, gen), k = rnd(n, kvh * 128, gen), v = rnd(n, kvh * 128, gen);
    KeySegment seg{&k, &v, MaskKind::CausalWithin, nullptr};
    MultiHeadPartial p = mha_lse(q, std::span<const KeySegment>(&seg, 1), heads, false, nullptr, kvh);
    std::vector<std::vector<int>> vis(n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j <= i; ++j) vis[i].push_back(j);
    CHECK(max_abs(p.out, naive(q, k, v, heads, kvh, vis)) < 1.5e-2f);
  }
  // ---- acceptance.cpp:91-127 (criterion 2): merge over disjoint partitions == dense
  {
    const int nq = 5, nk = 300, heads = 2;
    Matrix q = rnd(nq, heads * 128, gen), k = rnd(nk, heads * 128, gen), v = rnd(nk, heads * 128, gen);
    std::vector<MultiHeadPartial> parts;
    std::vector<Matrix> ks, vs;
    for (int s = 0; s < 3; ++s) {
      Matrix kp(100, heads * 128), vp(100, heads * 128);
      for (int r = 0; r < 100; ++r)
        for (int c = 0; c < heads * 128; ++c) {
          kp.at(r, c) = k.at(s * 100 + r, c);
          vp.at(r, c) = v.at(s * 100 + r, c);
        }
      ks.push_back(kp);
      vs.push_back(vp);
    }
    for (int s = 0; s < 3; ++s) {
      KeySegment seg{&ks[s], &vs[s], MaskKind::FullyVisible, nullptr};
      parts.push_back(mha_lse(q, std::span<const KeySegment>(&seg, 1), heads));
    }
    std::vector<std::vector<int>> vis(nq);
    for (int i = 0; i < nq; ++i)
      for (int j = 0; j < nk; ++j) vis[i].push_back(j);
    CHECK(max_abs(mha_merge(parts, heads), naive(q, k, v, heads, heads, vis)) < 1.5e-2f);
  }
  // ---- test_approx.cpp:185-228 single-host query attention == dense; key audit
  {
    const int heads = 2, l_a = 6, l_b = 40, n_t = 9;
    Matrix ka = rnd(l_a, heads * 128, gen), va = rnd(l_a, heads * 128, gen);
    BlockQkv lo, hi;
    lo.k = rnd(l_b, heads * 128, gen);
    lo.v = rnd(l_b, heads * 128, gen);
    lo.global_offset = l_a;
    hi.vhost = 1;
    hi.k = rnd(l_b, heads * 128, gen);
    hi.v = rnd(l_b, heads * 128, gen);
    hi.global_offset = l_a + l_b;
    Matrix qq = rnd(n_t, heads * 128, gen), kq = rnd(n_t, heads * 128, gen), vq = rnd(n_t, heads * 128, gen);
    std::vector<int> keys;
    MultiHeadPartial part = query_attention(qq, ka, va, {0, l_a}, lo, hi, &kq, &vq, true, heads,
                                            l_a + 2 * l_b, &keys);
    std::vector<MultiHeadPartial> parts = {part};
    Matrix merged = mha_merge(parts, heads);
    // dense: [anchor | lo | hi | query causal]
    const int N = l_a + 2 * l_b + n_t;
    Matrix K(N, heads * 128), V(N, heads * 128);
    auto put = [&](const Matrix& s, int r0, Matrix& d) {
      for (int r = 0; r < s.rows; ++r)
        for (int c = 0; c < s.cols; ++c) d.at(r0 + r, c) = s.at(r, c);
    };
    put(ka, 0, K); put(va, 0, V); put(lo.k, l_a, K); put(lo.v, l_a, V);
    put(hi.k, l_a + l_b, K); put(hi.v, l_a + l_b, V); put(kq, l_a + 2 * l_b, K); put(vq, l_a + 2 * l_b, V);
    std::vector<std::vector<int>> vis(n_t);
    for (int i = 0; i < n_t; ++i)
      for (int j = 0; j < l_a + 2 * l_b + i + 1; ++j) vis[i].push_back(j);
    CHECK(max_abs(merged, naive(qq, K, V, heads, heads, vis)) < 1.5e-2f);
    std::sort(keys.begin(), keys.end());
    std::vector<int> want(N);
    std::iota(want.begin(), want.end(), 0);
    CHECK(keys == want);
  }
  // ---- test_approx.cpp:130-158 assemble_passing strictly-earlier sources
  {
    std::vector<PassingBlock> blocks;
    for (int s = 0; s < 4; ++s) {
      PassingBlock pb;
      pb.source = s;
      pb.k = Matrix(2, 8);
      pb.v = Matrix(2, 8);
      pb.indices = {10 * s, 10 * s + 1};
      blocks.push_back(pb);
    }
    CHECK(assemble_passing(0, blocks).k.rows == 0);
    CHECK((assemble_passing(3, blocks).indices == std::vector<int>{0, 1, 10, 11, 20, 21}));
    blocks.erase(blocks.begin() + 1);
    bool t3 = false;
    try { assemble_passing(3, blocks); } catch (const std::invalid_argument&) { t3 = true; }
    CHECK(t3);
  }
  // ---- test_partition.cpp:23-40 frame_partition closed forms and law
  {
    CHECK((frame_partition(64, 8) == std::vector<int>{8, 8, 8, 8, 8, 8, 8, 8}));
    CHECK((frame_partition(10, 3) == std::vector<int>{4, 3, 3}));
    CHECK((frame_partition(7, 8) == std::vector<int>{1, 1, 1, 1, 1, 1, 1, 0}));
    bool t4 = false;
    try { frame_partition(4, 0); } catch (const std::invalid_argument&) { t4 = true; }
    CHECK(t4);
    for (int f = 0; f <= 200; f += 7)
      for (int h = 1; h <= 16; ++h) {
        std::vector<int> c = frame_partition(f, h);
        const auto [mn, mx] = std::minmax_element(c.begin(), c.end());
        CHECK(std::accumulate(c.begin(), c.end(), 0) == f && *mx - *mn <= 1 && std::is_sorted(c.rbegin(), c.rend()));
      }
  }
  // ---- acceptance.cpp:91-127 (criterion 2) as written: single-head attention_lse with
  // d in [2, 12] over random disjoint key partitions, merge_partials == dense attention
  // (narrow heads run zero-padded to 128 columns; bf16 tolerance)
  {
    int bad = 0;
    for (uint64_t seed = 0; seed < 100; ++seed) {
      std::mt19937_64 g2(seed);
      std::uniform_int_distribution<int> nk_dist(2, 32), nq_dist(1, 6), d_dist(2, 12);
      const int n_k = nk_dist(g2), n_q = nq_dist(g2), d = d_dist(g2);
      Matrix q = rnd(n_q, d, g2), k = rnd(n_k, d, g2), v = rnd(n_k, d, g2);
      const float scale = 1.0f / std::sqrt(static_cast<float>(d));
      std::uniform_int_distribution<int> seg_dist(1, std::min(8, n_k));
      const int segments = seg_dist(g2);
      std::uniform_int_distribution<int> pick(0, segments - 1);
      std::vector<int> assign(n_k);
      for (int j = 0; j < n_k; ++j) assign[j] = j < segments ? j : pick(g2);
      std::shuffle(assign.begin(), assign.end(), g2);
      std::vector<AttnPartial> parts;
      std::vector<Matrix> kss, vss;
      for (int s2 = 0; s2 < segments; ++s2) {
        std::vector<int> members;
        for (int j = 0; j < n_k; ++j)
          if (assign[j] == s2) members.push_back(j);
        Matrix ks(static_cast<int>(members.size()), d), vs(static_cast<int>(members.size()), d);
        for (size_t t = 0; t < members.size(); ++t)
          for (int c = 0; c < d; ++c) {
            ks.at(static_cast<int>(t), c) = k.at(members[t], c);
            vs.at(static_cast<int>(t), c) = v.at(members[t], c);
          }
        kss.push_back(ks);
        vss.push_back(vs);
      }
      for (int s2 = 0; s2 < segments; ++s2) {
        KeySegment seg{&kss[s2], &vss[s2], MaskKind::FullyVisible, nullptr, AttnSite::Other};
        parts.push_back(attention_lse(q, std::span<const KeySegment>(&seg, 1), scale));
      }
      std::vector<std::vector<int>> vis(n_q);
      for (int i = 0; i < n_q; ++i)
        for (int j = 0; j < n_k; ++j) vis[i].push_back(j);
      if (max_abs(merge_partials(parts), naive(q, k, v, 1, 1, vis, scale)) > 1.5e-2f) ++bad;
    }
    CHECK(bad == 0);
  }
  // ---- acceptance criterion 1's head shape (d = 64, 4 heads: dh = 16): causal mha_lse
  // and per-site FLOP counters (costs.hpp; attention.cpp:33-36)
  {
    const int n = 96, heads = 4, d = 64;
    Matrix q = rnd(n, d, gen), k = rnd(n, d, gen), v = rnd(n, d, gen);
    CostCounters cc;
    Matrix o = anchor_attention(q, k, v, heads, &cc);
    std::vector<std::vector<int>> vis(n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j <= i; ++j) vis[i].push_back(j);
    CHECK(max_abs(o, naive(q, k, v, heads, heads, vis)) < 1.5e-2f);
    CHECK(cc.anchor_self == 2ull * n * n * d && cc.attention_total() == cc.anchor_self);
    BlockQkv blk;
    blk.q = rnd(40, d, gen);
    blk.k = rnd(40, d, gen);
    blk.v = rnd(40, d, gen);
    PassingAssembly pa;
    pa.k = rnd(12, d, gen);
    pa.v = rnd(12, d, gen);
    CostCounters cb;
    block_attention(blk, k, v, pa, heads, &cb);
    CHECK(cb.block_anchor == 4ull * 40 * n * d && cb.block_passing == 4ull * 40 * 12 * d &&
          cb.block_own == 2ull * 40 * 40 * d && cb.balanced_total() == cb.block_passing + cb.block_own);
  }
  // ---- score_context (approx.hpp:38-41) closed form at d = 16, explicit scale; equal to
  // score_block of one 16-wide head (same scale 1/sqrt(16)); Score counter
  {
    Matrix q(1, 16), k(2, 16);
    q.at(0, 0) = 1.f;
    k.at(1, 0) = bf(std::log(3.0f) * 4.f);
    CostCounters cs;
    ScoreVector s = score_context(q, k, 0.25f, nullptr, 3, true, &cs);
    CHECK(std::fabs(s.scores[0] - 0.25f) < 2e-3f && std::fabs(s.scores[1] - 0.75f) < 2e-3f && s.source == 3);
    CHECK(cs.score == 2ull * 1 * 2 * 16);
    Matrix q2 = rnd(7, 16, gen), k2 = rnd(50, 16, gen);
    CHECK(score_context(q2, k2, 0.25f, nullptr).scores == score_block(q2, k2, 1, nullptr).scores);
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "all seqpar_b200 checks passed", failures);
  return failures;
}
