// capi.cu -- the C ABI (include/spava_b200.h) and the per-layer runtime.
//
// The runtime is the B200 form of the reference's per-host layer schedule
// (run_host, simhost.cpp:317-437; Algorithm 1):
//   score(lo), score(hi) -> select+pack(lo) -> pass1 -------------------------.
//                        -> select+pack(hi) -> pass2 ---------------------.   |
//   query_attn(anchor slice | lo | hi | [self]) -> qpartial ---> merge     |   |
//   stage1 = anchor_self + block(lo)   (waits pass1; pass2 too if naive) <-+---'
//   stage2 = block(hi)                 (waits pass1 + pass2)
// The GatherFabric (simhost.cpp:61-166) becomes a spava_fabric:
//   local -> H simulated hosts on one device; the select+pack kernel of host h writes its
//            slot of a shared exchange buffer, so the allgather is free (in place);
//   nccl  -> one process per GPU; in-place ncclAllGather of the packed slots on a
//            dedicated comm stream, cudaEvent edges implementing the DAG above.
// The attention stages never copy the passing KV: the kernel's segment table points
// straight into the exchange buffers (assemble_passing, approx.cpp:104-132, is free).
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/spava_b200.h"
#include "spava_internal.h"

using namespace spava;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CU_TRY(expr)                                                                  \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess)                                                            \
      return fail(SPAVA_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));   \
  } while (0)

#define NCCL_TRY(expr)                                                                \
  do {                                                                                \
    ncclResult_t _r = (expr);                                                         \
    if (_r != ncclSuccess)                                                            \
      return fail(SPAVA_ENCCL, std::string(#expr) + ": " + ncclGetErrorString(_r));   \
  } while (0)

#define ST_TRY(expr)              \
  do {                            \
    int _s = (expr);              \
    if (_s != SPAVA_OK) return _s; \
  } while (0)

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

bool device_ok_impl() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) return false;
  int dev = 0, major = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess)
    return false;
  return major == 10;
}

int require_device() {
  if (!device_ok_impl())
    return fail(SPAVA_ECUDA, "no sm_100 (B200) CUDA device visible: the Spava path has no CPU fallback");
  return SPAVA_OK;
}

// -------------------------------------------------------------------- plan
int plan_impl(int n_v, int n_t, int hosts, int l_a, int l_p, int zigzag, spava_plan* out) {
  if (!out) return fail(SPAVA_EINVAL, "plan: null output");
  if (hosts < 1) return fail(SPAVA_EINVAL, "split_context: need at least one host");
  if (l_a < 0 || l_a >= n_v)
    return fail(SPAVA_EINVAL, "split_context: anchor length must satisfy 0 <= l_a < n_v");
  if (n_t < 0) return fail(SPAVA_EINVAL, "split_context: negative query length");
  const int vh = 2 * hosts;
  const int rem = n_v - l_a;
  const int pad = (vh - rem % vh) % vh;
  const int l_b = (rem + pad) / vh;
  if (l_p < 0 || l_p > l_b) return fail(SPAVA_EINVAL, "split_context: l_p must lie in [0, l_b]");
  *out = spava_plan{n_v, n_t, hosts, l_a, l_b, l_p, pad, vh, zigzag ? 1 : 0};
  return SPAVA_OK;
}

int valid_rows(const spava_plan& p, int v) {
  const int start = p.l_a + v * p.l_b;
  return std::max(0, std::min(p.l_b, p.n_v - start));
}

// slots of exchange round r (0 = lo blocks, 1 = hi blocks) whose virtual source < v
void passing_range(const spava_plan& p, int round, int v, int* s0, int* s1) {
  const int H = p.hosts;
  if (p.zigzag) {
    if (round == 0) {
      *s0 = 0;
      *s1 = std::min(v, H);
    } else {
      *s0 = std::max(0, 2 * H - v);
      *s1 = H;
    }
  } else {
    *s0 = 0;
    *s1 = round == 0 ? (v + 1) / 2 : v / 2;
  }
  if (*s1 < *s0) *s1 = *s0;
}

}  // namespace

// ============================================================ exchange + host
struct Exchange {
  void* passK[2] = {nullptr, nullptr};  // [H*l_p x hkv*dh] bf16
  void* passV[2] = {nullptr, nullptr};
  int32_t* passIdx[2] = {nullptr, nullptr};  // [H*l_p]
  int32_t* passCnt[2] = {nullptr, nullptr};  // [H]
  float* qOut = nullptr;                     // [H x n_t x hq*dh]
  float* qLse = nullptr;                     // [H x n_t x hq]
  // peer fabric flags (epochs): arrive[round][q] = last epoch whose round-`round` slot from
  // host q has landed here (rounds 0 pass1, 1 pass2, 2 qpartial); done[q] = last epoch host
  // q has finished reading its own exchange buffer (so this host may overwrite its slot there)
  // round 3 = the encode gather (arrive), doneEnc[q] = host q has read the encode regions
  static constexpr size_t kFlagBytes = 8192;
  static constexpr int kArrive = 0, kDone = 4 * 256, kDoneEnc = 5 * 256;
  uint32_t* flags = nullptr;
  void* encode = nullptr;  // peer fabric: this rank's share of E_v rows (encode_bytes)
  size_t encode_bytes = 0;
  void* base = nullptr;

  int alloc(const spava_layer_cfg& c, const spava_plan& p, size_t enc_bytes = 0) {
    const size_t H = p.hosts, dk = static_cast<size_t>(c.hkv) * c.dh, dq = static_cast<size_t>(c.hq) * c.dh;
    const size_t lp = std::max(p.l_p, 1);
    const size_t kv = H * lp * dk * 2;
    const size_t idx = H * lp * 4;
    const size_t cnt = 256;
    const size_t qo = H * std::max(p.n_t, 1) * dq * 4;
    const size_t ql = H * std::max(p.n_t, 1) * c.hq * 4;
    auto al = [](size_t x) { return (x + 255) / 256 * 256; };
    const size_t total = 2 * (2 * al(kv) + al(idx) + al(cnt)) + al(qo) + al(ql) + kFlagBytes + al(enc_bytes);
    CU_TRY(cudaMalloc(&base, total));
    CU_TRY(cudaMemset(base, 0, total));
    uint8_t* b = static_cast<uint8_t*>(base);
    for (int r = 0; r < 2; ++r) {
      passK[r] = b; b += al(kv);
      passV[r] = b; b += al(kv);
      passIdx[r] = reinterpret_cast<int32_t*>(b); b += al(idx);
      passCnt[r] = reinterpret_cast<int32_t*>(b); b += al(cnt);
    }
    qOut = reinterpret_cast<float*>(b); b += al(qo);
    qLse = reinterpret_cast<float*>(b); b += al(ql);
    flags = reinterpret_cast<uint32_t*>(b); b += kFlagBytes;
    encode = enc_bytes ? b : nullptr;
    encode_bytes = enc_bytes;
    return SPAVA_OK;
  }
  void release() {
    if (base) cudaFree(base);
    base = nullptr;
  }
};

struct spava_fabric {
  spava_layer_cfg cfg{};
  spava_plan plan{};
  int device = 0;
  bool nccl = false;
  int world = 1, rank = 0;
  ncclComm_t comm = nullptr;
  cudaStream_t comm_stream = nullptr;
  Exchange shared;  // local mode; the rank's own exchange buffer in peer mode
  cudaEvent_t trace_base = nullptr;  // common time origin of the hosts' traces
  // peer (NVLink P2P) mode: every rank's exchange buffer mapped here (IPC or same process)
  bool peer = false;
  bool peer_ready = false;
  uint32_t epoch = 0;                        // layers run on this fabric
  uint32_t enc_epoch = 0;                    // encode gathers run on this fabric
  uint8_t* peer_base[kMaxMergeParts] = {};   // [world]; own base at [rank]
  bool peer_ipc[kMaxMergeParts] = {};        // opened through cudaIpcOpenMemHandle
  uint32_t* flag_tmp[kMaxPeers] = {};        // scratch: the peers' flag addresses of one store
  // pointer p into the own exchange buffer, translated into peer q's copy (same layout)
  template <typename T>
  T* at_peer(int q, T* p) const {
    const auto off = reinterpret_cast<const uint8_t*>(p) - static_cast<const uint8_t*>(shared.base);
    return reinterpret_cast<T*>(peer_base[q] + off);
  }
};

struct spava_host {
  spava_fabric* fab = nullptr;
  int h = 0, v_lo = 0, v_hi = 0, a0 = 0, a1 = 0;
  bool self_keys = false;
  int splits = 1;
  Exchange own;       // nccl mode (per rank)
  Exchange* ex = nullptr;
  float* scores[2] = {nullptr, nullptr};
  void* score_ws = nullptr;
  size_t score_ws_bytes = 0;
  float* qsplit_out = nullptr;
  float* qsplit_lse = nullptr;
  int32_t* status = nullptr;
  unsigned* ctr = nullptr;  // [48] zeroed device words: peer-flag raise counters (rounds 0..2),
                            // [4] fused-scorer ready flag, [8..41) fused-scorer CTA counters
  uint32_t score_epoch = 0;  // fused fast scorer: value released into ctr[4] per layer
  cudaEvent_t ev_score = nullptr;  // fused fast scorer: scores ready (recorded after the query launch)
  void* base = nullptr;
  cudaEvent_t ev[6] = {};  // pass1_ready, pass2_ready, q_ready, pass1_done, pass2_done, q_done
  // scoring runs on a high-priority side stream forked from the caller's stream, so the
  // CUDA-core/FP64 scorer overlaps the query / stage-1 attention that does not need it
  cudaStream_t side = nullptr;
  // host-buffer layer: scoring on a LOW-priority side stream -- the copies, not the SMs,
  // bound that path, so the row-chunk attention (whose outputs feed the D2H stream) goes
  // first and the scorer fills the gaps (it is only needed by stage 2)
  cudaStream_t side_lo = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_sel = nullptr;
  // host-buffer layer (spava_host_layer_hostbuf): H2D / D2H copy streams and their edges
  cudaStream_t h2d = nullptr, d2h = nullptr;
  // row-chunk pipeline: q rows of block lo / hi arrive in kCopyChunks chunks each; the
  // stage-1/2 attention runs per chunk and each chunk's output leaves as soon as it is final
  static constexpr int kCopyChunks = 16;  // capacity; copy_edges picks the count
  cudaEvent_t ev_kvq = nullptr;                  // all k and the query rows of q are on device (scorer)
  cudaEvent_t ev_vhi = nullptr;                  // v rows of block hi and the query are on device
  cudaEvent_t ev_qc[2 * kCopyChunks] = {};       // q rows of chunk c (chunk 0 of lo + anchor)
  cudaEvent_t ev_oc[2 * kCopyChunks + 1] = {};   // output chunk c final (last: merged query)
  cudaEvent_t ev_d2h = nullptr;
  // optional per-kernel-class device timing (bench roofline): CUDA events recorded on the
  // launching stream around every launch; classes 0 attention, 1 score, 2 select, 3 merge
  bool timing = false;
  bool serial = false;  // timing mode 2: scoring on the caller's stream (isolated kernels)
  // schedule trace in the reference Event schema (simhost.hpp:17-40): program-order records
  // with a device timestamp each (cudaEvent on the stream the step runs on)
  struct TraceRec {
    int kind, layer;
    char label[16];
    char tag[24];
    cudaEvent_t ev;
  };
  bool trace = false;
  int trace_layer = 0;
  // DelayInjection analogue: ns of spin before a phase on its stream (0 score/select on the
  // side stream, 1 exchange rounds on the comm stream, 2 query attention, 3 stage 1)
  unsigned long long delay_ns[4] = {0, 0, 0, 0};
  // one captured layer (CUDA graph over the caller's, side and comm streams)
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  uint64_t graph_kernels = 0;
  std::vector<TraceRec> trace_recs;
  std::vector<cudaEvent_t> trace_pool;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<std::pair<size_t, size_t>> spans[4];
  double attn_flops = 0.0;
  uint64_t attn_launches = 0;
};

namespace {

cudaEvent_t pool_event(spava_host* H) {
  if (H->ev_used == H->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    H->ev_pool.push_back(e);
  }
  return H->ev_pool[H->ev_used++];
}

// records an event on st if timing is on; returns its pool index (or SIZE_MAX)
size_t mark(spava_host* H, cudaStream_t st) {
  if (!H || !H->timing) return SIZE_MAX;
  const size_t i = H->ev_used;
  cudaEventRecord(pool_event(H), st);
  return i;
}

void span(spava_host* H, int cls, size_t a, cudaStream_t st) {
  if (!H || !H->timing || a == SIZE_MAX) return;
  const size_t b = mark(H, st);
  H->spans[cls].push_back({a, b});
}

// kinds follow seqpar::EventKind (simhost.hpp:17)
enum TraceKind { kCommIssued = 0, kCommWaitStart = 1, kCommCompleted = 2, kComputeBegin = 3, kComputeEnd = 4 };

void trace_ev(spava_host* H, cudaStream_t st, int kind, const char* label, bool comm) {
  if (!H || !H->trace) return;
  spava_host::TraceRec r{};
  r.kind = kind;
  r.layer = H->trace_layer;
  std::snprintf(r.label, sizeof(r.label), "%s", label);
  if (comm) std::snprintf(r.tag, sizeof(r.tag), "%s.L%d", label, H->trace_layer);
  const size_t i = H->trace_recs.size();
  if (i == H->trace_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    H->trace_pool.push_back(e);
  }
  r.ev = H->trace_pool[i];
  cudaEventRecord(r.ev, st);
  H->trace_recs.push_back(r);
}

// reference FLOP convention (attention.cpp:33-36): 4*nq*nk*dh visible, 2*nq*nk*dh causal
double problem_flops(const ProbView* pv, int np, int hq, int dh) {
  double f = 0.0;
  for (int i = 0; i < np; ++i)
    for (int s = 0; s < pv[i].nseg; ++s)
      f += (pv[i].seg[s].causal ? 2.0 : 4.0) * pv[i].nq * static_cast<double>(pv[i].seg[s].len) * dh * hq;
  return f;
}

}  // namespace

namespace {

int cfg_check(const spava_layer_cfg* c, spava_plan* plan) {
  if (!c) return fail(SPAVA_EINVAL, "layer: null cfg");
  ST_TRY(plan_impl(c->n_v, c->n_t, c->hosts, c->l_a, c->l_p, c->zigzag, plan));
  if (c->dh != kHeadDim) return fail(SPAVA_EINVAL, "layer: only dh == 128 is implemented");
  if (c->hq < 1 || c->hkv < 1 || c->hq % c->hkv || c->hq > 32)
    return fail(SPAVA_EINVAL, "layer: need hkv | hq and hq <= 32");
  if (c->n_t < 1) return fail(SPAVA_EINVAL, "layer: empty query (score_context rejects it)");
  if (plan->pad > plan->l_b)
    return fail(SPAVA_EINVAL,
                "layer: degenerate plan (pad > l_b puts pad rows in a passing source block)");
  if (c->hosts > kMaxMergeParts) return fail(SPAVA_EINVAL, "layer: too many hosts");
  if (c->score_mode != 0 && c->score_mode != 1) return fail(SPAVA_EINVAL, "layer: score_mode is 0 or 1");
  if (c->score_mode == 1 && (!c->softmax_scores || c->n_t > 128 || c->hkv > 4))
    return fail(SPAVA_EINVAL, "layer: fast scoring needs softmax_scores, n_t <= 128, hkv <= 4");
  return SPAVA_OK;
}

// -------------------------------------------------------- op wrappers
int attention_impl(const ProbView* pv, int np, int hq, int hkv, int dh, cudaStream_t st,
                   spava_host* H = nullptr, const MergeJob* job = nullptr, const ScoreJob* sj = nullptr,
                   float scale = 0.f) {
  std::string err;
  const size_t t0 = mark(H, st);
  cudaError_t e = launch_attention(pv, np, hq, hkv, dh, st, &err, job, sj, scale);
  if (e != cudaSuccess)
    return fail(e == cudaErrorInvalidValue ? SPAVA_EINVAL : SPAVA_ECUDA,
                err.empty() ? std::string("attention: ") + cudaGetErrorString(e) : err);
  span(H, 0, t0, st);
  if (H && H->timing) {
    H->attn_flops += problem_flops(pv, np, hq, dh);
    ++H->attn_launches;
  }
  g_launches += 1;
  return SPAVA_OK;
}

int merge_impl(const MergeParams& mp, cudaStream_t st, spava_host* H = nullptr) {
  const size_t t0 = mark(H, st);
  cudaError_t e = launch_merge(mp, st);
  if (e != cudaSuccess) return fail(SPAVA_ECUDA, std::string("merge: ") + cudaGetErrorString(e));
  span(H, 3, t0, st);
  g_launches += 1;
  return SPAVA_OK;
}

// split-KV factor giving about one wave of CTAs (148 SMs) for a short query block
int auto_splits(int nq, int hq, int hkv, int total_keys) {
  const bool pair = nq <= kBlockM && (hq / hkv) % 2 == 0;  // mirrors launch_attention
  const int ctas = pair ? hq / 2 : hq * ((nq + 255) / 256);
  const int tiles = std::max(1, (total_keys + kBlockN - 1) / kBlockN);
  int s = 148 / ctas;  // one wave: ceil would leave a few CTAs for a second full-length wave
  s = std::min(s, tiles);
  s = std::min(s, 32);
  return std::max(1, s);
}

// ---------------------------------------------------------- layer phases
struct HostBufs {
  const uint8_t* q;
  const uint8_t* k;
  const uint8_t* v;
  uint8_t* out;
  int32_t* sel;
};

inline const void* row_ptr(const uint8_t* base, long long row, long long ld) {
  return base + row * ld * 2;
}

// score + select + pack (lo then hi) into this host's exchange slots
// ---- peer fabric: arrival / release flags (peer.cu) and the peers' copies of a slot
uint32_t* arrive_flag(uint32_t* flags, int round, int q) { return flags + Exchange::kArrive + round * 256 + q; }
uint32_t* done_flag(uint32_t* flags, int q) { return flags + Exchange::kDone + q; }

// this rank's round-`round` slot has been stored into every peer: raise arrive[round][me]
int peer_signal(spava_fabric* F, cudaStream_t s, int round) {
  int n = 0;
  for (int q = 0; q < F->world; ++q)
    if (q != F->rank) F->flag_tmp[n++] = arrive_flag(F->at_peer(q, F->shared.flags), round, F->rank);
  CU_TRY(peer_flags_store(s, F->flag_tmp, n, F->epoch));
  if (n > 0) ++g_launches;
  return SPAVA_OK;
}

// the producing kernel raises arrive[round][me] in every peer itself (last CTA, release)
FlagRaise peer_raise(spava_host* H, int round) {
  spava_fabric* F = H->fab;
  FlagRaise f{};
  for (int q = 0; q < F->world; ++q)
    if (q != F->rank) f.addr[f.n++] = arrive_flag(F->at_peer(q, F->shared.flags), round, F->rank);
  f.value = F->epoch;
  f.counter = H->ctr + round;
  return f;
}

// the stream waits until every peer's round-`round` slot of this epoch is here
int peer_wait_arrive(spava_fabric* F, cudaStream_t s, int round) {
  int n = 0;
  for (int q = 0; q < F->world; ++q)
    if (q != F->rank) F->flag_tmp[n++] = arrive_flag(F->shared.flags, round, q);
  CU_TRY(stream_wait_all_geq_u32(s, F->flag_tmp, n, F->epoch));
  return SPAVA_OK;
}

// the stream waits until every peer has finished reading the previous epoch's exchange, so
// this rank may overwrite its slots in their buffers
int peer_wait_done(spava_fabric* F, cudaStream_t s) {
  if (F->epoch <= 1) return SPAVA_OK;
  int n = 0;
  for (int q = 0; q < F->world; ++q)
    if (q != F->rank) F->flag_tmp[n++] = done_flag(F->shared.flags, q);
  CU_TRY(stream_wait_all_geq_u32(s, F->flag_tmp, n, F->epoch - 1));
  return SPAVA_OK;
}

// this rank has finished reading its exchange buffer for the epoch: tell every peer
int peer_release(spava_fabric* F, cudaStream_t s) {
  int n = 0;
  for (int q = 0; q < F->world; ++q)
    if (q != F->rank) F->flag_tmp[n++] = done_flag(F->at_peer(q, F->shared.flags), F->rank);
  CU_TRY(peer_flags_store(s, F->flag_tmp, n, F->epoch));
  if (n > 0) ++g_launches;
  return SPAVA_OK;
}

// N1 (fast scoring): the tensor-core scorer rides in the query attention launch -- the
// attention's online softmax yields the scorer's row statistics of blocks lo / hi, and
// trailing CTAs of the same launch run the column sums (K tiles L2-resident).  The
// host-buffer pipeline (query attention after stage 1) keeps the standalone scorer.
std::atomic<int> g_fused_score{-1};  // -1: SPAVA_FUSED_SCORE (default 1); dev override
bool fused_score(const spava_host* H, bool cp_on) {
  static const int v = [] {
    const char* e = getenv("SPAVA_FUSED_SCORE");
    return e ? atoi(e) : 1;
  }();
  const int o = g_fused_score.load();
  return H->fab->cfg.score_mode == 1 && !cp_on && (o >= 0 ? o : v) != 0;
}

// scores: 0 = launch the scorer here; 1 = produced earlier on this stream (fused query
// launch); 2 = produced on another stream, wait for H->ev_score
// dev: SPAVA_HOSTBUF_TIMELINE=1 prints when each copy / chunk of one host-buffer layer ends
// (ms after the fork point; synchronises -- never set while timing)
struct Timeline {
  bool on = false;
  std::vector<std::pair<std::string, cudaEvent_t>> ev;
  void mark(const std::string& name, cudaStream_t s) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.emplace_back(name, e);
  }
  void dump() {
    if (!on || ev.empty()) return;
    cudaDeviceSynchronize();
    for (auto& [n, e] : ev) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[0].second, e);
      fprintf(stderr, "timeline %-14s %8.3f ms\n", n.c_str(), ms);
    }
    for (auto& pe : ev) cudaEventDestroy(pe.second);
    ev.clear();
  }
};
Timeline& timeline() {
  static Timeline t;
  static bool init = [] {
    const char* e = getenv("SPAVA_HOSTBUF_TIMELINE");
    t.on = e && atoi(e) != 0;
    return true;
  }();
  (void)init;
  return t;
}

int phase_select(spava_host* H, const HostBufs& b, cudaStream_t st, bool record,
                 cudaEvent_t before_hi = nullptr, int scores = 0) {
  const spava_fabric& F = *H->fab;
  const spava_layer_cfg& c = F.cfg;
  const spava_plan& p = F.plan;
  const long long dq = static_cast<long long>(c.hq) * c.dh, dk = static_cast<long long>(c.hkv) * c.dh;
  const long long qrow = p.l_a + 2LL * p.l_b;
  const int vs[2] = {H->v_lo, H->v_hi};
  trace_ev(H, st, kComputeBegin, "score", false);
  if (scores == 2) CU_TRY(cudaStreamWaitEvent(st, H->ev_score, 0));
  // both blocks (lo, hi) scored in one launch of each scoring kernel
  if (scores == 0) {
    const void* ks[2] = {row_ptr(b.k, p.l_a, dk), row_ptr(b.k, p.l_a + static_cast<long long>(p.l_b), dk)};
    const int nv[2] = {valid_rows(p, vs[0]), valid_rows(p, vs[1])};
    float* sc[2] = {H->scores[0], H->scores[1]};
    const size_t t0 = mark(H, st);
    if (c.score_mode == 1) {
      std::string err;
      cudaError_t e = launch_score_fast2(2, row_ptr(b.q, qrow, dq), dq, p.n_t, ks, dk, p.l_b, nullptr, nv,
                                         c.hq, c.hkv, c.dh, sc, H->score_ws, H->score_ws_bytes, st, &err);
      if (e != cudaSuccess) return fail(SPAVA_ECUDA, "score (fast): " + (err.empty() ? std::string(cudaGetErrorString(e)) : err));
      g_launches += 3;
    } else {
      cudaError_t e = launch_score_exact2(2, row_ptr(b.q, qrow, dq), dq, p.n_t, ks, dk, p.l_b, nullptr,
                                          nv, c.hq, c.hkv, c.dh, c.softmax_scores, sc, H->score_ws,
                                          H->score_ws_bytes, st);
      if (e != cudaSuccess) return fail(SPAVA_ECUDA, std::string("score: ") + cudaGetErrorString(e));
      g_launches += c.softmax_scores ? 3 : 2;
    }
    span(H, 1, t0, st);
    timeline().mark("score done", st);
  }
  // both blocks in one select and one gather launch, unless select hi must wait for its
  // v rows (host-buffer pipeline) -- then lo goes first so pass1 is not held back
  SelectPackJob jobs[2];
  PeerSlots peers[2] = {};
  for (int r = 0; r < 2; ++r) {
    const long long krow = p.l_a + static_cast<long long>(r) * p.l_b;
    const long long slot = static_cast<long long>(H->h) * p.l_p;
    int32_t* idx_out = H->ex->passIdx[r] + slot;
    uint8_t* k_out = static_cast<uint8_t*>(H->ex->passK[r]) + slot * dk * 2;
    uint8_t* v_out = static_cast<uint8_t*>(H->ex->passV[r]) + slot * dk * 2;
    int32_t* cnt_out = H->ex->passCnt[r] + H->h;
    if (F.peer && p.l_p > 0)  // the gather also stores the slot into every peer's buffer
      for (int q = 0; q < F.world; ++q)
        if (q != F.rank) {
          PeerSlots& ps = peers[r];
          ps.k[ps.n] = F.at_peer(q, k_out);
          ps.v[ps.n] = F.at_peer(q, v_out);
          ps.idx[ps.n] = F.at_peer(q, idx_out);
          ps.cnt[ps.n] = F.at_peer(q, cnt_out);
          ++ps.n;
        }
    // a block below the last virtual block is some later block's passing source: its slot
    // is read as exactly l_p rows, so a short selection is reported (status bit 2)
    jobs[r] = SelectPackJob{H->scores[r], p.l_a + vs[r] * p.l_b, row_ptr(b.k, krow, dk), row_ptr(b.v, krow, dk),
                            idx_out, k_out, v_out, cnt_out, &peers[r], vs[r] < p.virtual_hosts - 1};
    if (F.peer && p.l_p > 0) jobs[r].fr = peer_raise(H, r);  // the gather's last CTA signals
  }
  auto finish = [&](int r) -> int {  // after round r's select + pack
    if (F.peer && p.l_p == 0) ST_TRY(peer_signal(H->fab, st, r));
    if (b.sel && p.l_p > 0)
      CU_TRY(cudaMemcpyAsync(b.sel + r * p.l_p, jobs[r].idx, sizeof(int32_t) * p.l_p,
                             cudaMemcpyDeviceToDevice, st));
    if (record) CU_TRY(cudaEventRecord(H->ev[r], st));
    return SPAVA_OK;
  };
  const int per = before_hi ? 1 : 2;  // blocks per launch
  for (int r0 = 0; r0 < 2; r0 += per) {
    if (r0 == 1) CU_TRY(cudaStreamWaitEvent(st, before_hi, 0));  // v rows of hi
    const size_t t0 = mark(H, st);
    cudaError_t e = launch_select_pack_n(jobs + r0, per, p.l_b, p.l_p, dk, static_cast<int>(dk), dk, H->status, st);
    if (e != cudaSuccess) return fail(SPAVA_ECUDA, std::string("select: ") + cudaGetErrorString(e));
    g_launches += p.l_p > 0 ? 2 : 1;
    span(H, 2, t0, st);
    for (int r = r0; r < r0 + per; ++r) ST_TRY(finish(r));
    timeline().mark(per == 2 ? "select lo+hi done" : r0 == 0 ? "select lo done" : "select hi done", st);
  }
  trace_ev(H, st, kComputeEnd, "score", false);
  return SPAVA_OK;
}

// per-host partial query attention (split-KV, merged over splits) into its qpartial slot
int phase_query(spava_host* H, const HostBufs& b, cudaStream_t st, bool record, bool with_score = false) {
  const spava_fabric& F = *H->fab;
  const spava_layer_cfg& c = F.cfg;
  const spava_plan& p = F.plan;
  const long long dq = static_cast<long long>(c.hq) * c.dh, dk = static_cast<long long>(c.hkv) * c.dh;
  const long long qrow = p.l_a + 2LL * p.l_b;
  ProbView pv{};
  pv.q = row_ptr(b.q, qrow, dq);
  pv.ldq = dq;
  pv.nq = p.n_t;
  int n = 0;
  if (H->a1 > H->a0)
    pv.seg[n++] = SegView{row_ptr(b.k, H->a0, dk), row_ptr(b.v, H->a0, dk), dk, H->a1 - H->a0, 0};
  int nvs[2];
  for (int r = 0; r < 2; ++r) {
    const int nv = nvs[r] = valid_rows(p, r == 0 ? H->v_lo : H->v_hi);
    const long long krow = p.l_a + static_cast<long long>(r) * p.l_b;
    if (nv > 0) {
      pv.stat_seg[r] = n;
      pv.seg[n++] = SegView{row_ptr(b.k, krow, dk), row_ptr(b.v, krow, dk), dk, nv, 0};
    }
  }
  // fused fast scorer (N1): statistics of the lo / hi segments + column-sum CTAs
  ScoreJob sj{};
  if (with_score) {
    const int splits = (H->splits <= 1 && !F.peer) ? 1 : H->splits;
    const size_t seg_bytes = (2ull * splits * p.n_t * c.hq * 4 + 255) / 256 * 256;
    if (seg_bytes + 2ull * c.hq * p.n_t * 4 > H->score_ws_bytes) return fail(SPAVA_EINVAL, "fused score: workspace");
    pv.seg_lse2 = static_cast<float*>(H->score_ws);
    FastArgs& fa = sj.fa;
    std::string err;
    if (!make_tmap_bf16(&fa.tq, row_ptr(b.q, qrow, dq), p.n_t, dq, dq, 128, &err)) return fail(SPAVA_EINVAL, err);
    for (int r = 0; r < 2; ++r) {
      const long long krow = p.l_a + static_cast<long long>(r) * p.l_b;
      if (!make_tmap_bf16(&fa.tk[r], row_ptr(b.k, krow, dk), p.l_b, dk, dk, 128, &err)) return fail(SPAVA_EINVAL, err);
      fa.n_valid[r] = nvs[r];
      fa.scores[r] = H->scores[r];
    }
    fa.lse2 = reinterpret_cast<float*>(static_cast<uint8_t*>(H->score_ws) + seg_bytes);
    fa.n_t = p.n_t;
    fa.l_b = p.l_b;
    fa.hq = c.hq;
    fa.hkv = c.hkv;
    fa.ntiles = (p.l_b + 127) / 128;
    fa.sl2 = (1.0f / sqrtf(128.f)) * 1.4426950408889634f;
    fa.ready = reinterpret_cast<const uint32_t*>(H->ctr + 4);
    fa.epoch = ++H->score_epoch;
    sj.ctas = 2 * fa.ntiles;
    sj.counter = H->ctr + 8;  // [ngroups + 1] (<= 33 words)
    sj.ready = reinterpret_cast<uint32_t*>(H->ctr + 4);
  }
  const ScoreJob* sjp = with_score ? &sj : nullptr;
  if (H->self_keys)
    pv.seg[n++] = SegView{row_ptr(b.k, qrow, dk), row_ptr(b.v, qrow, dk), dk, p.n_t, 1};
  pv.nseg = n;
  float* dst_out = H->ex->qOut + static_cast<long long>(H->h) * p.n_t * dq;
  float* dst_lse = H->ex->qLse + static_cast<long long>(H->h) * p.n_t * c.hq;
  // peer fabric: the split merge always runs (one part = exact copy) and stores the host's
  // partial into every peer's qpartial slot as well
  if (H->splits <= 1 && !F.peer) {
    pv.out = dst_out;
    pv.ldo = dq;
    pv.out_f32 = 1;
    pv.lse = dst_lse;
    pv.ld_lse = c.hq;
    pv.splits = 1;
    ST_TRY(attention_impl(&pv, 1, c.hq, c.hkv, c.dh, st, H, nullptr, sjp));
  } else {
    pv.out = H->qsplit_out;
    pv.ldo = dq;
    pv.out_f32 = 1;
    pv.lse = H->qsplit_lse;
    pv.ld_lse = c.hq;
    pv.splits = H->splits;
    pv.split_stride_out = static_cast<long long>(p.n_t) * dq;
    pv.split_stride_lse = static_cast<long long>(p.n_t) * c.hq;
    ST_TRY(attention_impl(&pv, 1, c.hq, c.hkv, c.dh, st, H, nullptr, sjp));
    MergeParams mp{};
    mp.nparts = H->splits;
    for (int s = 0; s < H->splits; ++s) {
      mp.out[s] = H->qsplit_out + s * pv.split_stride_out;
      mp.lse[s] = H->qsplit_lse + s * pv.split_stride_lse;
    }
    mp.rows = p.n_t;
    mp.hq = c.hq;
    mp.dh = c.dh;
    mp.ld_part = dq;
    mp.ld_lse = c.hq;
    mp.dst = dst_out;
    mp.ld_dst = dq;
    mp.dst_f32 = 1;
    mp.dst_lse = dst_lse;
    mp.status = nullptr;  // query partials may legitimately be empty rows
    if (F.peer)
      for (int q = 0; q < F.world; ++q)
        if (q != F.rank) {
          mp.peer_dst[mp.npeer] = F.at_peer(q, dst_out);
          mp.peer_lse[mp.npeer] = F.at_peer(q, dst_lse);
          ++mp.npeer;
        }
    if (F.peer) mp.fr = peer_raise(H, 2);  // the split merge's last CTA signals qpartial
    ST_TRY(merge_impl(mp, st, H));
  }
  if (with_score) CU_TRY(cudaEventRecord(H->ev_score, st));
  if (record) CU_TRY(cudaEventRecord(H->ev[2], st));
  return SPAVA_OK;
}

ProbView block_problem(spava_host* H, const HostBufs& b, int which) {
  const spava_fabric& F = *H->fab;
  const spava_layer_cfg& c = F.cfg;
  const spava_plan& p = F.plan;
  const long long dq = static_cast<long long>(c.hq) * c.dh, dk = static_cast<long long>(c.hkv) * c.dh;
  const int v = which == 0 ? H->v_lo : H->v_hi;
  const long long row = p.l_a + static_cast<long long>(which) * p.l_b;
  ProbView pv{};
  pv.q = row_ptr(b.q, row, dq);
  pv.ldq = dq;
  pv.nq = p.l_b;
  int n = 0;
  if (p.l_a > 0) pv.seg[n++] = SegView{b.k, b.v, dk, p.l_a, 0};
  for (int r = 0; r < 2; ++r) {
    int s0, s1;
    passing_range(p, r, v, &s0, &s1);
    if (s1 > s0 && p.l_p > 0)
      pv.seg[n++] = SegView{static_cast<uint8_t*>(H->ex->passK[r]) + static_cast<long long>(s0) * p.l_p * dk * 2,
                            static_cast<uint8_t*>(H->ex->passV[r]) + static_cast<long long>(s0) * p.l_p * dk * 2,
                            dk, (s1 - s0) * p.l_p, 0};
  }
  const int nv = valid_rows(p, v);
  pv.seg[n++] = SegView{row_ptr(b.k, row, dk), row_ptr(b.v, row, dk), dk, nv, 1};
  pv.nseg = n;
  pv.out = b.out + row * dq * 2;
  pv.ldo = dq;
  pv.out_f32 = 0;
  pv.splits = 1;
  return pv;
}

// rows [r0, r1) of block `which` as its own problem: the block's causal segment splits into
// keys [0, r0) (visible to every row of the chunk) and a causal segment starting at r0
ProbView block_chunk_problem(spava_host* H, const HostBufs& b, int which, int r0, int r1) {
  ProbView pv = block_problem(H, b, which);
  const spava_layer_cfg& c = H->fab->cfg;
  const long long dq = static_cast<long long>(c.hq) * c.dh, dk = static_cast<long long>(c.hkv) * c.dh;
  SegView own = pv.seg[pv.nseg - 1];  // the causal own segment, len = valid rows
  --pv.nseg;
  const int nv = own.len;
  const int pre = std::min(r0, nv);
  if (pre > 0) pv.seg[pv.nseg++] = SegView{own.k, own.v, own.ld, pre, 0};
  const int clen = std::min(r1, nv) - r0;
  if (clen > 0)
    pv.seg[pv.nseg++] = SegView{row_ptr(static_cast<const uint8_t*>(own.k), r0, dk),
                                row_ptr(static_cast<const uint8_t*>(own.v), r0, dk), own.ld, clen, 1};
  pv.q = row_ptr(static_cast<const uint8_t*>(pv.q), r0, dq);
  pv.nq = r1 - r0;
  pv.out = static_cast<uint8_t*>(pv.out) + static_cast<long long>(r0) * dq * 2;
  return pv;
}

ProbView anchor_problem(spava_host* H, const HostBufs& b) {
  const spava_layer_cfg& c = H->fab->cfg;
  const spava_plan& p = H->fab->plan;
  const long long dq = static_cast<long long>(c.hq) * c.dh, dk = static_cast<long long>(c.hkv) * c.dh;
  ProbView pv{};
  pv.q = b.q;
  pv.ldq = dq;
  pv.nq = p.l_a;
  pv.nseg = 1;
  pv.seg[0] = SegView{b.k, b.v, dk, p.l_a, 1};
  pv.out = b.out;
  pv.ldo = dq;
  pv.splits = 1;
  return pv;
}

// needs pass1 (and pass2 under naive pairing)
int phase_stage1(spava_host* H, const HostBufs& b, cudaStream_t st) {
  const spava_layer_cfg& c = H->fab->cfg;
  ProbView pv[2] = {block_problem(H, b, 0), anchor_problem(H, b)};  // heavier first
  return attention_impl(pv, H->fab->plan.l_a > 0 ? 2 : 1, c.hq, c.hkv, c.dh, st, H);
}

MergeParams query_merge_params(spava_host* H, const HostBufs& b);

// The final query merge (mha_merge over the H host partials, simhost.cpp:404-426) as the
// trailing CTAs of the last stage launch: with peers (peer fabric) they first wait for
// every peer's qpartial arrive flag, so no separate merge launch or stream wait remains.
// Same arithmetic as merge_kernel (fabric_dev.cuh).  SPAVA_FUSED_MERGE=0: separate launch.
std::atomic<int> g_fused_merge{-1};  // -1: SPAVA_FUSED_MERGE (default 1); dev override
bool fused_merge_enabled() {
  static const int v = [] {
    const char* e = getenv("SPAVA_FUSED_MERGE");
    return e ? atoi(e) : 1;
  }();
  const int o = g_fused_merge.load();
  return (o >= 0 ? o : v) != 0;
}

MergeJob query_merge_job(spava_host* H, const HostBufs& b) {
  spava_fabric* F = H->fab;
  MergeJob job{};
  job.mp = query_merge_params(H, b);
  if (F->peer)
    for (int q = 0; q < F->world; ++q)
      if (q != F->rank) job.wait[job.nwait++] = arrive_flag(F->shared.flags, 2, q);
  job.epoch = F->epoch;
  job.ctas = 64;  // fills SMs as the last attention wave drains
  return job;
}

int phase_stage2(spava_host* H, const HostBufs& b, cudaStream_t st, bool with_merge = false) {
  const spava_layer_cfg& c = H->fab->cfg;
  ProbView pv = block_problem(H, b, 1);
  if (!with_merge) return attention_impl(&pv, 1, c.hq, c.hkv, c.dh, st, H);
  const MergeJob job = query_merge_job(H, b);
  return attention_impl(&pv, 1, c.hq, c.hkv, c.dh, st, H, &job);
}

// stage 1 and stage 2 in ONE launch (block hi, block lo, anchor): once both passing rounds
// are in, the two block problems fill the GPU together -- at H > 1 a block has only
// l_b / 256 row units per head, and separate launches leave most SMs idle in the tail.
int phase_stage12(spava_host* H, const HostBufs& b, cudaStream_t st, bool with_merge = false) {
  const spava_layer_cfg& c = H->fab->cfg;
  ProbView pv[3] = {block_problem(H, b, 1), block_problem(H, b, 0), anchor_problem(H, b)};
  const int np = H->fab->plan.l_a > 0 ? 3 : 2;
  if (!with_merge) return attention_impl(pv, np, c.hq, c.hkv, c.dh, st, H);
  const MergeJob job = query_merge_job(H, b);
  return attention_impl(pv, np, c.hq, c.hkv, c.dh, st, H, &job);
}

// H > 1 runs the merged launch (measured on one B200, C1 sim: 0.365 -> 0.334 ms per host at
// H = 8, 0.517 -> 0.505 at H = 4); SPAVA_MERGE_STAGES=0 restores the two launches.
bool merged_stages() {
  static const int v = [] {
    const char* e = getenv("SPAVA_MERGE_STAGES");
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}

MergeParams query_merge_params(spava_host* H, const HostBufs& b) {
  const spava_layer_cfg& c = H->fab->cfg;
  const spava_plan& p = H->fab->plan;
  const long long dq = static_cast<long long>(c.hq) * c.dh;
  MergeParams mp{};
  mp.nparts = p.hosts;
  for (int g = 0; g < p.hosts; ++g) {
    mp.out[g] = H->ex->qOut + static_cast<long long>(g) * p.n_t * dq;
    mp.lse[g] = H->ex->qLse + static_cast<long long>(g) * p.n_t * c.hq;
  }
  mp.rows = p.n_t;
  mp.hq = c.hq;
  mp.dh = c.dh;
  mp.ld_part = dq;
  mp.ld_lse = c.hq;
  mp.dst = b.out + (p.l_a + 2LL * p.l_b) * dq * 2;
  mp.ld_dst = dq;
  mp.dst_f32 = 0;
  mp.status = H->status;
  return mp;
}

int phase_merge(spava_host* H, const HostBufs& b, cudaStream_t st) {
  return merge_impl(query_merge_params(H, b), st, H);
}

int nccl_round(spava_fabric* F, Exchange* ex, int r) {
  const spava_plan& p = F->plan;
  const size_t dk = static_cast<size_t>(F->cfg.hkv) * F->cfg.dh;
  const size_t n_kv = static_cast<size_t>(p.l_p) * dk * 2;  // bytes per slot
  uint8_t* K = static_cast<uint8_t*>(ex->passK[r]);
  uint8_t* V = static_cast<uint8_t*>(ex->passV[r]);
  uint8_t* I = reinterpret_cast<uint8_t*>(ex->passIdx[r]);
  uint8_t* C = reinterpret_cast<uint8_t*>(ex->passCnt[r]);
  NCCL_TRY(ncclGroupStart());
  NCCL_TRY(ncclAllGather(K + F->rank * n_kv, K, n_kv, ncclUint8, F->comm, F->comm_stream));
  NCCL_TRY(ncclAllGather(V + F->rank * n_kv, V, n_kv, ncclUint8, F->comm, F->comm_stream));
  NCCL_TRY(ncclAllGather(I + F->rank * p.l_p * 4, I, static_cast<size_t>(p.l_p) * 4, ncclUint8, F->comm,
                         F->comm_stream));
  NCCL_TRY(ncclAllGather(C + F->rank * 4, C, 4, ncclUint8, F->comm, F->comm_stream));
  NCCL_TRY(ncclGroupEnd());
  return SPAVA_OK;
}

int nccl_qround(spava_fabric* F, Exchange* ex) {
  const spava_plan& p = F->plan;
  const size_t dq = static_cast<size_t>(F->cfg.hq) * F->cfg.dh;
  const size_t no = static_cast<size_t>(p.n_t) * dq * 4, nl = static_cast<size_t>(p.n_t) * F->cfg.hq * 4;
  uint8_t* O = reinterpret_cast<uint8_t*>(ex->qOut);
  uint8_t* L = reinterpret_cast<uint8_t*>(ex->qLse);
  NCCL_TRY(ncclGroupStart());
  NCCL_TRY(ncclAllGather(O + F->rank * no, O, no, ncclUint8, F->comm, F->comm_stream));
  NCCL_TRY(ncclAllGather(L + F->rank * nl, L, nl, ncclUint8, F->comm, F->comm_stream));
  NCCL_TRY(ncclGroupEnd());
  return SPAVA_OK;
}

}  // namespace

// ================================================================= C ABI
extern "C" {

const char* spava_last_error(void) { return g_err.c_str(); }
const char* spava_version(void) { return "spava-b200 0.1 (sm_100a)"; }
int spava_device_ok(void) { return device_ok_impl() ? 1 : 0; }
uint64_t spava_kernel_launches(void) { return g_launches.load(); }

int spava_debug_attn_prof(uint64_t* out16) {
  attn_prof_read(reinterpret_cast<unsigned long long*>(out16));
  return SPAVA_OK;
}

int spava_debug_fused_score(int on) {
  g_fused_score.store(on < 0 ? -1 : (on ? 1 : 0));
  return SPAVA_OK;
}

int spava_debug_fused_merge(int on) {
  g_fused_merge.store(on < 0 ? -1 : (on ? 1 : 0));
  return SPAVA_OK;
}

int spava_debug_attn_variant(int variant) {
  if (attn_set_variant(variant) != 0) return fail(SPAVA_EINVAL, "attn_variant: -1, 0, or 1..14 in a dev build (SPAVA_DEV_VARIANTS=1)");
  return SPAVA_OK;
}

int spava_make_plan(int n_v, int n_t, int hosts, int l_a, int l_p, int zigzag, spava_plan* out) {
  return plan_impl(n_v, n_t, hosts, l_a, l_p, zigzag, out);
}

int spava_default_plan(int n, int hosts, spava_plan* out) {
  if (n < 128) return fail(SPAVA_EINVAL, "default_plan: n must be at least 128");
  if (hosts < 1) return fail(SPAVA_EINVAL, "default_plan: need at least one host");
  const int l_a = n / 64, vh = 2 * hosts, rem = n - l_a;
  const int pad = (vh - rem % vh) % vh;
  const int l_b = (rem + pad) / vh;
  if (l_b == 0) return fail(SPAVA_EINVAL, "default_plan: n too small for nonempty blocks");
  *out = spava_plan{n, 0, hosts, l_a, l_b, std::min(n / 128, l_b), pad, vh, 1};
  return SPAVA_OK;
}

int spava_virtual_pair(const spava_plan* p, int h, int* lo, int* hi) {
  if (!p || h < 0 || h >= p->hosts) return fail(SPAVA_ERANGE, "virtual_pair: host index");
  if (p->zigzag) {
    *lo = h;
    *hi = 2 * p->hosts - 1 - h;
  } else {
    *lo = 2 * h;
    *hi = 2 * h + 1;
  }
  return SPAVA_OK;
}

int spava_physical_of(const spava_plan* p, int v, int* h) {
  if (!p || v < 0 || v >= 2 * p->hosts) return fail(SPAVA_ERANGE, "physical_of: virtual index");
  *h = p->zigzag ? (v < p->hosts ? v : 2 * p->hosts - 1 - v) : v / 2;
  return SPAVA_OK;
}

int spava_slice_anchor(int l_a, int hosts, int h, int* begin, int* end) {
  if (h < 0 || h >= hosts) return fail(SPAVA_ERANGE, "slice_anchor: host index");
  const int base = l_a / hosts, extra = l_a % hosts;
  *begin = h * base + std::min(h, extra);
  *end = *begin + base + (h < extra ? 1 : 0);
  return SPAVA_OK;
}

int spava_block_offset(const spava_plan* p, int v) { return p->l_a + v * p->l_b; }
int spava_query_offset(const spava_plan* p) { return p->l_a + p->virtual_hosts * p->l_b; }
int spava_block_valid_rows(const spava_plan* p, int v) { return valid_rows(*p, v); }

int spava_passing_ranges(const spava_plan* p, int v, int* r0b, int* r0e, int* r1b, int* r1e) {
  if (!p || v < 0 || v >= p->virtual_hosts) return fail(SPAVA_ERANGE, "passing_ranges: virtual index");
  passing_range(*p, 0, v, r0b, r0e);
  passing_range(*p, 1, v, r1b, r1e);
  return SPAVA_OK;
}

int spava_pad_mask(const spava_plan* p, int v, uint8_t* mask) {
  if (!p || v < 0 || v >= p->virtual_hosts) return fail(SPAVA_ERANGE, "pad_mask: virtual index");
  for (int r = 0; r < p->l_b; ++r) mask[r] = (p->l_a + v * p->l_b + r) >= p->n_v ? 1 : 0;
  return SPAVA_OK;
}

int spava_split_rows(const spava_plan* p, int h, const void* src, int64_t ld_src_bytes, void* dst,
                     int64_t ld_dst_bytes, int row_bytes, void* stream) {
  if (!p || !src || !dst) return fail(SPAVA_EINVAL, "split_rows: null argument");
  if (h < 0 || h >= p->hosts) return fail(SPAVA_ERANGE, "split_rows: host index");
  int lo, hi;
  ST_TRY(spava_virtual_pair(p, h, &lo, &hi));
  ST_TRY(require_device());
  cudaError_t e = launch_split_rows(p->l_a, p->l_b, p->n_t, p->n_v, lo, hi, src, ld_src_bytes, dst,
                                    ld_dst_bytes, row_bytes, false, false, as_stream(stream));
  if (e != cudaSuccess) return fail(e == cudaErrorInvalidValue ? SPAVA_EINVAL : SPAVA_ECUDA,
                                    "split_rows: rows and strides must be 16-byte multiples");
  ++g_launches;
  return SPAVA_OK;
}

int spava_merge_rows(const spava_plan* p, int h, const void* src, int64_t ld_src_bytes, void* dst,
                     int64_t ld_dst_bytes, int row_bytes, int write_shared, void* stream) {
  if (!p || !src || !dst) return fail(SPAVA_EINVAL, "merge_rows: null argument");
  if (h < 0 || h >= p->hosts) return fail(SPAVA_ERANGE, "merge_rows: host index");
  int lo, hi;
  ST_TRY(spava_virtual_pair(p, h, &lo, &hi));
  ST_TRY(require_device());
  cudaError_t e = launch_split_rows(p->l_a, p->l_b, p->n_t, p->n_v, lo, hi, src, ld_src_bytes, dst,
                                    ld_dst_bytes, row_bytes, true, write_shared != 0, as_stream(stream));
  if (e != cudaSuccess) return fail(e == cudaErrorInvalidValue ? SPAVA_EINVAL : SPAVA_ECUDA,
                                    "merge_rows: rows and strides must be 16-byte multiples");
  ++g_launches;
  return SPAVA_OK;
}

size_t spava_score_workspace(int n_t, int l_b, int hq) { return score_workspace_bytes(n_t, l_b, hq); }

int spava_score_block(const void* q, int64_t ldq, int n_t, const void* k, int64_t ldk, int l_b,
                      const uint8_t* pad, int n_valid, int hq, int hkv, int dh, int softmax,
                      float* scores, void* ws, size_t ws_bytes, void* stream) {
  return spava_score_block_ex(q, ldq, n_t, k, ldk, l_b, pad, n_valid, hq, hkv, dh, softmax, scores, ws,
                              ws_bytes, stream, 0.f);
}

int spava_score_block_ex(const void* q, int64_t ldq, int n_t, const void* k, int64_t ldk, int l_b,
                         const uint8_t* pad, int n_valid, int hq, int hkv, int dh, int softmax,
                         float* scores, void* ws, size_t ws_bytes, void* stream, float scale) {
  if (n_t < 1) return fail(SPAVA_EINVAL, "score_context: empty query");
  if (dh != kHeadDim || hq < 1 || hkv < 1 || hq % hkv || hq > 32)
    return fail(SPAVA_EINVAL, "score_block: need dh == 128, hkv | hq, hq <= 32");
  if (ldq % 8 || ldk % 8) return fail(SPAVA_EINVAL, "score_block: row strides must be multiples of 8");
  if (ws_bytes < score_workspace_bytes(n_t, l_b, hq))
    return fail(SPAVA_EINVAL, "score_block: workspace too small");
  ST_TRY(require_device());
  if (!(scale >= 0.f) || std::isinf(scale)) return fail(SPAVA_EINVAL, "score_block: scale must be finite, >= 0");
  cudaError_t e = launch_score_exact(q, ldq, n_t, k, ldk, l_b, pad, n_valid, hq, hkv, dh, softmax,
                                     scores, ws, ws_bytes, as_stream(stream), scale);
  if (e != cudaSuccess) return fail(SPAVA_ECUDA, std::string("score_block: ") + cudaGetErrorString(e));
  g_launches += softmax ? 3 : 2;
  return SPAVA_OK;
}

size_t spava_score_fast_workspace(int n_t, int l_b, int hq) { return score_fast_workspace_bytes(n_t, l_b, hq); }

int spava_score_block_fast(const void* q, int64_t ldq, int n_t, const void* k, int64_t ldk, int l_b,
                           const uint8_t* pad, int n_valid, int hq, int hkv, int dh,
                           float* scores, void* ws, size_t ws_bytes, void* stream) {
  if (n_t < 1) return fail(SPAVA_EINVAL, "score_context: empty query");
  if (ldq % 8 || ldk % 8) return fail(SPAVA_EINVAL, "score_block_fast: row strides must be multiples of 8");
  ST_TRY(require_device());
  const void* ks[1] = {k};
  const uint8_t* pads[1] = {pad};
  const int nv[1] = {n_valid};
  float* sc[1] = {scores};
  std::string err;
  cudaError_t e = launch_score_fast2(1, q, ldq, n_t, ks, ldk, l_b, pad ? pads : nullptr, nv, hq, hkv, dh,
                                     sc, ws, ws_bytes, as_stream(stream), &err);
  if (e != cudaSuccess)
    return fail(e == cudaErrorInvalidValue ? SPAVA_EINVAL : SPAVA_ECUDA,
                "score_block_fast: " + (err.empty() ? std::string(cudaGetErrorString(e)) : err));
  g_launches += 3;
  return SPAVA_OK;
}

int spava_select_pack(const float* scores, int l_b, int l_p, int global_offset, const void* k,
                      const void* v, int64_t ld, int width, int32_t* idx_out, void* k_out,
                      void* v_out, int64_t ld_out, int32_t* count_out, int32_t* status_out,
                      void* stream) {
  if (l_p < 0 || l_p > l_b) return fail(SPAVA_EINVAL, "select_essential: l_p out of range");
  if (width % 8 || ld % 8 || ld_out % 8)
    return fail(SPAVA_EINVAL, "select_essential: widths/strides must be multiples of 8");
  ST_TRY(require_device());
  cudaError_t e = launch_select_pack(scores, l_b, l_p, global_offset, k, v, ld, width, idx_out, k_out,
                                     v_out, ld_out, count_out, status_out, as_stream(stream));
  if (e != cudaSuccess) return fail(SPAVA_ECUDA, std::string("select_pack: ") + cudaGetErrorString(e));
  g_launches += (l_p > 0 && k_out && v_out) ? 2 : 1;
  return SPAVA_OK;
}

size_t spava_attention_workspace(int nq, int hq, int dh, int splits) {
  if (splits <= 1) return 0;
  return static_cast<size_t>(splits) * nq * hq * (dh + 1) * sizeof(float) + 512;
}

int spava_attention(const void* q, int64_t ldq, int nq, const spava_segment* segs, int nseg,
                    int hq, int hkv, int dh, void* out, int64_t ldo, int out_f32, float* lse,
                    int splits, void* ws, size_t ws_bytes, void* stream) {
  return spava_attention_ex(q, ldq, nq, segs, nseg, hq, hkv, dh, out, ldo, out_f32, lse, splits, ws,
                            ws_bytes, stream, 0.f);
}

int spava_attention_ex(const void* q, int64_t ldq, int nq, const spava_segment* segs, int nseg,
                       int hq, int hkv, int dh, void* out, int64_t ldo, int out_f32, float* lse,
                       int splits, void* ws, size_t ws_bytes, void* stream, float scale) {
  if (!(scale >= 0.f) || std::isinf(scale)) return fail(SPAVA_EINVAL, "attention: scale must be finite, >= 0");
  if (nseg < 0 || nseg > kMaxSegs) return fail(SPAVA_EINVAL, "attention: at most 5 key segments");
  if (splits < 1) splits = 1;
  if (splits > kMaxMergeParts) return fail(SPAVA_EINVAL, "attention: too many splits");
  for (int s = 0; s < nseg; ++s)
    if (segs[s].causal && segs[s].rows > nq)
      return fail(SPAVA_EINVAL, "attention_lse: causal segment must match query rows");
  ST_TRY(require_device());
  ProbView pv{};
  pv.q = q;
  pv.ldq = ldq;
  pv.nq = nq;
  pv.nseg = nseg;
  for (int s = 0; s < nseg; ++s)
    pv.seg[s] = SegView{segs[s].k, segs[s].v, segs[s].ld, segs[s].rows, segs[s].causal};
  cudaStream_t st = as_stream(stream);
  const long long dq = static_cast<long long>(hq) * dh;
  if (splits == 1) {
    pv.out = out;
    pv.ldo = ldo;
    pv.out_f32 = out_f32;
    pv.lse = lse;
    pv.ld_lse = hq;
    pv.splits = 1;
    return attention_impl(&pv, 1, hq, hkv, dh, st, nullptr, nullptr, nullptr, scale);
  }
  if (ws_bytes < spava_attention_workspace(nq, hq, dh, splits))
    return fail(SPAVA_EINVAL, "attention: workspace too small for splits");
  float* po = static_cast<float*>(ws);
  float* pl = po + static_cast<size_t>(splits) * nq * dq;
  pv.out = po;
  pv.ldo = dq;
  pv.out_f32 = 1;
  pv.lse = pl;
  pv.ld_lse = hq;
  pv.splits = splits;
  pv.split_stride_out = static_cast<long long>(nq) * dq;
  pv.split_stride_lse = static_cast<long long>(nq) * hq;
  ST_TRY(attention_impl(&pv, 1, hq, hkv, dh, st, nullptr, nullptr, nullptr, scale));
  MergeParams mp{};
  mp.nparts = splits;
  for (int s = 0; s < splits; ++s) {
    mp.out[s] = po + s * pv.split_stride_out;
    mp.lse[s] = pl + s * pv.split_stride_lse;
  }
  mp.rows = nq;
  mp.hq = hq;
  mp.dh = dh;
  mp.ld_part = dq;
  mp.ld_lse = hq;
  mp.dst = out;
  mp.ld_dst = ldo;
  mp.dst_f32 = out_f32;
  mp.dst_lse = lse;
  return merge_impl(mp, st);
}

int spava_mha_merge(int nparts, const float* const* outs, const float* const* lses, int rows,
                    int64_t ld_part, int hq, int dh, void* dst, int64_t ld_dst, int dst_f32,
                    float* dst_lse, int32_t* status, void* stream) {
  if (nparts < 1) return fail(SPAVA_EINVAL, "mha_merge: empty part list");
  if (nparts > kMaxMergeParts) return fail(SPAVA_EINVAL, "mha_merge: too many parts");
  ST_TRY(require_device());
  MergeParams mp{};
  mp.nparts = nparts;
  for (int i = 0; i < nparts; ++i) {
    mp.out[i] = outs[i];
    mp.lse[i] = lses[i];
  }
  mp.rows = rows;
  mp.hq = hq;
  mp.dh = dh;
  mp.ld_part = ld_part;
  mp.ld_lse = hq;
  mp.dst = dst;
  mp.ld_dst = ld_dst;
  mp.dst_f32 = dst_f32;
  mp.dst_lse = dst_lse;
  mp.status = status;
  return merge_impl(mp, as_stream(stream));
}

// ------------------------------------------------------------- fabric/host
int spava_fabric_create_local(const spava_layer_cfg* cfg, int device, spava_fabric** out) {
  spava_plan plan;
  ST_TRY(cfg_check(cfg, &plan));
  CU_TRY(cudaSetDevice(device));
  ST_TRY(require_device());
  auto* F = new spava_fabric();
  F->cfg = *cfg;
  F->plan = plan;
  F->device = device;
  int s = F->shared.alloc(*cfg, plan);
  if (s != SPAVA_OK) {
    delete F;
    return s;
  }
  *out = F;
  return SPAVA_OK;
}

int spava_nccl_unique_id(void* uid) {
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  std::memcpy(uid, &id, sizeof(id));
  return SPAVA_OK;
}

int spava_fabric_create_nccl(const spava_layer_cfg* cfg, int device, const void* uid, int world,
                             int rank, spava_fabric** out) {
  spava_plan plan;
  ST_TRY(cfg_check(cfg, &plan));
  if (world != cfg->hosts) return fail(SPAVA_EINVAL, "nccl fabric: world size must equal hosts");
  if (rank < 0 || rank >= world) return fail(SPAVA_ERANGE, "nccl fabric: rank");
  CU_TRY(cudaSetDevice(device));
  ST_TRY(require_device());
  auto* F = new spava_fabric();
  F->cfg = *cfg;
  F->plan = plan;
  F->device = device;
  F->nccl = true;
  F->world = world;
  F->rank = rank;
  ncclUniqueId id;
  std::memcpy(&id, uid, sizeof(id));
  ncclResult_t r = ncclCommInitRank(&F->comm, world, id, rank);
  if (r != ncclSuccess) {
    delete F;
    return fail(SPAVA_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  }
  const cudaError_t e = cudaStreamCreateWithFlags(&F->comm_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    spava_fabric_destroy(F);
    return fail(SPAVA_ECUDA, std::string("nccl fabric: comm stream: ") + cudaGetErrorString(e));
  }
  *out = F;
  return SPAVA_OK;
}

int spava_fabric_create_peer(const spava_layer_cfg* cfg, int device, int world, int rank,
                             int64_t encode_bytes, spava_fabric** out) {
  if (encode_bytes < 0) return fail(SPAVA_EINVAL, "peer fabric: encode_bytes");
  spava_plan plan;
  ST_TRY(cfg_check(cfg, &plan));
  if (world != cfg->hosts) return fail(SPAVA_EINVAL, "peer fabric: world size must equal hosts");
  if (world > kMaxPeers + 1) return fail(SPAVA_EINVAL, "peer fabric: at most 8 GPUs");
  if (rank < 0 || rank >= world) return fail(SPAVA_ERANGE, "peer fabric: rank");
  CU_TRY(cudaSetDevice(device));
  ST_TRY(require_device());
  auto* F = new spava_fabric();
  F->cfg = *cfg;
  F->plan = plan;
  F->device = device;
  F->peer = true;
  F->world = world;
  F->rank = rank;
  const int s = F->shared.alloc(*cfg, plan, static_cast<size_t>(encode_bytes));
  if (s != SPAVA_OK) {
    delete F;
    return s;
  }
  F->peer_base[rank] = static_cast<uint8_t*>(F->shared.base);
  F->peer_ready = world == 1;
  *out = F;
  return SPAVA_OK;
}

int spava_fabric_peer_handle(spava_fabric* F, void* handle) {
  if (!F || !F->peer) return fail(SPAVA_EINVAL, "peer_handle: not a peer fabric");
  if (!handle) return fail(SPAVA_EINVAL, "peer_handle: null handle buffer");
  static_assert(sizeof(cudaIpcMemHandle_t) == SPAVA_PEER_HANDLE_BYTES, "IPC handle size");
  CU_TRY(cudaSetDevice(F->device));
  cudaIpcMemHandle_t h;
  CU_TRY(cudaIpcGetMemHandle(&h, F->shared.base));
  std::memcpy(handle, &h, sizeof(h));
  return SPAVA_OK;
}

int spava_fabric_peer_open(spava_fabric* F, const void* handles) {
  if (!F || !F->peer) return fail(SPAVA_EINVAL, "peer_open: not a peer fabric");
  if (F->peer_ready) return fail(SPAVA_EINVAL, "peer_open: peers already open");
  if (!handles) return fail(SPAVA_EINVAL, "peer_open: null handles");
  CU_TRY(cudaSetDevice(F->device));
  const auto* hb = static_cast<const uint8_t*>(handles);
  for (int q = 0; q < F->world; ++q) {
    if (q == F->rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, hb + static_cast<size_t>(q) * SPAVA_PEER_HANDLE_BYTES, sizeof(h));
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(SPAVA_ECUDA, std::string("peer_open: rank ") + std::to_string(q) + ": " + cudaGetErrorString(e));
    F->peer_base[q] = static_cast<uint8_t*>(p);
    F->peer_ipc[q] = true;
  }
  F->peer_ready = true;
  return SPAVA_OK;
}

int spava_fabric_peer_attach(spava_fabric* const* fabrics, int world) {
  if (!fabrics || world < 1) return fail(SPAVA_EINVAL, "peer_attach: no fabrics");
  for (int r = 0; r < world; ++r) {
    const spava_fabric* F = fabrics[r];
    if (!F || !F->peer || F->world != world || F->rank != r || F->peer_ready != (world == 1))
      return fail(SPAVA_EINVAL, "peer_attach: fabrics[r] must be a fresh peer fabric of rank r");
    if (F->device != fabrics[0]->device) return fail(SPAVA_EINVAL, "peer_attach: one device only");
  }
  for (int r = 0; r < world; ++r)
    for (int q = 0; q < world; ++q) fabrics[r]->peer_base[q] = static_cast<uint8_t*>(fabrics[q]->shared.base);
  for (int r = 0; r < world; ++r) fabrics[r]->peer_ready = true;
  return SPAVA_OK;
}

// ------------------------------------------------- frame-parallel encode gather (f4)
int spava_frame_partition(int frames, int hosts, int* counts) {
  if (hosts < 1) return fail(SPAVA_EINVAL, "frame_partition: need at least one host");
  if (!counts) return fail(SPAVA_EINVAL, "frame_partition: null counts");
  for (int h = 0; h < hosts; ++h) counts[h] = frames / hosts + (h < frames % hosts ? 1 : 0);
  return SPAVA_OK;
}

namespace {
int make_parts(const spava_plan* p, const void* const* parts, const int64_t* part_rows, int64_t ld,
               GatherParts* gp) {
  if (p->hosts > kMaxPeers + 1) return fail(SPAVA_EINVAL, "gather_split: at most 8 hosts");
  gp->n = p->hosts;
  gp->ld = ld;
  gp->off[0] = 0;
  for (int q = 0; q < p->hosts; ++q) {
    if (part_rows[q] < 0) return fail(SPAVA_EINVAL, "gather_split: negative part rows");
    if (part_rows[q] > 0 && !parts[q]) return fail(SPAVA_EINVAL, "gather_split: null part");
    gp->base[q] = parts[q];
    gp->off[q + 1] = gp->off[q] + part_rows[q];
  }
  // concat_rows of the gathered parts is E_v (simhost.cpp:296-298)
  if (gp->off[p->hosts] != p->n_v) return fail(SPAVA_EINVAL, "gather_split: part rows must sum to n_v");
  return SPAVA_OK;
}

int gather_split_impl(const spava_plan* p, int h, const GatherParts& gp, const void* e_q, int64_t ld_q,
                      void* dst, int64_t ld_dst, int row_bytes, cudaStream_t st) {
  int lo, hi;
  ST_TRY(spava_virtual_pair(p, h, &lo, &hi));
  cudaError_t e = launch_gather_split(p->l_a, p->l_b, p->n_t, p->n_v, lo, hi, gp, e_q, ld_q, dst, ld_dst,
                                      row_bytes, st);
  if (e != cudaSuccess)
    return fail(e == cudaErrorInvalidValue ? SPAVA_EINVAL : SPAVA_ECUDA,
                "gather_split: rows, strides and pointers must be 16-byte aligned");
  ++g_launches;
  return SPAVA_OK;
}
}  // namespace

int spava_gather_split_rows(const spava_plan* p, int h, const void* const* parts, const int64_t* part_rows,
                            int64_t ld_part_bytes, const void* e_q, int64_t ld_q_bytes, void* dst,
                            int64_t ld_dst_bytes, int row_bytes, void* stream) {
  if (!p || !parts || !part_rows || !dst || (p->n_t > 0 && !e_q))
    return fail(SPAVA_EINVAL, "gather_split_rows: null argument");
  if (h < 0 || h >= p->hosts) return fail(SPAVA_ERANGE, "gather_split_rows: host index");
  ST_TRY(require_device());
  GatherParts gp{};
  ST_TRY(make_parts(p, parts, part_rows, ld_part_bytes, &gp));
  return gather_split_impl(p, h, gp, e_q, ld_q_bytes, dst, ld_dst_bytes, row_bytes, as_stream(stream));
}

int spava_fabric_encode_region(spava_fabric* F, void** ptr, int64_t* bytes) {
  if (!F || !F->peer) return fail(SPAVA_EINVAL, "encode_region: not a peer fabric");
  if (ptr) *ptr = F->shared.encode;
  if (bytes) *bytes = static_cast<int64_t>(F->shared.encode_bytes);
  return SPAVA_OK;
}

int spava_fabric_encode_acquire(spava_fabric* F, void* stream) {
  if (!F || !F->peer || !F->peer_ready) return fail(SPAVA_EINVAL, "encode_acquire: peer fabric not open");
  CU_TRY(cudaSetDevice(F->device));
  if (F->enc_epoch == 0) return SPAVA_OK;
  int n = 0;
  for (int q = 0; q < F->world; ++q)
    if (q != F->rank) F->flag_tmp[n++] = F->shared.flags + Exchange::kDoneEnc + q;
  CU_TRY(stream_wait_all_geq_u32(as_stream(stream), F->flag_tmp, n, F->enc_epoch));
  return SPAVA_OK;
}

int spava_host_gather_context(spava_host* H, const int64_t* part_rows, int64_t ld_part_bytes, const void* e_q,
                              int64_t ld_q_bytes, void* dst, int64_t ld_dst_bytes, int row_bytes, void* stream) {
  if (!H || !part_rows || !dst) return fail(SPAVA_EINVAL, "gather_context: null argument");
  spava_fabric* F = H->fab;
  if (!F->peer || !F->peer_ready) return fail(SPAVA_EINVAL, "gather_context: needs an open peer fabric");
  if (!F->shared.encode) return fail(SPAVA_EINVAL, "gather_context: fabric created with encode_bytes = 0");
  const spava_plan& p = F->plan;
  for (int q = 0; q < p.hosts; ++q)
    if (part_rows[q] < 0 || static_cast<uint64_t>(part_rows[q]) * static_cast<uint64_t>(ld_part_bytes) >
                                F->shared.encode_bytes)
      return fail(SPAVA_EINVAL, "gather_context: a host's part exceeds the encode region");
  CU_TRY(cudaSetDevice(F->device));
  cudaStream_t st = as_stream(stream);
  std::vector<const void*> parts(p.hosts);
  for (int q = 0; q < p.hosts; ++q) parts[q] = F->at_peer(q, static_cast<uint8_t*>(F->shared.encode));
  GatherParts gp{};
  ST_TRY(make_parts(&p, parts.data(), part_rows, ld_part_bytes, &gp));
  const uint32_t e = ++F->enc_epoch;
  uint32_t* fl = F->shared.flags;
  // the encoder's writes to this rank's region precede this call on `stream`: announce them
  int n = 0;
  for (int q = 0; q < F->world; ++q)
    if (q != F->rank) F->flag_tmp[n++] = F->at_peer(q, fl) + Exchange::kArrive + 3 * 256 + F->rank;
  CU_TRY(peer_flags_store(st, F->flag_tmp, n, e));
  if (n > 0) ++g_launches;
  n = 0;
  for (int q = 0; q < F->world; ++q)
    if (q != F->rank) F->flag_tmp[n++] = fl + Exchange::kArrive + 3 * 256 + q;
  CU_TRY(stream_wait_all_geq_u32(st, F->flag_tmp, n, e));
  ST_TRY(gather_split_impl(&p, H->h, gp, e_q, ld_q_bytes, dst, ld_dst_bytes, row_bytes, st));
  n = 0;
  for (int q = 0; q < F->world; ++q)  // this rank has read every peer's region
    if (q != F->rank) F->flag_tmp[n++] = F->at_peer(q, fl) + Exchange::kDoneEnc + F->rank;
  CU_TRY(peer_flags_store(st, F->flag_tmp, n, e));
  if (n > 0) ++g_launches;
  return SPAVA_OK;
}

int spava_fabric_destroy(spava_fabric* F) {
  if (!F) return SPAVA_OK;
  for (int q = 0; q < kMaxMergeParts; ++q)
    if (F->peer_ipc[q]) cudaIpcCloseMemHandle(F->peer_base[q]);
  if (F->comm) ncclCommDestroy(F->comm);
  if (F->comm_stream) cudaStreamDestroy(F->comm_stream);
  if (F->trace_base) cudaEventDestroy(F->trace_base);
  F->shared.release();
  delete F;
  return SPAVA_OK;
}

namespace {
int host_init_streams(spava_host* H) {
  for (auto& e : H->ev) CU_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CU_TRY(cudaEventCreateWithFlags(&H->ev_fork, cudaEventDisableTiming));
  CU_TRY(cudaEventCreateWithFlags(&H->ev_sel, cudaEventDisableTiming));
  CU_TRY(cudaEventCreateWithFlags(&H->ev_score, cudaEventDisableTiming));
  int prio_lo = 0, prio_hi = 0;
  CU_TRY(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  CU_TRY(cudaStreamCreateWithPriority(&H->side, cudaStreamNonBlocking, prio_hi));
  CU_TRY(cudaStreamCreateWithPriority(&H->side_lo, cudaStreamNonBlocking, prio_lo));
  CU_TRY(cudaStreamCreateWithFlags(&H->h2d, cudaStreamNonBlocking));
  CU_TRY(cudaStreamCreateWithFlags(&H->d2h, cudaStreamNonBlocking));
  CU_TRY(cudaEventCreateWithFlags(&H->ev_kvq, cudaEventDisableTiming));
  CU_TRY(cudaEventCreateWithFlags(&H->ev_vhi, cudaEventDisableTiming));
  CU_TRY(cudaEventCreateWithFlags(&H->ev_d2h, cudaEventDisableTiming));
  for (auto& e : H->ev_qc) CU_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : H->ev_oc) CU_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return SPAVA_OK;
}
}  // namespace

int spava_host_create(spava_fabric* F, int h, spava_host** out) {
  if (!F) return fail(SPAVA_EINVAL, "host_create: null fabric");
  const spava_plan& p = F->plan;
  const spava_layer_cfg& c = F->cfg;
  if (h < 0 || h >= p.hosts) return fail(SPAVA_ERANGE, "host_create: host index");
  if ((F->nccl || F->peer) && h != F->rank) return fail(SPAVA_EINVAL, "host_create: nccl/peer host must equal rank");
  CU_TRY(cudaSetDevice(F->device));
  auto* H = new spava_host();
  H->fab = F;
  H->h = h;
  spava_virtual_pair(&p, h, &H->v_lo, &H->v_hi);
  spava_slice_anchor(p.l_a, p.hosts, h, &H->a0, &H->a1);
  const int designated = c.designated < 0 ? p.hosts - 1 : c.designated;
  H->self_keys = c.query_self_all || h == designated;
  const int keys = (H->a1 - H->a0) + 2 * p.l_b + (H->self_keys ? p.n_t : 0);
  H->splits = c.query_splits > 0 ? std::min(c.query_splits, kMaxMergeParts) : auto_splits(p.n_t, c.hq, c.hkv, keys);
  if (F->nccl) {
    int s = H->own.alloc(c, p);
    if (s != SPAVA_OK) {
      delete H;
      return s;
    }
    H->ex = &H->own;
  } else {
    H->ex = &F->shared;
  }
  const size_t dq = static_cast<size_t>(c.hq) * c.dh;
  H->score_ws_bytes = std::max(score_workspace_bytes(p.n_t, p.l_b, c.hq),
                               score_fast_workspace_bytes(p.n_t, p.l_b, c.hq));
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  const size_t sc = al(static_cast<size_t>(p.l_b) * 4);
  const size_t qo = al(static_cast<size_t>(H->splits) * p.n_t * dq * 4);
  const size_t ql = al(static_cast<size_t>(H->splits) * p.n_t * c.hq * 4);
  const size_t total = 2 * sc + al(H->score_ws_bytes) + qo + ql + 256;
  if (cudaMalloc(&H->base, total) != cudaSuccess) {
    delete H;
    return fail(SPAVA_ECUDA, "host_create: out of device memory");
  }
  cudaMemset(H->base, 0, total);
  uint8_t* b = static_cast<uint8_t*>(H->base);
  H->scores[0] = reinterpret_cast<float*>(b); b += sc;
  H->scores[1] = reinterpret_cast<float*>(b); b += sc;
  H->score_ws = b; b += al(H->score_ws_bytes);
  H->qsplit_out = reinterpret_cast<float*>(b); b += qo;
  H->qsplit_lse = reinterpret_cast<float*>(b); b += ql;
  H->status = reinterpret_cast<int32_t*>(b);
  H->ctr = reinterpret_cast<unsigned*>(b + 64);
  const int rc = host_init_streams(H);
  if (rc != SPAVA_OK) {
    spava_host_destroy(H);  // releases whatever was created before the failure
    return rc;
  }
  *out = H;
  return SPAVA_OK;
}

int spava_host_destroy(spava_host* H) {
  if (!H) return SPAVA_OK;
  for (auto& e : H->ev)
    if (e) cudaEventDestroy(e);
  if (H->ev_fork) cudaEventDestroy(H->ev_fork);
  if (H->ev_score) cudaEventDestroy(H->ev_score);
  if (H->ev_sel) cudaEventDestroy(H->ev_sel);
  if (H->graph_exec) cudaGraphExecDestroy(H->graph_exec);
  if (H->graph) cudaGraphDestroy(H->graph);
  if (H->side) cudaStreamDestroy(H->side);
  if (H->side_lo) cudaStreamDestroy(H->side_lo);
  if (H->h2d) cudaStreamDestroy(H->h2d);
  if (H->d2h) cudaStreamDestroy(H->d2h);
  for (auto& e : H->ev_qc)
    if (e) cudaEventDestroy(e);
  for (auto& e : H->ev_oc)
    if (e) cudaEventDestroy(e);
  if (H->ev_kvq) cudaEventDestroy(H->ev_kvq);
  if (H->ev_vhi) cudaEventDestroy(H->ev_vhi);
  if (H->ev_d2h) cudaEventDestroy(H->ev_d2h);
  for (auto& e : H->ev_pool) cudaEventDestroy(e);
  for (auto& e : H->trace_pool) cudaEventDestroy(e);
  H->own.release();
  if (H->base) cudaFree(H->base);
  delete H;
  return SPAVA_OK;
}

int spava_host_plan(const spava_host* H, spava_plan* out) {
  *out = H->fab->plan;
  return SPAVA_OK;
}

int spava_host_rows(const spava_host* H) {
  const spava_plan& p = H->fab->plan;
  return p.l_a + 2 * p.l_b + p.n_t;
}


namespace {

// Optional host<->device copy pipeline around one layer: each compute phase waits only for
// the rows it reads (ev_in) and each finished output row range is copied back while later
// phases still run (ev_out).  Inputs arrive in the order the phases need them.
struct CopyEdges {
  bool on = false;
  int n = 0;                                  // row chunks per block
  int cb[spava_host::kCopyChunks + 1] = {};  // row bounds of the block chunks
};

CopyEdges copy_edges(const spava_plan& p) {
  // uneven row chunks (multiples of 256 rows, one ping-pong CTA unit): block lo runs its
  // chunks in row order and block hi in REVERSE order, so the first output is ready early
  // (small first lo chunks) and the last chunks to arrive are the smallest and lightest
  // (causal rows [0, l_b/16) of hi) -- the tail after the last H2D byte is short.  Eleven
  // chunks per block keep the D2H stream fed between chunks (C1 e2e 4.19 -> 4.11 ms against
  // five, tools/e2e_chunks.sh).  SPAVA_COPY_CHUNKS="0,..,32" (fractions of 32, dev A/B)
  // overrides the table.
  static const std::vector<int> frac = [] {
    std::vector<int> f = {0, 1, 2, 4, 6, 8, 12, 16, 20, 24, 28, 32};
    if (const char* e = getenv("SPAVA_COPY_CHUNKS")) {
      std::vector<int> g;
      for (const char* c = e; *c;) {
        g.push_back(atoi(c));
        while (*c && *c != ',') ++c;
        if (*c) ++c;
      }
      if (g.size() >= 2 && g.size() <= spava_host::kCopyChunks + 1 && g.front() == 0 && g.back() == 32) f = g;
    }
    return f;
  }();
  CopyEdges cp;
  cp.on = true;
  cp.n = static_cast<int>(frac.size()) - 1;
  for (int c = 0; c <= cp.n; ++c) {
    const long long r = (static_cast<long long>(p.l_b) * frac[c] / 32 + 255) / 256 * 256;
    cp.cb[c] = static_cast<int>(std::min<long long>(r, p.l_b));
  }
  cp.cb[cp.n] = p.l_b;
  return cp;
}

// row chunk of block `which` processed at position k (hi runs in reverse)
inline int chunk_of(const CopyEdges& cp, int which, int k) { return which == 0 ? k : cp.n - 1 - k; }

// stage 1 / stage 2 as row chunks (copy pipeline) or whole blocks; events are indexed by
// processing position
int stage_chunks(spava_host* H, const HostBufs& b, cudaStream_t st, const CopyEdges& cp, int which,
                 bool with_merge = false) {
  if (!cp.on) return which == 0 ? phase_stage1(H, b, st) : phase_stage2(H, b, st, with_merge);
  const spava_layer_cfg& c = H->fab->cfg;
  const int n = cp.n;
  for (int k = 0; k < n; ++k) {
    const int idx = which * n + k, rc = chunk_of(cp, which, k);
    CU_TRY(cudaStreamWaitEvent(st, H->ev_qc[idx], 0));
    const bool anchor = which == 0 && k == 0 && H->fab->plan.l_a > 0;  // anchor with lo chunk 0
    if (cp.cb[rc + 1] > cp.cb[rc]) {
      ProbView pv[2] = {block_chunk_problem(H, b, which, cp.cb[rc], cp.cb[rc + 1]), anchor_problem(H, b)};
      ST_TRY(attention_impl(pv, anchor ? 2 : 1, c.hq, c.hkv, c.dh, st, H));
    } else if (anchor) {
      ProbView pa = anchor_problem(H, b);
      ST_TRY(attention_impl(&pa, 1, c.hq, c.hkv, c.dh, st, H));
    }
    CU_TRY(cudaEventRecord(H->ev_oc[idx], st));
  }
  return SPAVA_OK;
}

// dev A/B: SPAVA_SERIAL_SCORE=1 runs the scorer on the caller's stream (no overlap) in the
// device-resident layer
bool serial_score_env() {
  static const bool v = [] {
    const char* e = getenv("SPAVA_SERIAL_SCORE");
    return e && atoi(e) != 0;
  }();
  return v;
}

int layer_impl(spava_host* H, const HostBufs& b, cudaStream_t st, const CopyEdges& cp) {
  spava_fabric* F = H->fab;
  cudaStream_t ss = (H->serial || (!cp.on && serial_score_env())) ? st : cp.on ? H->side_lo : H->side;
  auto merged = [&](cudaStream_t s) -> cudaError_t {
    return cp.on ? cudaEventRecord(H->ev_oc[2 * cp.n], s) : cudaSuccess;
  };
  // trace records follow run_host's overlapped program order (simhost.cpp:343-426)
  auto T = [&](cudaStream_t s, int kind, const char* label, bool comm = false) {
    trace_ev(H, s, kind, label, comm);
  };
  // host-buffer pipeline (cp.on): the side stream starts once all k and the query rows are
  // in (scorer); select hi additionally waits for v of block hi; the caller's stream waits
  // per row chunk, and the query attention (it reads every key) runs after stage 1
  cudaEvent_t before_hi = cp.on ? H->ev_vhi : nullptr;
  // fork: scoring + selection on the side stream (its inputs are this step's q/k on st)
  CU_TRY(cudaEventRecord(H->ev_fork, st));
  CU_TRY(cudaStreamWaitEvent(ss, H->ev_fork, 0));
  if (cp.on) CU_TRY(cudaStreamWaitEvent(ss, H->ev_kvq, 0));
  CU_TRY(launch_delay(H->delay_ns[0], ss));
  CU_TRY(launch_delay(H->delay_ns[2], st));
  const bool fscore = fused_score(H, cp.on);  // N1: scorer inside the query launch
  if (!F->nccl && !F->peer) {
    // H = 1: block lo (v = 0) has no passing segment, so only stage 2 waits for selection
    auto query = [&](cudaStream_t qs) -> int {
      T(qs, kComputeBegin, "query_attn");
      if (cp.on) CU_TRY(cudaStreamWaitEvent(qs, H->ev_vhi, 0));
      ST_TRY(phase_query(H, b, qs, false, fscore));
      T(qs, kComputeEnd, "query_attn");
      T(qs, kCommIssued, "qpartial", true);
      return SPAVA_OK;
    };
    // fused scorer: the query launch (which now also scores) goes on the side stream ahead
    // of select, so stage 1 on the caller's stream overlaps it; stage 2 joins via ev_sel
    if (fscore) ST_TRY(query(ss));
    ST_TRY(phase_select(H, b, ss, false, before_hi, fscore ? 1 : 0));
    CU_TRY(cudaEventRecord(H->ev_sel, ss));
    timeline().mark("select done", ss);
    T(ss, kCommIssued, "pass1", true);
    T(ss, kCommIssued, "pass2", true);
    if (!cp.on && !fscore) ST_TRY(query(st));
    T(st, kCommWaitStart, "pass1", true);
    T(st, kCommCompleted, "pass1", true);
    CU_TRY(launch_delay(H->delay_ns[3], st));
    T(st, kComputeBegin, "stage1");
    ST_TRY(stage_chunks(H, b, st, cp, 0));
    T(st, kComputeEnd, "stage1");
    timeline().mark("stage1 done", st);
    if (cp.on) ST_TRY(query(st));
    timeline().mark("query done", st);
    T(st, kCommWaitStart, "pass2", true);
    CU_TRY(cudaStreamWaitEvent(st, H->ev_sel, 0));
    T(st, kCommCompleted, "pass2", true);
    timeline().mark("stage2 start", st);
    // the merge of the query partial(s) rides in the stage-2 launch (trailing CTAs)
    const bool fused = !cp.on && fused_merge_enabled();
    T(st, kComputeBegin, "stage2");
    ST_TRY(stage_chunks(H, b, st, cp, 1, fused));
    T(st, kComputeEnd, "stage2");
    T(st, kCommWaitStart, "qpartial", true);
    T(st, kCommCompleted, "qpartial", true);
    T(st, kComputeBegin, "merge");
    if (!fused) ST_TRY(phase_merge(H, b, st));
    T(st, kComputeEnd, "merge");
    if (H->trace) ++H->trace_layer;
    return merged(st) == cudaSuccess ? SPAVA_OK : fail(SPAVA_ECUDA, "event record");
  }
  // exchange rounds: NCCL in-place allgathers on the comm stream, or (peer fabric) stores
  // by the producing kernels into every peer's slot + epoch flags (no comm stream)
  cudaStream_t cs = F->comm_stream;
  if (F->peer) {
    if (!F->peer_ready) return fail(SPAVA_EINVAL, "peer fabric: peers not opened");
    ++F->epoch;
    ST_TRY(peer_wait_done(F, ss));  // peers have released the previous epoch's slots
    ST_TRY(peer_wait_done(F, st));
  }
  // peer fabric: the final query merge rides in the merged stage launch (receive side)
  const bool fused_merge = F->peer && !cp.on && merged_stages() && fused_merge_enabled();
  auto query = [&]() -> int {
    T(st, kComputeBegin, "query_attn");
    if (cp.on) CU_TRY(cudaStreamWaitEvent(st, H->ev_vhi, 0));
    ST_TRY(phase_query(H, b, st, true, fscore));  // overlaps scoring and the pass rounds
    T(st, kComputeEnd, "query_attn");
    if (F->peer) {
      T(st, kCommIssued, "qpartial", true);
    } else {
      CU_TRY(cudaStreamWaitEvent(cs, H->ev[2], 0));
      T(cs, kCommIssued, "qpartial", true);
      ST_TRY(nccl_qround(F, H->ex));
      CU_TRY(cudaEventRecord(H->ev[5], cs));
    }
    return SPAVA_OK;
  };
  if (fscore) ST_TRY(query());  // first: it produces the scores select waits for
  ST_TRY(phase_select(H, b, ss, true, before_hi, fscore ? 2 : 0));  // records pass1_ready, pass2_ready on ss
  CU_TRY(cudaEventRecord(H->ev_sel, ss));
  if (F->peer) {
    T(ss, kCommIssued, "pass1", true);
    T(ss, kCommIssued, "pass2", true);
  } else {
    CU_TRY(cudaStreamWaitEvent(cs, H->ev[0], 0));
    CU_TRY(launch_delay(H->delay_ns[1], cs));
    T(cs, kCommIssued, "pass1", true);
    ST_TRY(nccl_round(F, H->ex, 0));
    CU_TRY(cudaEventRecord(H->ev[3], cs));
    CU_TRY(cudaStreamWaitEvent(cs, H->ev[1], 0));
    T(cs, kCommIssued, "pass2", true);
    ST_TRY(nccl_round(F, H->ex, 1));
    CU_TRY(cudaEventRecord(H->ev[4], cs));
  }
  if (!cp.on && !fscore) ST_TRY(query());
  // st waits for round k (0 pass1, 1 pass2, 2 qpartial) of every host
  auto wait_round = [&](int k) -> int {
    if (!F->peer) {
      CU_TRY(cudaStreamWaitEvent(st, H->ev[3 + k], 0));
      return SPAVA_OK;
    }
    ST_TRY(peer_wait_arrive(F, st, k));
    if (k < 2) CU_TRY(cudaStreamWaitEvent(st, H->ev[k], 0));  // own slot, written on ss
    return SPAVA_OK;
  };
  T(st, kCommWaitStart, "pass1", true);
  ST_TRY(wait_round(0));
  T(st, kCommCompleted, "pass1", true);
  if (!F->plan.zigzag) {  // simhost.cpp:392-402
    T(st, kCommWaitStart, "pass2", true);
    ST_TRY(wait_round(1));
    T(st, kCommCompleted, "pass2", true);
  }
  CU_TRY(launch_delay(H->delay_ns[3], st));
  if (!cp.on && merged_stages()) {  // both rounds in, then one launch for both blocks
    if (F->plan.zigzag) {
      T(st, kCommWaitStart, "pass2", true);
      ST_TRY(wait_round(1));
      T(st, kCommCompleted, "pass2", true);
    }
    CU_TRY(cudaStreamWaitEvent(st, H->ev_sel, 0));
    T(st, kComputeBegin, "stage1");
    T(st, kComputeBegin, "stage2");
    ST_TRY(phase_stage12(H, b, st, fused_merge));
    T(st, kComputeEnd, "stage1");
    T(st, kComputeEnd, "stage2");
  } else {
    T(st, kComputeBegin, "stage1");
    ST_TRY(stage_chunks(H, b, st, cp, 0));
    T(st, kComputeEnd, "stage1");
    if (cp.on) ST_TRY(query());
    if (F->plan.zigzag) {
      T(st, kCommWaitStart, "pass2", true);
      ST_TRY(wait_round(1));
      T(st, kCommCompleted, "pass2", true);
    }
    CU_TRY(cudaStreamWaitEvent(st, H->ev_sel, 0));  // join the side stream (sel copy-out)
    T(st, kComputeBegin, "stage2");
    ST_TRY(stage_chunks(H, b, st, cp, 1));
    T(st, kComputeEnd, "stage2");
  }
  T(st, kCommWaitStart, "qpartial", true);
  if (!fused_merge) ST_TRY(wait_round(2));  // else: the stage launch's merge CTAs waited
  T(st, kCommCompleted, "qpartial", true);
  T(st, kComputeBegin, "merge");
  if (!fused_merge) ST_TRY(phase_merge(H, b, st));
  T(st, kComputeEnd, "merge");
  if (F->peer) ST_TRY(peer_release(F, st));  // the exchange buffer of this epoch is read
  if (H->trace) ++H->trace_layer;
  return merged(st) == cudaSuccess ? SPAVA_OK : fail(SPAVA_ECUDA, "event record");
}

}  // namespace

int spava_host_layer(spava_host* H, const void* q, const void* k, const void* v, void* out,
                     int32_t* sel, void* stream) {
  spava_fabric* F = H->fab;
  if (!F->nccl && !F->peer && F->plan.hosts != 1)
    return fail(SPAVA_EINVAL, "host_layer: local fabric with H > 1 must be driven by spava_sim_layer");
  CU_TRY(cudaSetDevice(F->device));
  HostBufs b{static_cast<const uint8_t*>(q), static_cast<const uint8_t*>(k),
             static_cast<const uint8_t*>(v), static_cast<uint8_t*>(out), sel};
  return layer_impl(H, b, as_stream(stream), CopyEdges{});
}


int spava_host_layer_hostbuf(spava_host* H, const void* q_h, const void* k_h, const void* v_h,
                             void* out_h, int32_t* sel_h, void* q_d, void* k_d, void* v_d,
                             void* out_d, int32_t* sel_d, void* stream) {
  spava_fabric* F = H->fab;
  if (!F->nccl && !F->peer && F->plan.hosts != 1)
    return fail(SPAVA_EINVAL, "host_layer_hostbuf: local fabric with H > 1 must be driven by spava_sim_layer");
  if (!q_h || !k_h || !v_h || !out_h || !q_d || !k_d || !v_d || !out_d)
    return fail(SPAVA_EINVAL, "host_layer_hostbuf: null buffer");
  CU_TRY(cudaSetDevice(F->device));
  const spava_layer_cfg& c = F->cfg;
  const spava_plan& p = F->plan;
  cudaStream_t st = as_stream(stream);
  const size_t rq = static_cast<size_t>(c.hq) * c.dh * 2, rk = static_cast<size_t>(c.hkv) * c.dh * 2;
  const size_t rows = static_cast<size_t>(p.l_a) + 2ull * p.l_b + p.n_t;
  const size_t qrow = static_cast<size_t>(p.l_a) + 2ull * p.l_b, lo_end = static_cast<size_t>(p.l_a) + p.l_b;
  auto* qd = static_cast<uint8_t*>(q_d);
  auto* od = static_cast<uint8_t*>(out_d);
  const auto* qh = static_cast<const uint8_t*>(q_h);
  auto* oh = static_cast<uint8_t*>(out_h);
  cudaStream_t hs = H->h2d, ds = H->d2h;
  // inputs, in the order the phases consume them (the previous step's work on st is done
  // before the buffers are overwritten: h2d waits for the fork point of this step):
  //   k, v of [anchor | lo]  ->  q query rows  ->  q lo chunk 0 (+ anchor rows)  -> k of
  //   [hi | query] (ev_kvq: the scorer starts)  ->  q lo chunks 1..  ->  v of [hi | query]
  //   (ev_vhi: select hi, query attention)  ->  q hi chunks, heaviest (last rows) first
  const CopyEdges cp = copy_edges(p);
  const int nc = cp.n;
  const size_t lo_rows = lo_end, rest = rows - lo_end;
  Timeline& TL = timeline();
  auto* kd = static_cast<uint8_t*>(k_d);
  auto* vd = static_cast<uint8_t*>(v_d);
  const auto* kh = static_cast<const uint8_t*>(k_h);
  const auto* vh = static_cast<const uint8_t*>(v_h);
  // q rows of the chunk at processing position idx (chunk 0 of block lo carries the anchor)
  auto chunk_rows = [&](int idx, size_t* r0, size_t* r1) {
    const int which = idx / nc, c = chunk_of(cp, which, idx % nc);
    const size_t base = static_cast<size_t>(p.l_a) + static_cast<size_t>(which) * p.l_b;
    *r0 = (which == 0 && c == 0) ? 0 : base + cp.cb[c];
    *r1 = base + cp.cb[c + 1];
  };
  auto put_q = [&](int idx) -> int {
    size_t r0, r1;
    chunk_rows(idx, &r0, &r1);
    if (r1 > r0)
      CU_TRY(cudaMemcpyAsync(qd + r0 * rq, qh + r0 * rq, (r1 - r0) * rq, cudaMemcpyHostToDevice, hs));
    CU_TRY(cudaEventRecord(H->ev_qc[idx], hs));
    TL.mark("h2d q" + std::to_string(idx), hs);
    return SPAVA_OK;
  };
  TL.mark("fork", st);
  CU_TRY(cudaEventRecord(H->ev_fork, st));
  CU_TRY(cudaStreamWaitEvent(hs, H->ev_fork, 0));
  CU_TRY(cudaMemcpyAsync(kd, kh, lo_rows * rk, cudaMemcpyHostToDevice, hs));
  CU_TRY(cudaMemcpyAsync(vd, vh, lo_rows * rk, cudaMemcpyHostToDevice, hs));
  CU_TRY(cudaMemcpyAsync(qd + qrow * rq, qh + qrow * rq, static_cast<size_t>(p.n_t) * rq, cudaMemcpyHostToDevice, hs));
  ST_TRY(put_q(0));
  CU_TRY(cudaMemcpyAsync(kd + lo_rows * rk, kh + lo_rows * rk, rest * rk, cudaMemcpyHostToDevice, hs));
  CU_TRY(cudaEventRecord(H->ev_kvq, hs));
  TL.mark("h2d k all", hs);
  for (int idx = 1; idx < nc; ++idx) ST_TRY(put_q(idx));
  CU_TRY(cudaMemcpyAsync(vd + lo_rows * rk, vh + lo_rows * rk, rest * rk, cudaMemcpyHostToDevice, hs));
  CU_TRY(cudaEventRecord(H->ev_vhi, hs));
  TL.mark("h2d v hi", hs);
  for (int idx = nc; idx < 2 * nc; ++idx) ST_TRY(put_q(idx));
  HostBufs b{static_cast<const uint8_t*>(q_d), static_cast<const uint8_t*>(k_d),
             static_cast<const uint8_t*>(v_d), od, sel_d};
  ST_TRY(layer_impl(H, b, st, cp));
  TL.mark("compute end", st);
  // outputs as soon as each row chunk is final
  for (int idx = 0; idx < 2 * nc; ++idx) {
    size_t r0, r1;
    chunk_rows(idx, &r0, &r1);
    CU_TRY(cudaStreamWaitEvent(ds, H->ev_oc[idx], 0));
    TL.mark("out ready " + std::to_string(idx), ds);
    if (r1 > r0)
      CU_TRY(cudaMemcpyAsync(oh + r0 * rq, od + r0 * rq, (r1 - r0) * rq, cudaMemcpyDeviceToHost, ds));
    TL.mark("d2h done " + std::to_string(idx), ds);
  }
  CU_TRY(cudaStreamWaitEvent(ds, H->ev_oc[2 * nc], 0));
  CU_TRY(cudaMemcpyAsync(oh + qrow * rq, od + qrow * rq, static_cast<size_t>(p.n_t) * rq,
                         cudaMemcpyDeviceToHost, ds));
  if (sel_h && sel_d && p.l_p > 0)
    CU_TRY(cudaMemcpyAsync(sel_h, sel_d, 2ull * p.l_p * sizeof(int32_t), cudaMemcpyDeviceToHost, ds));
  CU_TRY(cudaEventRecord(H->ev_d2h, ds));
  CU_TRY(cudaStreamWaitEvent(st, H->ev_d2h, 0));  // the caller's stream covers the copies
  TL.mark("end", st);
  TL.dump();
  return SPAVA_OK;
}

int spava_sim_layer(spava_fabric* F, spava_host* const* hosts, const void* const* q,
                    const void* const* k, const void* const* v, void* const* out,
                    int32_t* const* sel, void* stream) {
  if (!F || F->nccl || F->peer) return fail(SPAVA_EINVAL, "sim_layer: needs a local fabric");
  CU_TRY(cudaSetDevice(F->device));
  cudaStream_t st = as_stream(stream);
  const int H = F->plan.hosts;
  std::vector<HostBufs> b(H);
  for (int h = 0; h < H; ++h) {
    if (!hosts[h] || hosts[h]->fab != F || hosts[h]->h != h)
      return fail(SPAVA_EINVAL, "sim_layer: hosts[h] must be host h of this fabric");
    b[h] = HostBufs{static_cast<const uint8_t*>(q[h]), static_cast<const uint8_t*>(k[h]),
                    static_cast<const uint8_t*>(v[h]), static_cast<uint8_t*>(out[h]),
                    sel ? sel[h] : nullptr};
  }
  // phase 1 on every host fills the shared exchange (the GatherFabric rounds); trace
  // records keep each host's run_host program order (simhost.cpp:343-426)
  for (int h = 0; h < H; ++h) {
    spava_host* X = hosts[h];
    const bool fs = fused_score(X, false);  // N1: the query launch also scores
    if (fs) {
      trace_ev(X, st, kComputeBegin, "query_attn", false);
      ST_TRY(phase_query(X, b[h], st, false, true));
      trace_ev(X, st, kComputeEnd, "query_attn", false);
    }
    ST_TRY(phase_select(X, b[h], st, false, nullptr, fs ? 1 : 0));
    trace_ev(X, st, kCommIssued, "pass1", true);
    trace_ev(X, st, kCommIssued, "pass2", true);
    if (!fs) {
      trace_ev(X, st, kComputeBegin, "query_attn", false);
      ST_TRY(phase_query(X, b[h], st, false));
      trace_ev(X, st, kComputeEnd, "query_attn", false);
    }
    trace_ev(X, st, kCommIssued, "qpartial", true);
  }
  for (int h = 0; h < H; ++h) {
    spava_host* X = hosts[h];
    trace_ev(X, st, kCommWaitStart, "pass1", true);
    trace_ev(X, st, kCommCompleted, "pass1", true);
    if (!F->plan.zigzag) {
      trace_ev(X, st, kCommWaitStart, "pass2", true);
      trace_ev(X, st, kCommCompleted, "pass2", true);
    }
    if (merged_stages()) {
      if (F->plan.zigzag) {
        trace_ev(X, st, kCommWaitStart, "pass2", true);
        trace_ev(X, st, kCommCompleted, "pass2", true);
      }
      trace_ev(X, st, kComputeBegin, "stage1", false);
      trace_ev(X, st, kComputeBegin, "stage2", false);
      ST_TRY(phase_stage12(X, b[h], st));
      trace_ev(X, st, kComputeEnd, "stage1", false);
      trace_ev(X, st, kComputeEnd, "stage2", false);
    } else {
      trace_ev(X, st, kComputeBegin, "stage1", false);
      ST_TRY(phase_stage1(X, b[h], st));
      trace_ev(X, st, kComputeEnd, "stage1", false);
      if (F->plan.zigzag) {
        trace_ev(X, st, kCommWaitStart, "pass2", true);
        trace_ev(X, st, kCommCompleted, "pass2", true);
      }
      trace_ev(X, st, kComputeBegin, "stage2", false);
      ST_TRY(phase_stage2(X, b[h], st));
      trace_ev(X, st, kComputeEnd, "stage2", false);
    }
    trace_ev(X, st, kCommWaitStart, "qpartial", true);
    trace_ev(X, st, kCommCompleted, "qpartial", true);
    trace_ev(X, st, kComputeBegin, "merge", false);
    ST_TRY(phase_merge(X, b[h], st));
    trace_ev(X, st, kComputeEnd, "merge", false);
    if (X->trace) ++X->trace_layer;
  }
  return SPAVA_OK;
}

int spava_sim_layer_timed(spava_fabric* F, spava_host* const* hosts, const void* const* q,
                          const void* const* k, const void* const* v, void* const* out,
                          int32_t* const* sel, void* stream, float* ms_per_host) {
  if (!F || F->nccl) return fail(SPAVA_EINVAL, "sim_layer_timed: needs a local fabric");
  if (!ms_per_host) return fail(SPAVA_EINVAL, "sim_layer_timed: null ms_per_host");
  CU_TRY(cudaSetDevice(F->device));
  cudaStream_t st = as_stream(stream);
  const int H = F->plan.hosts;
  std::vector<HostBufs> b(H);
  std::vector<char> seen(H, 0);
  for (int h = 0; h < H; ++h) {
    if (!hosts[h] || hosts[h]->fab != F || hosts[h]->h < 0 || hosts[h]->h >= H || seen[hosts[h]->h]++)
      return fail(SPAVA_EINVAL, "sim_layer_timed: hosts must be the fabric's H hosts, each once");
    b[h] = HostBufs{static_cast<const uint8_t*>(q[h]), static_cast<const uint8_t*>(k[h]),
                    static_cast<const uint8_t*>(v[h]), static_cast<uint8_t*>(out[h]),
                    sel ? sel[h] : nullptr};
  }
  // events bracket each host's phase-1 and phase-2 work (run alone on the GPU, in order)
  std::vector<cudaEvent_t> ev(4 * H);
  for (auto& e : ev) CU_TRY(cudaEventCreate(&e));
  int rc = SPAVA_OK;
  for (int h = 0; h < H && rc == SPAVA_OK; ++h) {
    cudaEventRecord(ev[4 * h], st);
    const bool fs = fused_score(hosts[h], false);
    if (fs) rc = phase_query(hosts[h], b[h], st, false, true);
    if (rc == SPAVA_OK) rc = phase_select(hosts[h], b[h], st, false, nullptr, fs ? 1 : 0);
    if (rc == SPAVA_OK && !fs) rc = phase_query(hosts[h], b[h], st, false);
    cudaEventRecord(ev[4 * h + 1], st);
  }
  for (int h = 0; h < H && rc == SPAVA_OK; ++h) {
    cudaEventRecord(ev[4 * h + 2], st);
    if (merged_stages()) {
      rc = phase_stage12(hosts[h], b[h], st);
    } else {
      rc = phase_stage1(hosts[h], b[h], st);
      if (rc == SPAVA_OK) rc = phase_stage2(hosts[h], b[h], st);
    }
    if (rc == SPAVA_OK) rc = phase_merge(hosts[h], b[h], st);
    cudaEventRecord(ev[4 * h + 3], st);
  }
  if (rc == SPAVA_OK && cudaStreamSynchronize(st) != cudaSuccess) rc = fail(SPAVA_ECUDA, "sim_layer_timed: sync");
  for (int h = 0; h < H && rc == SPAVA_OK; ++h) {
    float a = 0.f, c = 0.f;
    cudaEventElapsedTime(&a, ev[4 * h], ev[4 * h + 1]);
    cudaEventElapsedTime(&c, ev[4 * h + 2], ev[4 * h + 3]);
    ms_per_host[h] = a + c;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return rc;
}

int spava_host_set_delay(spava_host* H, int which, uint64_t ns) {
  if (!H) return fail(SPAVA_EINVAL, "set_delay: null host");
  if (which < 0 || which > 3) return fail(SPAVA_ERANGE, "set_delay: which is 0..3");
  H->delay_ns[which] = ns;
  return SPAVA_OK;
}

int spava_host_set_trace(spava_host* H, int enable) {
  if (!H) return fail(SPAVA_EINVAL, "set_trace: null host");
  CU_TRY(cudaSetDevice(H->fab->device));
  H->trace = enable != 0;
  H->trace_layer = 0;
  H->trace_recs.clear();
  if (enable && !H->fab->trace_base) {
    CU_TRY(cudaEventCreate(&H->fab->trace_base));
    CU_TRY(cudaEventRecord(H->fab->trace_base, 0));
  }
  return SPAVA_OK;
}

int spava_host_trace_read(spava_host* H, spava_trace_event* out, int cap, int* n) {
  if (!H || !n) return fail(SPAVA_EINVAL, "trace_read: null argument");
  CU_TRY(cudaSetDevice(H->fab->device));
  *n = static_cast<int>(H->trace_recs.size());
  if (!out) return SPAVA_OK;
  if (cap < *n) return fail(SPAVA_EINVAL, "trace_read: capacity too small");
  for (int i = 0; i < *n; ++i) {
    const auto& r = H->trace_recs[i];
    CU_TRY(cudaEventSynchronize(r.ev));
    float ms = 0.f;
    CU_TRY(cudaEventElapsedTime(&ms, H->fab->trace_base, r.ev));
    out[i].kind = r.kind;
    out[i].layer = r.layer;
    std::memcpy(out[i].label, r.label, sizeof(out[i].label));
    std::memcpy(out[i].tag, r.tag, sizeof(out[i].tag));
    out[i].t_us = 1e3 * static_cast<double>(ms);
  }
  return SPAVA_OK;
}

int spava_host_set_timing(spava_host* H, int enable) {
  H->timing = enable != 0;
  H->serial = enable == 2;
  H->ev_used = 0;
  for (auto& s : H->spans) s.clear();
  H->attn_flops = 0.0;
  H->attn_launches = 0;
  return SPAVA_OK;
}

int spava_host_timing(spava_host* H, double* ms_by_class, double* attn_flops,
                      uint64_t* attn_launches) {
  for (int c = 0; c < 4; ++c) {
    double ms = 0.0;
    for (auto& pr : H->spans[c]) {
      CU_TRY(cudaEventSynchronize(H->ev_pool[pr.second]));
      float t = 0.f;
      CU_TRY(cudaEventElapsedTime(&t, H->ev_pool[pr.first], H->ev_pool[pr.second]));
      ms += t;
    }
    if (ms_by_class) ms_by_class[c] = ms;
  }
  if (attn_flops) *attn_flops = H->attn_flops;
  if (attn_launches) *attn_launches = H->attn_launches;
  return SPAVA_OK;
}

namespace {
struct DecoderWs {
  size_t xn, q, k, v, a, h, total;
};
DecoderWs decoder_ws(const spava_host* H, const spava_decoder_weights* w) {
  const spava_layer_cfg& c = H->fab->cfg;
  const spava_plan& p = H->fab->plan;
  const size_t rows = static_cast<size_t>(p.l_a) + 2ull * p.l_b + p.n_t;
  auto al = [](size_t x) { return (x + 255) / 256 * 256; };
  DecoderWs d{};
  size_t o = 0;
  d.xn = o; o += al(rows * w->d_model * 2);
  d.q = o; o += al(rows * c.hq * c.dh * 2);
  d.k = o; o += al(rows * c.hkv * c.dh * 2);
  d.v = o; o += al(rows * c.hkv * c.dh * 2);
  d.a = o; o += al(rows * c.hq * c.dh * 2);
  d.h = o; o += al(rows * static_cast<size_t>(w->ffn) * 2);
  d.total = o;
  return d;
}
}  // namespace

int spava_gemm(int M, int N, int K, const void* A, int64_t lda, const void* B, int64_t ldb, void* C,
               int64_t ldc, float beta, int relu, void* stream) {
  if (!A || !B || !C) return fail(SPAVA_EINVAL, "gemm: null argument");
  ST_TRY(require_device());
  std::string err;
  const int col0 = 0;
  const long long ldo = ldc;
  const cudaError_t e = launch_gemm_bf16(M, N, K, A, lda, B, ldb, 1, &col0, &C, &ldo, beta, relu != 0,
                                         as_stream(stream), &err);
  if (e != cudaSuccess)
    return fail(e == cudaErrorInvalidValue ? SPAVA_EINVAL : SPAVA_ECUDA,
                "gemm: " + (err.empty() ? std::string(cudaGetErrorString(e)) : err));
  ++g_launches;
  return SPAVA_OK;
}

size_t spava_decoder_workspace(const spava_host* H, const spava_decoder_weights* w) {
  return (H && w) ? decoder_ws(H, w).total : 0;
}

int spava_host_decoder_layer(spava_host* H, const spava_decoder_weights* w, void* x, int64_t ldx,
                             void* ws, size_t ws_bytes, void* stream) {
  if (!H || !w || !x || !ws) return fail(SPAVA_EINVAL, "decoder_layer: null argument");
  spava_fabric* F = H->fab;
  if (!F->nccl && F->plan.hosts != 1)
    return fail(SPAVA_EINVAL, "decoder_layer: local fabric with H > 1 must be driven by the simulator");
  if (!w->w_qkv || !w->w_o || !w->w_1 || !w->w_2 || w->d_model <= 0 || w->d_model % 8 || w->ffn <= 0 ||
      w->ffn % 8 || ldx < w->d_model || ldx % 8)
    return fail(SPAVA_EINVAL, "decoder_layer: weights / d_model / ffn / ldx");
  if (w->norm && (!w->g_1 || !w->g_2)) return fail(SPAVA_EINVAL, "decoder_layer: norm needs g_1, g_2");
  const DecoderWs d = decoder_ws(H, w);
  if (ws_bytes < d.total) return fail(SPAVA_EINVAL, "decoder_layer: workspace too small");
  CU_TRY(cudaSetDevice(F->device));
  const spava_layer_cfg& c = F->cfg;
  const spava_plan& p = F->plan;
  const int rows = p.l_a + 2 * p.l_b + p.n_t;
  const int D = w->d_model, dq = c.hq * c.dh, dk = c.hkv * c.dh, wqkv = dq + 2 * dk;
  cudaStream_t st = as_stream(stream);
  uint8_t* base = static_cast<uint8_t*>(ws);
  void* xn = base + d.xn;
  void* q = base + d.q;
  void* k = base + d.k;
  void* v = base + d.v;
  void* a = base + d.a;
  void* hbuf = base + d.h;
  std::string err;
  auto G3 = [&](int M, int N, int K, const void* A, long long lda, const void* B, long long ldb, int nout,
                const int* col0, void* const* outs, const long long* ldo, float beta, bool relu) -> int {
    const cudaError_t e = launch_gemm_bf16(M, N, K, A, lda, B, ldb, nout, col0, outs, ldo, beta, relu, st, &err);
    if (e != cudaSuccess)
      return fail(e == cudaErrorInvalidValue ? SPAVA_EINVAL : SPAVA_ECUDA,
                  "decoder_layer: " + (err.empty() ? std::string(cudaGetErrorString(e)) : err));
    ++g_launches;
    return SPAVA_OK;
  };
  auto G = [&](int M, int N, int K, const void* A, long long lda, const void* B, long long ldb, void* Cm,
               long long ldc, float beta, bool relu) -> int {
    const int col0 = 0;
    const long long ldo = ldc;
    return G3(M, N, K, A, lda, B, ldb, 1, &col0, &Cm, &ldo, beta, relu);
  };
  const uint8_t* wq = static_cast<const uint8_t*>(w->w_qkv);
  // project (simhost.cpp:196-199): xn = layer_norm(x, g1); q, k, v = xn [Wq | Wk | Wv]
  const void* xin = x;
  long long ldin = ldx;
  if (w->norm) {
    CU_TRY(launch_layer_norm(x, ldx, w->g_1, D, xn, D, rows, st));
    xin = xn;
    ldin = D;
  }
  {  // one GEMM against [Wq | Wk | Wv], its epilogue routes the column ranges to q, k, v
    const int col0[3] = {0, dq, dq + dk};
    void* outs[3] = {q, k, v};
    const long long ldo[3] = {dq, dk, dk};
    ST_TRY(G3(rows, wqkv, D, xin, ldin, wq, wqkv, 3, col0, outs, ldo, 0.f, false));
  }
  // Spava attention (the hot path)
  HostBufs b{static_cast<const uint8_t*>(q), static_cast<const uint8_t*>(k), static_cast<const uint8_t*>(v),
             static_cast<uint8_t*>(a), nullptr};
  ST_TRY(layer_impl(H, b, st, CopyEdges{}));
  // finish_group (simhost.cpp:202-207): x += a Wo; f = layer_norm(x, g2); x += relu(f W1) W2
  ST_TRY(G(rows, D, dq, a, dq, w->w_o, D, x, ldx, 1.f, false));
  const void* fin = x;
  long long ldf = ldx;
  if (w->norm) {
    CU_TRY(launch_layer_norm(x, ldx, w->g_2, D, xn, D, rows, st));
    fin = xn;
    ldf = D;
  }
  ST_TRY(G(rows, w->ffn, D, fin, ldf, w->w_1, w->ffn, hbuf, w->ffn, 0.f, true));
  ST_TRY(G(rows, D, w->ffn, hbuf, w->ffn, w->w_2, D, x, ldx, 1.f, false));
  g_launches += w->norm ? 2 : 0;
  return SPAVA_OK;
}

int spava_host_capture_layer(spava_host* H, const void* q, const void* k, const void* v, void* out,
                             int32_t* sel, void* stream) {
  spava_fabric* F = H->fab;
  if (!F->nccl && F->plan.hosts != 1)
    return fail(SPAVA_EINVAL, "capture_layer: local fabric with H > 1 must be driven by spava_sim_layer");
  if (F->peer) return fail(SPAVA_EINVAL, "capture_layer: the peer fabric's epoch flags change every layer");
  if (H->timing || H->trace) return fail(SPAVA_EINVAL, "capture_layer: disable timing and trace first");
  if (!stream) return fail(SPAVA_EINVAL, "capture_layer: needs a non-default stream");
  CU_TRY(cudaSetDevice(F->device));
  cudaStream_t st = as_stream(stream);
  if (H->graph_exec) cudaGraphExecDestroy(H->graph_exec);
  if (H->graph) cudaGraphDestroy(H->graph);
  H->graph_exec = nullptr;
  H->graph = nullptr;
  HostBufs b{static_cast<const uint8_t*>(q), static_cast<const uint8_t*>(k),
             static_cast<const uint8_t*>(v), static_cast<uint8_t*>(out), sel};
  const uint64_t k0 = g_launches.load();
  CU_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  const int rc = layer_impl(H, b, st, CopyEdges{});
  cudaGraph_t g = nullptr;
  const cudaError_t e = cudaStreamEndCapture(st, &g);
  if (rc != SPAVA_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  CU_TRY(e);
  H->graph = g;
  CU_TRY(cudaGraphInstantiate(&H->graph_exec, g, 0));
  H->graph_kernels = g_launches.load() - k0;
  g_launches -= H->graph_kernels;  // captured, not launched
  return SPAVA_OK;
}

int spava_host_replay_layer(spava_host* H, void* stream) {
  if (!H || !H->graph_exec) return fail(SPAVA_EINVAL, "replay_layer: nothing captured");
  CU_TRY(cudaSetDevice(H->fab->device));
  CU_TRY(cudaGraphLaunch(H->graph_exec, as_stream(stream)));
  g_launches += H->graph_kernels;
  return SPAVA_OK;
}

int spava_host_status(spava_host* H, void* stream, int32_t* status_out) {
  CU_TRY(cudaMemcpyAsync(status_out, H->status, sizeof(int32_t), cudaMemcpyDeviceToHost,
                         as_stream(stream)));
  CU_TRY(cudaStreamSynchronize(as_stream(stream)));
  return SPAVA_OK;
}

}  // extern "C"
