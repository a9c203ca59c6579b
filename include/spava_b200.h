/* spava_b200.h -- C ABI of the B200-native Spava sequence-parallel prefill path.
 *
 * Drop-in boundary for the reference's C++ operator API (namespace seqpar,
 * /root/reference/proj/core/include/seqpar/{partition,approx,attention}.hpp).
 * Every entry point below names the reference interface it replaces.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Tensors are token-major row-major
 *    [rows x heads*dh]; "ld" arguments are row strides in ELEMENTS.
 *    Q/K/V/passing blocks are bf16 in device memory (dh = 128); scores are f32.
 *  - Heads: q-head h reads kv-head h / (hq/hkv) (GQA).  The reference has no
 *    GQA; hq == hkv reproduces it exactly.
 *  - Every function returns a spava_status; on failure spava_last_error()
 *    (thread-local) describes it.  No C++ exception crosses this ABI.  The
 *    reference's std::invalid_argument maps to SPAVA_EINVAL, std::out_of_range
 *    to SPAVA_ERANGE, std::runtime_error to SPAVA_ERUNTIME.
 *  - Device work is asynchronous on the caller's stream (cudaStream_t passed as
 *    void*; NULL = legacy default stream).  Caller owns all buffers.
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point fails with SPAVA_ECUDA.
 */
#ifndef SPAVA_B200_H
#define SPAVA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SPAVA_OK = 0,
  SPAVA_EINVAL = 1,   /* std::invalid_argument in the reference */
  SPAVA_ERANGE = 2,   /* std::out_of_range                       */
  SPAVA_ERUNTIME = 3, /* std::runtime_error                      */
  SPAVA_ECUDA = 4,    /* CUDA failure / no sm_100 device          */
  SPAVA_ENCCL = 5     /* NCCL failure                             */
} spava_status;

const char* spava_last_error(void);
const char* spava_version(void);
/* 1 if a CUDA device of compute capability 10.x is visible. */
int spava_device_ok(void);

/* ------------------------------------------------------------------ plan
 * BlockPlan / HostTopology (partition.hpp:13-45).                          */
typedef struct {
  int n_v;           /* video context length                      */
  int n_t;           /* query length                              */
  int hosts;         /* physical hosts H                          */
  int l_a;           /* anchor length                             */
  int l_b;           /* per-virtual-block length incl. pad        */
  int l_p;           /* essential KVs passed per block            */
  int pad;           /* zero rows appended to the context         */
  int virtual_hosts; /* 2H                                        */
  int zigzag;        /* 1: pairs (h, 2H-1-h); 0: naive (2h, 2h+1) */
} spava_plan;

/* split_context geometry (partition.cpp:40-85); zigzag_map/naive_map (:21-29). */
int spava_make_plan(int n_v, int n_t, int hosts, int l_a, int l_p, int zigzag, spava_plan* out);
/* default_plan (partition.cpp:96-113): l_a = n/64, l_p = min(n/128, l_b). */
int spava_default_plan(int n, int hosts, spava_plan* out);
/* HostTopology::virtual_pair (partition.cpp:9-13) */
int spava_virtual_pair(const spava_plan* plan, int h, int* lo, int* hi);
/* HostTopology::physical_of (partition.cpp:15-19) */
int spava_physical_of(const spava_plan* plan, int v, int* h);
/* slice_anchor (partition.cpp:87-94) */
int spava_slice_anchor(int l_a, int hosts, int h, int* begin, int* end);
/* BlockPlan::block_offset / query_offset (partition.hpp:35-36) */
int spava_block_offset(const spava_plan* plan, int v);
int spava_query_offset(const spava_plan* plan);
/* ContextSplit::pad_mask[v] (partition.cpp:71-79) -> l_b bytes, 1 = pad row */
int spava_pad_mask(const spava_plan* plan, int v, uint8_t* mask_out);
/* number of non-pad rows of virtual block v */
int spava_block_valid_rows(const spava_plan* plan, int v);
/* assemble_passing (approx.cpp:104-132) in exchange-slot terms: the sources < v
 * arrive in round 0 (lo blocks, pass1) slots [r0_begin, r0_end) and round 1
 * (hi blocks, pass2) slots [r1_begin, r1_end) of the host-ordered allgather.   */
int spava_passing_ranges(const spava_plan* plan, int v, int* r0_begin, int* r0_end,
                         int* r1_begin, int* r1_end);

/* split_context on the device (partition.cpp:40-85): gather host h's local rows
 * [anchor | block lo | block hi | query] from the global sequence [E_v (n_v) | E_Q (n_t)]
 * (src, row stride ld_src_bytes), pad rows zero-filled.  Any row width (row_bytes, a
 * multiple of 16), so one call per Q / K / V tensor.  Rows: l_a + 2*l_b + n_t.          */
int spava_split_rows(const spava_plan* plan, int h, const void* src, int64_t ld_src_bytes,
                     void* dst, int64_t ld_dst_bytes, int row_bytes, void* stream);
/* Inverse of spava_split_rows for outputs: host h's block rows (non-pad) to their global
 * positions; with write_shared also the anchor and query rows (identical on every host:
 * anchor_attention is replicated and the merged query is the same after mha_merge).    */
int spava_merge_rows(const spava_plan* plan, int h, const void* src, int64_t ld_src_bytes,
                     void* dst, int64_t ld_dst_bytes, int row_bytes, int write_shared, void* stream);

/* --------------------------------------------------------------- scoring
 * score_block (simhost.cpp:209-224) -> score_context (approx.cpp:15-69),
 * softmax or raw-logit aggregation, "exact" arithmetic.
 * q: [n_t x ldq] bf16, k: [l_b x ldk] bf16, pad: device u8[l_b] or NULL,
 * keys j >= n_valid are pads too.  scores: device f32[l_b] (pads -> -inf).  */
size_t spava_score_workspace(int n_t, int l_b, int hq);
int spava_score_block(const void* q, int64_t ldq, int n_t, const void* k, int64_t ldk, int l_b,
                      const uint8_t* pad, int n_valid, int hq, int hkv, int dh, int softmax,
                      float* scores, void* workspace, size_t workspace_bytes, void* stream);
/* score_context (approx.cpp:15-69, approx.hpp:38-41) with the caller's logit scale
 * (scale == 0: 1/sqrtf(dh)).  Heads narrower than 128 are passed zero-padded to dh = 128
 * columns (the padding adds exact zeros to the c-ascending fp32 dot products, so the
 * scores are those of the narrow heads).                                               */
int spava_score_block_ex(const void* q, int64_t ldq, int n_t, const void* k, int64_t ldk, int l_b,
                         const uint8_t* pad, int n_valid, int hq, int hkv, int dh, int softmax,
                         float* scores, void* workspace, size_t workspace_bytes, void* stream,
                         float scale);
/* Fast score_block on the tensor cores (score_fast.cu): same definition, logits from bf16
 * tcgen05 MMAs with fp32 accumulation, softmax via exp2 -- NOT bit-faithful (the exact
 * entry point above is); passing indices agree except where two scores tie within that
 * error.  Softmax aggregation only; n_t <= 128, hkv <= 4, dh = 128.
 * ws_bytes >= spava_score_fast_workspace(n_t, l_b, hq). */
size_t spava_score_fast_workspace(int n_t, int l_b, int hq);
int spava_score_block_fast(const void* q, int64_t ldq, int n_t, const void* k, int64_t ldk, int l_b,
                           const uint8_t* pad, int n_valid, int hq, int hkv, int dh,
                           float* scores, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------- select + pack
 * select_essential (approx.cpp:71-102): top-l_p by score, ties -> lower index,
 * non-finite never selected, indices ascending (+global_offset) in idx_out;
 * K/V rows gathered into k_out/v_out (ld_out; rows >= count zero-filled,
 * idx_out entries >= count set to -1).
 * count_out, status_out: device int32 (status |= 1: NaN score rejected).     */
int spava_select_pack(const float* scores, int l_b, int l_p, int global_offset, const void* k,
                      const void* v, int64_t ld, int width, int32_t* idx_out, void* k_out,
                      void* v_out, int64_t ld_out, int32_t* count_out, int32_t* status_out,
                      void* stream);

/* ----------------------------------------------------------- attention
 * attention_lse / mha_lse (attention.cpp:18-86, 158-178) over a segment table
 * (KeySegment, attention.hpp:16-23).  Key j of a segment is visible to query
 * row i iff j < rows and (!causal || j <= i) -- pads are a shorter `rows`.
 * Used for anchor_attention (approx.cpp:134-138), block_attention (:140-154)
 * and query_attention (:156-188).  out: [nq x ldo] bf16 (out_f32=0) or f32;
 * lse (nullable): [nq x hq] f32, natural log, -inf for rows with no key.
 * splits > 1 computes split-KV partials internally and merges them (needs
 * workspace of spava_attention_workspace bytes).                            */
typedef struct {
  const void* k; /* bf16 [rows x ld], kv head h at columns [h*dh, (h+1)*dh) */
  const void* v;
  int64_t ld;
  int rows;
  int causal; /* MaskKind::CausalWithin (requires rows <= nq) */
} spava_segment;

size_t spava_attention_workspace(int nq, int hq, int dh, int splits);
int spava_attention(const void* q, int64_t ldq, int nq, const spava_segment* segs, int nseg,
                    int hq, int hkv, int dh, void* out, int64_t ldo, int out_f32, float* lse,
                    int splits, void* workspace, size_t workspace_bytes, void* stream);
/* attention_lse's explicit logit scale (attention.hpp:40-41; scale == 0: 1/sqrtf(dh)).
 * Narrower heads go zero-padded to dh = 128 columns (q, k and v); the padded output
 * columns come out zero.                                                                */
int spava_attention_ex(const void* q, int64_t ldq, int nq, const spava_segment* segs, int nseg,
                       int hq, int hkv, int dh, void* out, int64_t ldo, int out_f32, float* lse,
                       int splits, void* workspace, size_t workspace_bytes, void* stream, float scale);

/* --------------------------------------------------------------- merge
 * mha_merge (attention.cpp:180-197) over nparts partials in host order.
 * outs[p]: device f32 [rows x ld_part], lses[p]: device f32 [rows x hq]
 * (host arrays of device pointers).  dst: bf16 or f32 [rows x ld_dst];
 * dst_lse (nullable) receives the merged lse.  status: device int32, |= 4
 * if a row is invalid in every part (the reference throws).                  */
int spava_mha_merge(int nparts, const float* const* outs, const float* const* lses, int rows,
                    int64_t ld_part, int hq, int dh, void* dst, int64_t ld_dst, int dst_f32,
                    float* dst_lse, int32_t* status, void* stream);

/* ---------------------------------------------------------- the layer
 * One Spava attention layer of physical host h: the body of run_host's
 * per-layer loop (simhost.cpp:321-426) minus projections/FFN.
 *
 * Host-local device buffers, token-major rows
 *   [ anchor (l_a) | block lo (l_b) | block hi (l_b) | query (n_t) ]
 * q: hq*dh columns, k/v: hkv*dh columns (bf16).  out: same rows, hq*dh bf16
 * (anchor_attention, block_attention lo/hi, merged query attention).
 * sel: int32 [2 x l_p] global indices of the lo/hi passing blocks (may be NULL).
 *
 * The exchange (GatherFabric, simhost.cpp:61-166) is a spava_fabric:
 *  - local: H simulated hosts on ONE device, exchange buffers shared in place
 *    (the reference's in-process mailbox); drive with spava_sim_layer.
 *  - nccl: one process per GPU; pass1/pass2/qpartial are in-place
 *    ncclAllGather on a dedicated comm stream, overlapped per Algorithm 1.
 *  - peer: one process per GPU (<= 8, one node); no collective library -- the
 *    select gather and the query split-merge kernels store their slot straight
 *    into every peer GPU's exchange buffer over NVLink (IPC-mapped), and 32-bit
 *    epoch flags written / waited by stream memory operations order the rounds. */
typedef struct {
  int n_v, n_t, hosts, l_a, l_p;
  int zigzag;         /* HostTopology pairing                                 */
  int designated;     /* host carrying query self keys; -1 = last (simhost.cpp:276) */
  int query_self_all; /* SimOptions::query_self_all_hosts                     */
  int softmax_scores; /* SimOptions::softmax_scores                           */
  int hq, hkv, dh;
  int query_splits;   /* split-KV factor of query attention; 0 = auto         */
  int score_mode;     /* 0 = exact (bit-faithful to score_block), 1 = fast:
                         tcgen05 logits + exp2 (needs softmax_scores, n_t <= 128,
                         hkv <= 4); indices agree except near-ties              */
} spava_layer_cfg;

typedef struct spava_fabric spava_fabric;
typedef struct spava_host spava_host;

int spava_fabric_create_local(const spava_layer_cfg* cfg, int device, spava_fabric** out);
/* unique_id: 128-byte ncclUniqueId from spava_nccl_unique_id on rank 0. */
int spava_nccl_unique_id(void* unique_id_128);
int spava_fabric_create_nccl(const spava_layer_cfg* cfg, int device, const void* unique_id_128,
                             int world, int rank, spava_fabric** out);
/* Peer fabric (replaces GatherFabric::issue/wait, simhost.cpp:73-124).  Setup:
 * create on every rank, exchange the 64-byte handles (any host channel, e.g.
 * torch.distributed all_gather_object), then spava_fabric_peer_open with the
 * world x 64-byte array in rank order.  All ranks must run the same number of
 * layers.  Destroy only after every rank has synchronised its last layer (a
 * barrier), since peers store into this rank's buffer.                        */
#define SPAVA_PEER_HANDLE_BYTES 64
int spava_fabric_create_peer(const spava_layer_cfg* cfg, int device, int world, int rank,
                             int64_t encode_bytes, spava_fabric** out);
int spava_fabric_peer_handle(spava_fabric* fab, void* handle_64);
int spava_fabric_peer_open(spava_fabric* fab, const void* handles_world_x_64);
/* In-process variant (tests, one device): fabrics[r] = the peer fabric of rank r;
 * each rank's layer must then run on its own stream (the flag waits are in-stream). */
int spava_fabric_peer_attach(spava_fabric* const* fabrics, int world);
int spava_fabric_destroy(spava_fabric* fab);

/* ---------------------------------------------- frame-parallel encode gather
 * frame_partition (partition.cpp:30-37): counts[h] = frames/hosts + (h < frames%hosts).
 * Host h encodes frames [sum counts[<h], +counts[h]) (simhost.cpp:285-291), i.e. global
 * E_v rows [off_h, off_h + part_rows[h]).                                      */
int spava_frame_partition(int frames, int hosts, int* counts);
/* The encode AllGather + concat_rows + split_context of run_host (simhost.cpp:293-302)
 * fused into one row gather: host h's [anchor | lo | hi | query] rows are read straight
 * from the owning host's part (parts[q], rows part_rows[q], stride ld_part_bytes; the
 * query rows from e_q) -- only l_a + 2*l_b + n_t rows move, E_v is never assembled.
 * part_rows must sum to n_v.  parts may be IPC-mapped peer pointers.            */
int spava_gather_split_rows(const spava_plan* plan, int h, const void* const* parts,
                            const int64_t* part_rows, int64_t ld_part_bytes, const void* e_q,
                            int64_t ld_q_bytes, void* dst, int64_t ld_dst_bytes, int row_bytes,
                            void* stream);
/* Peer fabric (created with encode_bytes > 0): each rank's encoder writes its E_v rows
 * into its encode region; spava_host_gather_context then announces them (epoch flag),
 * waits for every peer's, and gathers this host's rows over NVLink.  Before writing
 * the region again, enqueue spava_fabric_encode_acquire on the writer's stream (waits
 * until every peer has read the previous round).                               */
int spava_fabric_encode_region(spava_fabric* fab, void** ptr, int64_t* bytes);
int spava_fabric_encode_acquire(spava_fabric* fab, void* stream);
int spava_host_gather_context(spava_host* host, const int64_t* part_rows, int64_t ld_part_bytes,
                              const void* e_q, int64_t ld_q_bytes, void* dst, int64_t ld_dst_bytes,
                              int row_bytes, void* stream);

int spava_host_create(spava_fabric* fab, int h, spava_host** out);
int spava_host_destroy(spava_host* host);
int spava_host_plan(const spava_host* host, spava_plan* out);
/* rows of the host-local buffers: l_a + 2*l_b + n_t */
int spava_host_rows(const spava_host* host);

/* NCCL fabric: the whole layer of this rank, exchange overlapped.            */
int spava_host_layer(spava_host* host, const void* q, const void* k, const void* v, void* out,
                     int32_t* sel, void* stream);
/* Local fabric: every host of the fabric, phase by phase, on one stream.
 * q/k/v/out/sel are arrays of H per-host pointers (host arrays).            */
/* spava_host_layer with HOST buffers (the reference's run_host takes host Matrix inputs,
 * simhost.cpp:317-437): q/k/v host rows are copied to the caller-owned device staging
 * buffers in the order the phases consume them (k, v and query rows; anchor + block-lo rows
 * of q; block-hi rows of q) on an internal copy stream, each phase waits only for its rows,
 * and each output row range (anchor + lo after stage 1, hi after stage 2, query after the
 * merge) is copied back while later phases still run.  Host buffers should be pinned for
 * the copies to overlap.  `stream` waits for the last copy before returning control to the
 * caller's stream order; sel_h/sel_d may be NULL. */
int spava_host_layer_hostbuf(spava_host* host, const void* q_h, const void* k_h, const void* v_h,
                             void* out_h, int32_t* sel_h, void* q_d, void* k_d, void* v_d,
                             void* out_d, int32_t* sel_d, void* stream);
/* One spava_host_layer captured as a CUDA graph (caller, side and comm streams, NCCL
 * rounds included) on `stream` (not the legacy default stream), then replayed with one
 * launch per layer: the buffers are those of the capture (fill them before each replay).
 * Timing and trace must be off while capturing.                                       */
int spava_host_capture_layer(spava_host* host, const void* q, const void* k, const void* v,
                             void* out, int32_t* sel, void* stream);
int spava_host_replay_layer(spava_host* host, void* stream);

/* The decoder layer around the path (simhost.cpp:196-207, 431-436):
 *   xn = norm ? layer_norm(x, g_1) : x;  q, k, v = xn [Wq | Wk | Wv];  a = spava layer;
 *   x += a Wo;  f = norm ? layer_norm(x, g_2) : x;  x += relu(f W1) W2.
 * x: host-local rows [anchor | lo | hi | query] x d_model, bf16, updated in place.  All
 * matrices are row-major bf16 on the device (w_qkv: d_model x (hq+2*hkv)*128, w_o:
 * hq*128 x d_model, w_1: d_model x ffn, w_2: ffn x d_model); gains fp32 [d_model].
 * GEMMs are cuBLASLt bf16 library GEMMs with fp32 accumulation.                       */
typedef struct {
  const void* w_qkv;
  const void* w_o;
  const void* w_1;
  const void* w_2;
  const float* g_1;
  const float* g_2;
  int d_model, ffn, norm;
} spava_decoder_weights;
/* The decoder layer's GEMM (tcgen05, gemm.cu): row-major bf16 C[M x N] = A[M x K] B[K x N]
 * (+ beta * C) (ReLU if relu), fp32 accumulation; strides and N multiples of 8.          */
int spava_gemm(int M, int N, int K, const void* A, int64_t lda, const void* B, int64_t ldb, void* C,
               int64_t ldc, float beta, int relu, void* stream);
size_t spava_decoder_workspace(const spava_host* host, const spava_decoder_weights* w);
int spava_host_decoder_layer(spava_host* host, const spava_decoder_weights* w, void* x, int64_t ldx,
                             void* ws, size_t ws_bytes, void* stream);

int spava_sim_layer(spava_fabric* fab, spava_host* const* hosts, const void* const* q,
                    const void* const* k, const void* const* v, void* const* out,
                    int32_t* const* sel, void* stream);
/* spava_sim_layer with every host's phases bracketed by events and run alone on the GPU:
 * ms_per_host[h] = host h's device time for one layer (excluding any exchange cost).  The
 * max over hosts is the per-GPU layer time an H-GPU run would see before communication --
 * used to measure load balance (zigzag vs naive pairing) on real kernels.  hosts may list
 * the fabric's H hosts in any order (q..sel and ms_per_host follow that order): phase 1 of
 * every host runs first, then phase 2 host by host in the given order -- rotating the order
 * lets each host be timed early in a run, before a sustained-load power cap lowers the
 * clocks.  Synchronises. */
int spava_sim_layer_timed(spava_fabric* fab, spava_host* const* hosts, const void* const* q,
                          const void* const* k, const void* const* v, void* const* out,
                          int32_t* const* sel, void* stream, float* ms_per_host);
/* Device-side status word of the last layer (0 ok; bit 0: NaN score; bit 1: a
 * passing source selected fewer than l_p keys (non-finite scores) -- its fixed
 * l_p-row exchange slot would be attended with zero rows where the reference drops
 * them (approx.cpp:83-90); bit 2: a merged query row invalid in every part).
 * Synchronises the given stream.                                      */
int spava_host_status(spava_host* host, void* stream, int32_t* status_out);

/* DelayInjection analogue (simhost.hpp:51-55): spin `ns` nanoseconds on a stream before
 * a phase of every layer -- 0: scoring/selection (side stream), 1: exchange rounds (comm
 * stream), 2: query attention (caller stream), 3: stage 1.  Results must not change
 * (tests/test_gpu_layer.py, acceptance.cpp:221-268 criterion 5).                     */
int spava_host_set_delay(spava_host* host, int which, uint64_t ns);

/* Schedule trace in the reference Event schema (simhost.hpp:17-46): while enabled, every
 * layer call records run_host's events (score, pass1/pass2/qpartial issue / wait-start /
 * completed, query_attn, stage1, stage2, merge begin/end; simhost.cpp:322-426) in program
 * order with the device time of the stream position each one marks (microseconds from a
 * per-fabric origin).  Tags are "<round>.L<layer>" as in the reference.  The caller
 * assigns seq and Lamport clocks across hosts and can run seqpar::validate_trace
 * (simhost.cpp:567-657) on the result (tests/test_gpu_trace.py).                   */
typedef struct {
  int kind;        /* 0 CommIssued, 1 CommWaitStart, 2 CommCompleted, 3 ComputeBegin, 4 ComputeEnd */
  int layer;
  char label[16];
  char tag[24];    /* "" for compute events */
  double t_us;
} spava_trace_event;
int spava_host_set_trace(spava_host* host, int enable);  /* resets the record and layer count */
/* out == NULL: *n = number of records; else copies (synchronising on the events). */
int spava_host_trace_read(spava_host* host, spava_trace_event* out, int cap, int* n);

/* Device timing of this host's launches, by kernel class (0 attention, 1 score,
 * 2 select+pack, 3 merge): CUDA events on the launching stream around every
 * launch while enabled (enable = 2 additionally runs the scorer on the caller's stream
 * instead of the overlapping side stream, so kernels are timed in isolation).
 * spava_host_set_timing resets the counters;
 * spava_host_timing synchronises on the recorded events and returns the summed
 * milliseconds per class, the algorithmic attention FLOPs launched (reference
 * convention, attention.cpp:33-36) and the attention launch count.           */
int spava_host_set_timing(spava_host* host, int enable);
int spava_host_timing(spava_host* host, double* ms_by_class4, double* attn_flops,
                      uint64_t* attn_launches);

/* Development: read-and-reset the cycle counters of the instrumented attention
 * variant (SPAVA_ATTN_VARIANT=5): 16 uint64 (see attention.cu).            */
int spava_debug_attn_prof(uint64_t* out16);
/* Development: force an attention kernel variant for this process (-1 = default or the
 * SPAVA_ATTN_VARIANT environment variable); lets the tests cover every variant.        */
int spava_debug_attn_variant(int variant);
/* Development: 1 = the final query merge runs as trailing CTAs of the last stage launch
 * (default; peer fabric: they wait for the peers' qpartial flags in-kernel), 0 = a separate
 * merge launch after a stream wait, -1 = default / SPAVA_FUSED_MERGE.                     */
int spava_debug_fused_merge(int on);
/* Development: 1 = fast-mode scoring (score_mode 1) rides in the query attention launch
 * (default: row statistics from its softmax + trailing column-sum CTAs), 0 = the standalone
 * three-launch tensor-core scorer, -1 = default / SPAVA_FUSED_SCORE.                     */
int spava_debug_fused_score(int on);

/* Number of kernels the library launched since process start (for bench's
 * gpu_launches claim). */
uint64_t spava_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* SPAVA_B200_H */
