/*
 * treepipe_b200.h — C ABI of the B200-native SpecPipe step (arXiv 2504.04104).
 *
 * The reference (`/root/reference/pkg/src/treepipe`) is pure Python; its seam
 * for this path is duck-typed module globals that `pipeline.py` binds at import
 * (`pipeline.py:35`).  Each entry point below replaces one of those calls; the
 * Python host mirror (`paper_2504_04104_b200/model.py`) binds them with ctypes
 * under the reference names.  Plain pointers and sizes only: "host" arrays are
 * CPU memory, "dev" pointers are CUDA device memory on the model's device.
 *
 * Status codes map onto the reference exception hierarchy (errors.py:4-49):
 *   TP_ESHAPE -> ShapeError, TP_ECONTRACT -> ContractViolation,
 *   TP_EINVARIANT / TP_ECUDA -> InvariantViolation, TP_ECONFIG -> ConfigError.
 *
 * Threading: calls on distinct stages may run concurrently (the reference's
 * worker mode, pipeline.py:195-199,303-307); calls on one stage are serialised
 * by the caller.  All kernels are deterministic (no float atomics) and
 * batch-invariant: a node's result does not depend on which other nodes
 * share the launch.
 */
#ifndef TREEPIPE_B200_H
#define TREEPIPE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TP_OK 0
#define TP_ESHAPE 1
#define TP_ECONTRACT 2
#define TP_EINVARIANT 3
#define TP_ECONFIG 4
#define TP_ECUDA 5

#define TP_ARCH_TOY 0   /* reference ToyModel: f64, LN, sinusoid, 1 head, ReLU FFN, tied head */
#define TP_ARCH_LLAMA 1 /* Llama-shape: bf16 weights, RMSNorm, RoPE, GQA, SwiGLU, LM head */

typedef struct tp_model tp_model; /* weights of a layer range on one device   */
typedef struct tp_stage tp_stage; /* KV cache + workspace of one pipeline stage */

typedef struct tp_model_config {
  int32_t arch;
  int32_t vocab, hidden, layers;             /* full-model shape                    */
  int32_t heads, kv_heads, head_dim, ffn;    /* llama (toy: 1, 1, hidden, 2*hidden) */
  int32_t layer_lo, layer_hi;                /* layers hosted by this object        */
  int32_t with_embed, with_head;             /* embedding table / final norm + head */
  int32_t device;
  int32_t max_nodes;                         /* nodes per forward launch (<= 1024; Llama <= 256) */
  float rope_theta, norm_eps;
  int32_t weight_scale;                      /* llama: 1 = x sqrt(3/fan_in)/0.1     */
} tp_model_config;

/* One tree level (or prompt chunk) to push through a stage's layers.
 * Node i attends cache rows [0, prefix_rows[i]) then, in increasing order,
 * rows bits_base + b for every set bit b of anc_bits[i*words .. +words), then
 * itself (self last) — the reference's `rows_for` + self
 * (model.py:157-163, 265-271).  With append=1 node i's K/V become cache row
 * rows()+i (KvCache.begin_row/append, model.py:136-152).                    */
typedef struct tp_level {
  int32_t n;
  int32_t append;
  const int32_t* tokens;      /* host [n]; read when hidden_in == NULL       */
  const int32_t* positions;   /* host [n]                                     */
  const int32_t* prefix_rows; /* host [n]                                     */
  int32_t words;              /* u64 words per node mask (0 = none)          */
  int32_t bits_base;          /* cache row addressed by bit 0                 */
  const uint64_t* anc_bits;   /* host [n*words], self bit excluded           */
  int32_t layer_lo, layer_hi; /* sub-range of the stage's layers (0,0 = all)  */
  /* Tree form (optional; prefix_rows / anc_bits may then be NULL): node i is
   * tree node tree_lo + i; it attends rows [0, tree_prefix) and, for every
   * ancestor t >= tree_off in its packed ancestor-or-self tree row
   * tree_bits[(tree_lo+i)*words ...] (self excluded), row tree_prefix - tree_off + t.
   * This is invariant I1/I2 of the reference cache evaluated here
   * instead of in Python for every stage and request.                          */
  const uint64_t* tree_bits;
  int32_t tree_lo, tree_off, tree_prefix;
} tp_level;

const char* tp_last_error(void);
int tp_device_count(int32_t* out);

/* ---- model: replaces ToyModel(cfg) / init_model (model.py:207-236) ------- */
int tp_model_create(const tp_model_config* cfg, tp_model** out);
int tp_model_destroy(tp_model* m);
/* LCG weight stream (model.py:28-44) generated on device, jump-ahead per thread. */
int tp_model_init_lcg(tp_model* m, uint64_t seed, void* stream);
/* The reference weight stream itself (lcg_uniform_stream, model.py:33-44): count
 * f64 samples starting at stream index `start`, written to dev memory.          */
int tp_lcg_uniform(int32_t device, uint64_t seed, int64_t start, int64_t count, void* out_dev, void* stream);
/* Raw tensor I/O (checkpoint import/export, model.py:388-435; tests).
 * which: 0 embedding, 1..6 toy Wq,Wk,Wv,Wo,W1,W2 ([in,out] row-major f64);
 *        llama: 1 Wq 2 Wk 3 Wv 4 Wo 5 Wgate 6 Wup 7 Wdown ([out,in] bf16), 8 lm_head. */
int tp_model_tensor_bytes(const tp_model* m, int32_t which, int32_t layer, int64_t* nbytes);
int tp_model_write_tensor(tp_model* m, int32_t which, int32_t layer, const void* host, int64_t nbytes);
int tp_model_read_tensor(const tp_model* m, int32_t which, int32_t layer, void* host, int64_t nbytes);

/* ToyModel.embed (model.py:239-240) / Llama token embedding, n rows -> dev. */
int tp_model_embed(tp_model* m, int32_t n, const int32_t* tokens, const int32_t* positions,
                   void* out_dev, void* stream);
/* ToyModel.head (model.py:242-244): final norm + head, n rows -> f32/f64 logits (dev). */
int tp_model_logits(tp_model* m, tp_stage* ws, int32_t n, const void* hidden_dev, void* logits_dev,
                    void* stream);
/* Verify (model.py:247-248 + pipeline.py:328-339): greedy token of one hidden
 * row (first argmax) and the first child whose token matches.  result_host =
 * {token, child_index or -1}; synchronises the stream.                        */
int tp_model_verify(tp_model* m, tp_stage* ws, const void* hidden_dev, const int32_t* child_tokens,
                    int32_t n_children, int32_t* result_host, void* stream);
/* The same verification split in two so the host never drains the stream:
 * _async enqueues head + argmax + child match + the 8-byte D2H and returns;
 * _wait blocks on that work only (not on anything enqueued after it).        */
int tp_model_verify_async(tp_model* m, tp_stage* ws, const void* hidden_dev, const int32_t* child_tokens,
                          int32_t n_children, void* stream);
int tp_model_verify_wait(tp_stage* ws, int32_t* result_host);
/* greedy_token of n rows at once (one per request in a SpecPipe-DB tick):
 * _async enqueues final norm + LM head (one GEMM for all rows) + per-row first
 * argmax + the D2H; _wait returns the n tokens.                              */
int tp_model_greedy_rows_async(tp_model* m, tp_stage* ws, int32_t n, const void* hidden_dev, void* stream);
int tp_model_greedy_rows_wait(tp_model* m, int32_t n, int32_t* tokens_host);

/* ---- stage: replaces KvCache (model.py:105-204) + forward_tree (:312-349) - */
int tp_stage_create(tp_model* m, int32_t layer_lo, int32_t layer_hi, int32_t capacity_rows,
                    tp_stage** out);
int tp_stage_destroy(tp_stage* s);
int tp_stage_rows(const tp_stage* s, int32_t* rows);
/* forward_tree / forward_position for the stage's layers.  hidden: [n, hidden]
 * (f64 toy, f32 llama residual stream).  hidden_in == NULL embeds tokens.  */
int tp_stage_forward(tp_stage* s, const tp_level* level, const void* hidden_in, void* hidden_out,
                     void* stream);
/* Phase 1 of PipelineRunner.step (pipeline.py:289-312) for several stages hosted on
 * ONE device: stage g pushes levels[g] through its layers.  Llama stages run
 * layer slot by layer slot with one grouped GEMM launch per slot (up to 8
 * stages per launch); results are bit-identical to `count` separate
 * tp_stage_forward calls.  Stages must be distinct and share device + arch.   */
int tp_stages_forward(int32_t count, tp_stage* const* stages, const tp_level* levels, const void* const* hidden_in,
                      void* const* hidden_out, void* stream);
/* Ragged multi-request form (SpecPipe-DB combined step, batching.py:226-264):
 * every item is one request's level on one of its stage caches; items with the
 * same `member` (same layers, same model object) are concatenated into one
 * ragged batch — one GEMM over all their node rows (weights streamed once per
 * tick, not once per request), K/V scattered into each request's own cache,
 * attention per request (block-diagonal by construction, batching.py:90-126).
 * member_hidden_out[g] is the [sum_n, hidden] fp32 residual stream of member g,
 * items in their order; member ids must be first-use ordered from 0.          */
typedef struct tp_item {
  tp_stage* stage;
  tp_level level;
  const void* hidden_in; /* device [n, hidden] rows, or NULL to embed level.tokens */
  int32_t member;
} tp_item;
int tp_items_forward(int32_t n_items, const tp_item* items, void* const* member_hidden_out, void* stream);
/* The same with the model's scratch workspaces taken from slot ws_base on: two
 * calls with disjoint slot ranges may run concurrently on two streams.        */
int tp_items_forward_ws(int32_t n_items, const tp_item* items, void* const* member_hidden_out, int32_t ws_base,
                        void* stream);
/* Pruning propagation (KvCache.promote/prune/_restrict/drop_speculative,
 * model.py:169-194): rows < first_row stay; of rows [first_row, first_row+count)
 * those with keep bit set are compacted stably to follow them; the rest and
 * every row beyond are dropped.                                              */
int tp_stage_compact(tp_stage* s, int32_t first_row, int32_t count, const uint64_t* keep_bits,
                     void* stream);
int tp_stage_truncate(tp_stage* s, int32_t rows);
/* tp_stage_compact for several stages of one device (every stage's prune of one
 * verification, pipeline.py:341-361) in one upload + one launch.            */
int tp_stages_compact(int32_t count, tp_stage* const* stages, const int32_t* first_rows, const int32_t* counts,
                      const uint64_t* const* keep_bits, void* stream);
/* Copy K (kind 0) or V (kind 1) of one layer, rows [lo,hi), as [rows][kv_heads][head_dim]. */
int tp_stage_read_kv(const tp_stage* s, int32_t layer, int32_t kind, int32_t lo, int32_t hi, void* host);

/* ---- K3 driven by the device-resident verification (pipeline.py:333-400) ---
 * Enqueued right after tp_model_verify_async, before the host knows tau: the
 * device reads tau from the verify stage's result, finds the first level-1 child
 * carrying it (level-1 tokens given here, BFS order), and for every stage
 *   - compacts the K/V rows: rows < prefix_rows stay; speculative row r (tree node
 *     tree_off + r, invariant I2) is kept iff it is an ancestor-or-self or a
 *     descendant-or-self of the child (row | col of the tree mask); on a miss
 *     only the root row (tree node 0, promoted) is kept;
 *   - gathers the surviving hidden rows of its resident level (tree nodes
 *     level_lo .. +level_n, kept iff descendant-or-self of the child) from
 *     hidden_src to hidden_dst (hidden_src may live on a peer GPU).
 * The stages' host row counts are then set with tp_stage_truncate once the
 * caller has tau (the K/V data is final when the stream reaches the kernels).
 * keep_out (optional, device int32 [2 + spec_rows + level_n]) receives the kept
 * counts and row lists — the reference's _restrict keep lists (tests).
 * stage may be NULL for a hidden-rows-only entry (prefix/spec rows 0): the
 * receiver side of a cross-device hand-off, whose rows were sent before the
 * verification (tp_peer_copy) and are compacted on the receiving device.     */
typedef struct tp_prune_stage {
  tp_stage* stage;
  int32_t prefix_rows, spec_rows, tree_off;
  int32_t level_lo, level_n;
  const void* hidden_src;
  void* hidden_dst;
  int32_t* keep_out;
} tp_prune_stage;
int tp_prune_device(int32_t count, const tp_prune_stage* stages, const tp_stage* verify_ws,
                    const uint64_t* tree_bits, int32_t tree_n, int32_t words, const int32_t* level1_tokens,
                    int32_t n_level1, int64_t hidden_row_bytes, void* stream);

/* ---- cross-device step (stage-per-GPU; pipeline.py:373-439) --------------
 * tp_result_mirror: the 16-byte verification result of src_ws (K4, possibly on
 * a peer GPU) -> dst_ws's result word, ordered on `stream` (the receiving
 * device's stream; the caller makes it wait for the K4 launch first).  Every
 * device then runs tp_prune_device from its own copy.
 * tp_peer_copy: cudaMemcpyPeerAsync on `stream` (the send-before-verify
 * hand-off of a stage's output rows to the next stage's device).            */
int tp_result_mirror(tp_stage* dst_ws, const tp_stage* src_ws, void* stream);
int tp_peer_copy(void* dst, int32_t dst_device, const void* src, int32_t src_device, int64_t bytes, void* stream);

/* ---- transmit: in-flight embedding filter (pipeline.py:379-400) ---------- */
/* dst[j] = src[i_j] for the set bits i_0 < i_1 < ... of keep_bits (n_src rows of row_bytes). */
// Draft model proposals (BASELINE configs 2 and 4): the k (<= 32) best token ids of
// each of n_rows fp32 logit rows, value descending, lowest id first on ties (no
// reference counterpart: the reference's drafts are synthetic; CostModel.draft_ms).
int tp_topk_rows(int32_t device, const void* logits_dev, int32_t vocab, int32_t n_rows, int32_t k, void* out_dev,
                 void* stream);
int tp_rows_compact(tp_stage* ws, const void* src_dev, void* dst_dev, int64_t row_bytes, int32_t n_src,
                    const uint64_t* keep_bits, int32_t* n_out, void* stream);
/* tp_rows_compact for up to 64 row sets (every stage's in-flight filter of one
 * step, pipeline.py:379-400) in one upload + one launch; n_out[i] returned.  */
int tp_rows_compact_many(int32_t count, tp_stage* ws, const void* const* src_dev, void* const* dst_dev,
                         int64_t row_bytes, const int32_t* n_src, const uint64_t* const* keep_bits, int32_t* n_out,
                         void* stream);
/* Grow the KV capacity (reference KvCache grow-by-doubling, model.py:141-148). */
int tp_stage_reserve(tp_stage* s, int32_t capacity_rows);

/* ---- host control: synthetic draft (token_source.py:73-111), pure host code ---
 * Bit-exact restatement of the numpy draws of one synthetic_draft call
 * (SeedSequence([seed, call_index]) -> PCG64 -> random / geometric / choice).
 * oracle_next < 0 = no bound continuation.  TP_ECONFIG = a numpy branch not
 * restated here (geometric with p < 1/3, tail-shuffle choice): use numpy.     */
int tp_synthetic_draft(uint64_t seed, int64_t call_index, int32_t oracle_next, double top1_hit, double rank_decay,
                       double miss_prob, int32_t k, int32_t vocab, int32_t* tokens_out, int32_t* n_out);
int tp_synthetic_draft_batch(int32_t count, uint64_t seed, int64_t call_index0, const int32_t* oracle_next,
                             double top1_hit, double rank_decay, double miss_prob, int32_t k, int32_t vocab,
                             int32_t* tokens_out, int32_t* n_out);

/* ---- instrumentation (no reference counterpart; used by bench.py) ---------- */
/* Kernels launched by this library since load (every launch site counts). */
int tp_launch_count(int64_t* out);
// Instrumentation: CUDA-graph replays of lone forwards so far (TP_GRAPH mode, llama.cu).
int tp_graph_launches(int64_t* n);
/* Host<->device bytes moved by this library's own copies since load. */
int tp_io_bytes(int64_t* h2d, int64_t* d2h);
/* Time every K2 GEMM launch with CUDA events on its stream while enabled;
 * tp_profile_read returns summed ms, algorithmic bytes and launch count, then resets. */
int tp_profile_enable(int32_t on);
int tp_profile_read(double* gemm_ms, double* gemm_bytes, int64_t* launches);
// The same per-launch records split by the launch's member count: arrays of 8
// (index = members - 1: 1 = a lone stage, 2 = a stage + the fused draft model, ...).
int tp_profile_read_members(double* gemm_ms, double* gemm_bytes, int64_t* launches);

/* ---- test hook (no reference counterpart): the K2 weight-streaming GEMM alone.
 * out[n][n_out] (f32, dev) = x[n][k] (bf16, dev) . w[n_out][k]^T (bf16, dev).   */
int tp_debug_gemm(int32_t device, const void* w_dev, const void* x_dev, int32_t n, int32_t n_out, int32_t k,
                  void* out_dev, void* stream);
/* The same GEMM launched `iters` times back to back (programmatic dependent
 * launch between them); *ms_per_launch = CUDA-event time / iters.            */
int tp_debug_gemm_timed(int32_t device, const void* w_dev, const void* x_dev, int32_t n, int32_t n_out, int32_t k,
                        void* out_dev, int32_t iters, float* ms_per_launch, void* stream);

/* Grouped variant: `count` (<= 8) same-shape GEMMs in one launch, as phase 1 runs them. */
int tp_debug_gemm_group_timed(int32_t device, int32_t count, const void* const* w_dev, const void* const* x_dev,
                              const int32_t* n, int32_t n_out, int32_t k, void* const* out_dev, int32_t iters,
                              float* ms_per_launch, void* stream);
// Tests: one heterogeneous grouped K2 launch (member g: its own shape and plan).
int tp_debug_gemm_hetero(int32_t device, int32_t count, const void* const* w_dev, const void* const* x_dev,
                         const int32_t* n, const int32_t* n_out, const int32_t* k, void* const* out_dev, void* stream);
// Diagnostics: device buffer [launch < 64][grid][32] u64 receiving K2 phase timestamps, launches numbered
// from this call in start order (builds with -DTP_GEMM_TRACE).
int tp_debug_gemm_trace(int32_t device, void* dev_buf);
/* K4 on caller-provided device logits (tests): n_rows == 1 with children -> out[0] = first argmax,
 * out[1] = first child whose token equals it (or -1); otherwise out[r] = first argmax of row r (fp32). */
int tp_debug_argmax(int32_t device, const void* logits_dev, int32_t is_f64, int32_t vocab, int32_t n_rows,
                    const int32_t* children_host, int32_t n_children, int32_t* out_host);
/* K1 routing (tests): 1 runs uniform tree levels through the 16-node tile path,
 * 0 (default) the per-node tail path.                                          */
int tp_debug_attn_tile(int32_t on);
/* K1 knobs: 0 = tile path on/off (as above), 1 = shared-prefix chunks per CTA (1..4),
 * 2 = shared-prefix tail for uniform levels on/off, 3 = diagnostic skip mask for the
 * Llama layer loop (bit 1 attention, 2 RMSNorm, 4 GEMMs; results WRONG while set). */
int tp_debug_attn_knob(int32_t knob, int32_t value);
/* Diagnostics: K1 run-kernel event trace buffer ([grid][8][1024] u64; only -DTP_ATTN_TRACE builds write). */
int tp_debug_attn_trace(void* dev_buf);
/* Diagnostics: the next Llama forward call copies member 0's first-layer
 * intermediates into dev_buf (input RMSNorm bf16 [n][d], RoPE'd queries bf16
 * [n][q], attention out bf16 [n][q], x after the
 * o-projection f32 [n][d], RMSNorm out bf16 [n][d], SwiGLU product bf16 [n][f],
 * x after the down projection f32 [n][d]); one-shot.                          */
int tp_debug_dump(void* dev_buf);
/* GPU timeline (diagnostics): while enabled, CUDA events between kernel groups;
 * _read returns "tag=ms;..." (GPU time since the previous mark on the stream,
 * summed per tag) and resets.                                                 */
int tp_timeline_enable(int32_t on);
int tp_timeline_read(char* buf, int32_t len);
/* Tuning knobs of K2 (0: ring depth cap, 1: smem budget in KB, 2: fix-up diagnostics —
 * 1/2 skip the stream-K reduction / also the partial publish, WRONG results); process-wide. */
int tp_debug_gemm_knob(int32_t knob, int32_t value);

#ifdef __cplusplus
}
#endif
#endif /* TREEPIPE_B200_H */
