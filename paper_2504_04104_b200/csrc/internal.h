// Internal object layout shared by the C-ABI (api.cu) and the kernel files.
#pragma once

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "kvpage.cuh"

// Per-layer weights.  Toy: f64 [in,out] row-major as the reference stores
// them (model.py:72-80).  Llama: bf16 [out,in] (K-major for the swap-AB
// tcgen05 GEMM: weights are the MMA "A" operand, tree nodes the "B" operand).
struct tp_layer_weights {
  void* w[8] = {nullptr};
  int64_t bytes[8] = {0};
};

struct tp_model {
  tp_model_config cfg;
  void* embed = nullptr;  // [V, d] (f64 toy / bf16 llama)
  void* head = nullptr;   // llama lm_head [V, d] bf16 (toy: tied to embed)
  int64_t embed_bytes = 0, head_bytes = 0;
  std::vector<tp_layer_weights> layers;  // index layer - cfg.layer_lo
  // llama: tensor maps for TMA live beside the weights (filled lazily)
  void* tma_cache = nullptr;
  void* call_ring = nullptr;  // staging ring for multi-level / multi-stage calls (api.cu)
  int32_t* prune_plan = nullptr;  // device keep lists of tp_prune_device (prune.cu)
  size_t prune_plan_ints = 0;
  // Destroyed stages are parked here and reused by tp_stage_create (same layer
  // range, enough capacity): cudaFree / cudaFreeHost synchronise the device, and
  // a request finishing mid-stream (SpecPipe-DB) must not stall every other one.
  std::vector<tp_stage*> stage_pool;
  std::mutex pool_mu;
  // Stages keep their model alive: Python may finalise a model before its
  // caches (cyclic GC), so tp_model_destroy defers the free until the last
  // live stage is destroyed.
  int live_stages = 0;
  bool destroy_pending = false;
  // Llama KV page pool (kvpage.cuh): every stage / request of this model draws
  // its pages here (guarded by pool_mu); slabs are freed with the model.
  std::vector<char*> page_free;
  std::vector<void*> page_slabs;
};

struct tp_stage {
  tp_model* m = nullptr;
  int lo = 0, hi = 0;     // hosted layers
  int cap = 0, rows = 0;  // KV capacity / filled rows
  int kv_heads = 1, head_dim = 0, esize = 8;
  std::vector<void*> k, v;  // toy: per hosted layer [kv_heads][cap][head_dim] (flat planes)
  // llama: paged KV (kvpage.cuh), cap = pages * 64
  std::vector<char*> ptab;   // host copy of the page table [layers][max_pages]
  char** d_ptab = nullptr;   // device page table
  int max_pages = 0;
  // device workspace
  char* ws = nullptr;
  size_t ws_bytes = 0;
  // metadata uploads (tokens, positions, prefix rows, anc bits, index lists) go
  // through a ring of kMetaRing (pinned host, device) slot pairs, so the host
  // only waits when it laps an upload the stream has not executed yet
  static constexpr int kMetaRing = 8;
  char* meta = nullptr;       // device: kMetaRing slots of meta_bytes
  char* host_meta = nullptr;  // pinned host: same layout
  size_t meta_bytes = 0;      // bytes per slot
  int max_words = 0;
  cudaEvent_t meta_ev[kMetaRing] = {nullptr};
  int meta_next = 0;
  cudaEvent_t verify_ev = nullptr;  // async verify: result landed in h_result
  // verify result staging
  int32_t* d_result = nullptr;
  int32_t* h_result = nullptr;
  void** d_planes = nullptr;  // toy: [2*layers] K/V plane bases for the compaction kernels
  void* logits = nullptr;     // [logits_rows][vocab] verify scratch (f64 toy / f32 llama)
  int logits_rows = 0;
  void* ext = nullptr;        // arch-specific state (llama: tensor maps, attention partials)
};

namespace tp {

// Device view of one forward call's per-node metadata.
struct LevelDev {
  int n;
  int append;
  int row0;  // first appended row (== rows before the call)
  int words;
  int bits_base;
  int layer_lo, layer_hi;  // layers to run
  int max_t;               // longest logical key sequence (prefix + ancestors + self)
  int min_p;               // smallest prefix_rows over the level's nodes
  int uniform_a;           // every node has this many ancestors and prefix min_p (-1: ragged level)
  const int32_t* tokens;
  const int32_t* positions;
  const int32_t* prefix_rows;
  const uint64_t* anc;  // [n][words]
  const int32_t* anc_cnt;   // [n] speculative ancestors per node (<= 64)
  const int32_t* anc_rows;  // [n][anc_stride] their cache rows, increasing
  int anc_stride;
};

int fill_lcg_jump_table();
int lcg_fill_f64(double* out, int64_t count, uint64_t seed, int64_t start, cudaStream_t st);

// toy arch (toy.cu)
int toy_forward(tp_stage* s, const LevelDev& lv, const void* hidden_in, void* hidden_out,
                cudaStream_t st);
int toy_embed(tp_model* m, int n, const int32_t* d_tokens, const int32_t* d_pos, double* out,
              cudaStream_t st);
int toy_logits(tp_model* m, tp_stage* ws, int n, const double* x, double* logits, cudaStream_t st);
int toy_workspace_bytes(const tp_model* m, int max_nodes, size_t* bytes);

// llama arch (llama.cu)
int llama_forward(tp_stage* s, const LevelDev& lv, const void* hidden_in, void* hidden_out,
                  cudaStream_t st);
// One item = one request's level on one stage; a member = items sharing layers
// (a ragged batch: rows concatenated in x, one GEMM member).
struct FwdItem {
  tp_stage* s;
  LevelDev lv;
  const void* hin;  // device rows or nullptr (embed tokens)
};
struct FwdMember {
  const FwdItem* items;
  int count;
  float* x;  // [sum n, hidden] residual stream of the member
};
// ws_base: first model workspace slot used (concurrent calls on two streams use disjoint slots)
int llama_forward_members(const FwdMember* mem, int count, cudaStream_t st, int ws_base = 0);
int llama_greedy_rows_async(tp_model* m, int n, const float* x, float* logits, cudaStream_t st);
int llama_greedy_rows_wait(tp_model* m, int n, int32_t* out);
void timeline_mark(const char* tag, cudaStream_t st);  // no-op unless enabled
int argmax_rows(const void* logits_f32, int vocab, int n, int32_t* d_out, cudaStream_t st);
int call_slot(tp_model* m, size_t bytes, char** host, char** dev, int* slot);
int call_push(tp_model* m, int slot, size_t bytes, cudaStream_t st);
void call_ring_free(tp_model* m);
// metadata upload through a stage's staging ring (api.cu)
int upload(tp_stage* s, const void* host, size_t bytes, cudaStream_t st, const char** dev_out);
int llama_embed(tp_model* m, int n, const int32_t* d_tokens, float* out, cudaStream_t st);
int llama_logits(tp_model* m, tp_stage* ws, int n, const float* x, float* logits, cudaStream_t st);
int llama_workspace_bytes(const tp_model* m, int max_nodes, size_t* bytes);
int llama_init_weights(tp_model* m, uint64_t seed, cudaStream_t st);
int llama_stage_init(tp_stage* s);     // workspace tensor maps + attention scratch (after alloc_kv)
void llama_stage_free(tp_stage* s);
void llama_model_free(tp_model* m);
int lcg_fill_bf16(__nv_bfloat16* out, int64_t count, uint64_t seed, int64_t start, double scale,
                  cudaStream_t st);
// [rows_in, cols_out] stream block stored transposed into dst rows; gate/up interleave
// maps output column j to row (j/64)*128 + j%64 + row_offset.
int lcg_fill_bf16_rows(__nv_bfloat16* out, int64_t rows_in, int64_t cols_out, uint64_t seed, int64_t start,
                       double scale, int64_t row_offset, int interleave64, cudaStream_t st);

// shared (kv.cu)
int argmax_match(const void* logits, int is_f64, int vocab, const int32_t* d_children, int n_children,
                 int32_t* d_result, cudaStream_t st);
constexpr int kMaxMulti = 64;
struct MoveItem {
  KvView kv;            // the stage's K/V storage
  const int32_t* src;   // kept rows (device), increasing
  int n_keep, first, cta0;
};
struct MoveGroup {
  MoveItem m[kMaxMulti];
  int count;
};
struct RowsItem {
  const void* src;
  void* dst;
  const int32_t* idx;
  int n_out;
};
struct RowsGroup {
  RowsItem m[kMaxMulti];
  int count;
  int row_bytes;
};
int kv_compact_many(const MoveGroup& g, int ctas, cudaStream_t st);
int rows_compact_many(const RowsGroup& g, int max_rows, cudaStream_t st);
int kv_compact(tp_stage* s, const int32_t* d_src_rows, int n_keep, int first, cudaStream_t st);
KvView kv_view(const tp_stage* s);
// rows [lo, hi) of one layer's K (kind 0) or V plane -> device [rows][kv_heads][row bytes]
int kv_read_rows(const tp_stage* s, int layer, int kind, int lo, int hi, void* d_out, cudaStream_t st);
int rows_compact(const void* src, void* dst, int64_t row_bytes, const int32_t* d_idx, int n_out,
                 cudaStream_t st);

}  // namespace tp
