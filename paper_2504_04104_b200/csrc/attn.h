// K1: tree-masked attention for the Llama path (see attn.cu).
#pragma once

#include "internal.h"

namespace tp {

constexpr int kAttnChunk = 64;     // logical key slots per canonical chunk
constexpr int kAttnSuffix = 16;    // node-specific window at the end of the key sequence (> ancestors)
constexpr int kAttnMaxExtra = 64;  // speculative ancestor rows per node
constexpr int kAttnHeadDim = 128;
constexpr int kAttnMaxGroup = 64;  // (request, stage) items per grouped launch (large kernel params)

struct AttnArgs {
  const __nv_bfloat16* q;  // [n][H*128]
  int q_stride;
  const __nv_bfloat16* k;  // cache [KV][cap][128]
  const __nv_bfloat16* v;
  int cap;
  const __nv_bfloat16* kself;  // self rows: [n][KV][128] (recompute) or nullptr (cache rows row0+i)
  const __nv_bfloat16* vself;
  int H, KV;
  float scale;
  float* pm;  // [n][H][max_chunks] per-run max          (shared runs only)
  float* pl;  // per-run sum
  float* po;  // [n][H][max_chunks][128] per-run unnormalised output
  int max_chunks;
  __nv_bfloat16* out;  // [n][H*128]
  int out_stride;
};

// One grouped launch pair covers the same layer slot of several stages.
struct AttnMember {
  AttnArgs a;
  LevelDev lv;
  int c_shared;    // chunks of the member's longest chunked part (slots [0, T - kAttnSuffix))
  int max_c;       // slots of that part
  int zt;          // row blocks of the shared launch (64 rows; 16-row tiles when `small`)
  int small;       // few rows: the run's chunks in parallel across warps
  int cta_shared;  // first CTA of this member in the shared launch
  int cta_tail;    // first CTA of this member in the per-node tail launch (empty range for GQA)
  int cta_gqa;     // first CTA of this member in the GQA tail launch (one CTA per node and KV head)
};

struct AttnGroup {
  AttnMember m[kAttnMaxGroup];
  int count;
  int run;  // canonical chunks per run
};

int attn_tree(const AttnArgs& a, const LevelDev& lv, cudaStream_t st);
int attn_set_run(int run);
// members[0..count) -> two launches (shared chunks, then per-node tail + ordered combine)
int attn_tree_group(const AttnArgs* a, const LevelDev* lv, int count, cudaStream_t st);

}  // namespace tp
