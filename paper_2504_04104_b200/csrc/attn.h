// K1: tree-masked attention for the Llama path (see attn.cu).
#pragma once

#include <cuda.h>

#include "internal.h"
#include "kvpage.cuh"

namespace tp {

constexpr int kAttnChunk = kPageRows;  // logical key slots per canonical chunk (== one KV page)
constexpr int kAttnSuffix = 16;        // node-specific window at the end of the key sequence (> ancestors)
constexpr int kAttnMaxExtra = 64;      // speculative ancestor rows per node
constexpr int kAttnHeadDim = 128;
constexpr int kAttnMaxGroup = 64;  // (request, stage) items per grouped launch (large kernel params)

struct AttnArgs {
  CUtensorMap qmap;        // the workspace's query rows as [nodes][H][128] (make_tmap_q3d)
  int q_row0;              // this item's first node in qmap
  const __nv_bfloat16* q;  // [n][H*128] (= qmap rows q_row0 ..)
  int q_stride;
  const char* const* ptab;  // this layer's page table row: page base per 64 cache rows
  int cap;
  const __nv_bfloat16* kself;  // self rows: [n][KV][128] (recompute) or nullptr (cache rows row0+i)
  const __nv_bfloat16* vself;
  int H, KV;
  float scale;
  float* pm;  // [n][H][max_chunks] per-run max
  float* pl;  // per-run sum
  float* po;  // [n][H][max_chunks][128] per-run unnormalised output
  int max_chunks;
  __nv_bfloat16* out;  // [n][H*128]
  int out_stride;
};

// One grouped launch pair covers the same layer slot of several stages / requests.
struct AttnMember {
  AttnArgs a;
  LevelDev lv;
  int c_hi;      // chunks of the member's longest chunked part (slots [0, T - kAttnSuffix))
  int blocks;    // 128-row blocks of (node, query head) rows
  int cta_run;   // first CTA of this member in the run launch
  int cta_tail;  // first CTA of this member in the tail launch
};

// Kernel parameters are copied per launch, so a launch carries only as many member
// slots as it needs: 1 (a lone stage), 8 (a device's stages) or 64 (SpecPipe-DB).
template <int MG>
struct AttnGroupT {
  AttnMember m[MG];
  int count;
  int run;  // canonical chunks per run
};
using AttnGroup = AttnGroupT<kAttnMaxGroup>;
static_assert(sizeof(AttnGroup) <= 32000, "AttnGroup must fit the 32 KB kernel-parameter limit");

int attn_tree(const AttnArgs& a, const LevelDev& lv, cudaStream_t st);
int attn_set_run(int run);
int attn_set_trace(void* dev_buf);  // diagnostics (-DTP_ATTN_TRACE builds): [grid][8 roles][1024] u64
// members[0..count) -> two launches (run states on tcgen05, then per-node suffix + ordered merge)
int attn_tree_group(const AttnArgs* a, const LevelDev* lv, int count, cudaStream_t st);

}  // namespace tp
