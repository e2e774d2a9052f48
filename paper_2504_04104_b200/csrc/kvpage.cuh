// Paged KV cache of the Llama path (replaces the reference's grow-by-doubling
// per-layer arrays, `/root/reference/pkg/src/treepipe/model.py:105-148`).
//
// A stage's cache rows are grouped into pages of kPageRows = 64 rows (one
// canonical attention chunk).  One physical page holds those 64 rows of ONE
// layer for every KV head, K block then V block:
//
//   page = [K | V][kv_heads][2 dim-blocks][64 rows][64 dims]   (bf16)
//
// Each (K|V, kv head) block is 16 KB laid out exactly as a tcgen05 operand in
// shared memory with the 128-byte swizzle: row r of dim-block b at
// b * 8192 + r * 128, its 16-byte column chunk c stored at chunk position
// c ^ (r & 7).  K is then the K-major B operand of S = Q K^T and V the
// MN-major B operand of O = P V, so the attention kernel stages a whole chunk
// with one 16 KB bulk copy per operand and no re-layout.
//
// Pages come from a per-model pool (all requests / stages of a model object
// share it); a stage owns a page table [layers][max_pages] of page base
// pointers.  Growth appends pages (no copy); pruning compacts rows through the
// table (rows only move toward lower indices).
#pragma once

#include <stdint.h>

namespace tp {

constexpr int kPageRows = 64;
constexpr int kPageBlockBytes = kPageRows * 128 * 2;  // one (K|V, kv head) block: 16 KB

__host__ __device__ inline int64_t page_bytes(int kv_heads) { return 2 * (int64_t)kv_heads * kPageBlockBytes; }

// Byte offset of the 16-byte chunk e (dims 8e .. 8e+7, e in [0, 16)) of row r (< 64)
// inside a (K|V, kv head) block.
__host__ __device__ inline int page_chunk_off(int r, int e) {
  return ((e >> 3) << 13) + (r << 7) + (((e & 7) ^ (r & 7)) << 4);
}

// Device view of one stage's K/V storage (paged Llama cache, or the toy's flat
// [layer][K|V] planes of [heads][cap][row]).
struct KvView {
  char* const* tab;      // paged: [layers][max_pages] page bases; flat: [2 * layers] plane bases
  int paged;
  int max_pages;         // paged: table stride
  int heads;             // kv heads
  int row_bytes;         // flat rows (toy): bytes per row
  int64_t plane_stride;  // flat: bytes between kv-head planes
};

// 16-byte chunk e of (layer slot l, kind 0 = K / 1 = V, kv head h, row).
__device__ __forceinline__ char* kv_chunk(const KvView& v, int l, int kind, int h, int row, int e) {
  if (!v.paged)
    return v.tab[2 * l + kind] + (int64_t)h * v.plane_stride + (int64_t)row * v.row_bytes + 16 * e;
  char* pg = v.tab[(int64_t)l * v.max_pages + (row >> 6)];
  return pg + (int64_t)(kind * v.heads + h) * kPageBlockBytes + page_chunk_off(row & 63, e);
}

// Base of the (K|V, kv head) block of the page holding `row` (paged only).
__device__ __forceinline__ const char* kv_block(const char* const* layer_tab, int heads, int kind, int h, int row) {
  return layer_tab[row >> 6] + (int64_t)(kind * heads + h) * kPageBlockBytes;
}

// Stable in-place compaction of one (layer slot l, K|V, kv head) plane: kept
// rows (src_rows, increasing, src_rows[j] >= first + j) are staged through
// shared memory in chunks of kChunk bytes, then stored at first, first + 1, ...
// (rows only move toward lower indices, so a later chunk never overwrites a row
// an earlier one still has to read).  The leading run already in place is
// skipped.  Call from every thread of the CTA.
template <int kChunk>
__device__ __forceinline__ void kv_move_plane(const KvView& v, int l, int kind, int head,
                                              const int32_t* __restrict__ src_rows, int n_keep, int first,
                                              uint4* stage) {
  int j0 = 0;
  while (j0 < n_keep && src_rows[j0] == first + j0) ++j0;
  const int vec_per_row = v.row_bytes / 16;
  const int rows_per_chunk = max(1, kChunk / v.row_bytes);
  for (int c = j0; c < n_keep; c += rows_per_chunk) {
    const int cnt = min(rows_per_chunk, n_keep - c);
    const int total = cnt * vec_per_row;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
      const int r = t / vec_per_row, e = t % vec_per_row;
      stage[t] = *reinterpret_cast<const uint4*>(kv_chunk(v, l, kind, head, src_rows[c + r], e));
    }
    __syncthreads();
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
      const int r = t / vec_per_row, e = t % vec_per_row;
      *reinterpret_cast<uint4*>(kv_chunk(v, l, kind, head, first + c + r, e)) = stage[t];
    }
    __syncthreads();
  }
}

}  // namespace tp
