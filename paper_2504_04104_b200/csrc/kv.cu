// K3 (pruning propagation) and K4's argmax/child-match tail.
//
// kv_compact: stable in-place compaction of a stage's speculative KV rows
// (reference KvCache.promote/prune/_restrict, model.py:169-194).  Kept rows
// only ever move toward lower indices, so one CTA per (layer, K|V, kv-head)
// walks the kept list in chunks: stage CH rows in shared memory, barrier,
// store, barrier — a later chunk can never overwrite a row an earlier
// chunk still has to read.  Rows already in place (the leading kept run)
// are skipped, so a steady-state hit moves only the rows behind the first
// pruned sibling.
//
// argmax_match: deterministic first-argmax over the vocabulary (np.argmax
// semantics, lowest id wins ties, NaN ranks highest) followed by the
// first-level-1-child match of pipeline.py:333-339.
#include "internal.h"

namespace tp {

constexpr int kMoveThreads = 256;
constexpr int kMoveChunkBytes = 32 * 1024;

// One stage: CTA (plane = 2 * layer + kind, kv head).
__global__ void __launch_bounds__(kMoveThreads) kv_move_kernel(const KvView v, const int32_t* __restrict__ src_rows,
                                                               int n_keep, int first) {
  pdl_wait();
  pdl_trigger();
  __shared__ __align__(16) uint4 stage[kMoveChunkBytes / 16];
  kv_move_plane<kMoveChunkBytes>(v, blockIdx.x >> 1, blockIdx.x & 1, blockIdx.y, src_rows, n_keep, first, stage);
}

// Several stages' compactions in one launch: CTA -> (item, plane, kv-head).
__global__ void __launch_bounds__(kMoveThreads) kv_move_multi_kernel(const __grid_constant__ MoveGroup G) {
  pdl_wait();
  pdl_trigger();
  __shared__ __align__(16) uint4 stage[kMoveChunkBytes / 16];
  int it = 0;
  while (it + 1 < G.count && (int)blockIdx.x >= G.m[it + 1].cta0) ++it;
  const MoveItem& M = G.m[it];
  const int local = blockIdx.x - M.cta0;
  const int plane = local / M.kv.heads, head = local % M.kv.heads;
  kv_move_plane<kMoveChunkBytes>(M.kv, plane >> 1, plane & 1, head, M.src, M.n_keep, M.first, stage);
}

// rows [lo, hi) of one plane -> out [rows][heads][row bytes] (debug / test reads)
__global__ void kv_read_kernel(const KvView v, int l, int kind, int lo, uint4* __restrict__ out) {
  const int row = lo + blockIdx.x, head = blockIdx.y;
  const int vec_per_row = v.row_bytes / 16;
  uint4* o = out + ((size_t)blockIdx.x * v.heads + head) * vec_per_row;
  for (int e = threadIdx.x; e < vec_per_row; e += blockDim.x)
    o[e] = *reinterpret_cast<const uint4*>(kv_chunk(v, l, kind, head, row, e));
}

int kv_read_rows(const tp_stage* s, int layer, int kind, int lo, int hi, void* d_out, cudaStream_t st) {
  if (hi <= lo) return TP_OK;
  kv_read_kernel<<<dim3(hi - lo, s->kv_heads), 128, 0, st>>>(kv_view(s), layer - s->lo, kind, lo,
                                                               static_cast<uint4*>(d_out));
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

int kv_compact_many(const MoveGroup& g, int ctas, cudaStream_t st) {
  if (ctas == 0) return TP_OK;
  ::tp::count_launch();
  TP_CUDA(launch_pdl(kv_move_multi_kernel, dim3(ctas), dim3(kMoveThreads), 0, st, g));
  return TP_OK;
}

// Several row gathers in one launch: block (row, item).
__global__ void rows_gather_multi_kernel(const __grid_constant__ RowsGroup G) {
  pdl_wait();
  pdl_trigger();
  const int it = blockIdx.y, r = blockIdx.x;
  if (r >= G.m[it].n_out) return;
  const int rb = G.row_bytes;
  const uint4* s = reinterpret_cast<const uint4*>((const char*)G.m[it].src + (int64_t)G.m[it].idx[r] * rb);
  uint4* d = reinterpret_cast<uint4*>((char*)G.m[it].dst + (int64_t)r * rb);
  for (int e = threadIdx.x; e < rb / 16; e += blockDim.x) d[e] = s[e];
}

int rows_compact_many(const RowsGroup& g, int max_rows, cudaStream_t st) {
  if (g.count == 0 || max_rows == 0) return TP_OK;
  TP_CHECK(g.row_bytes % 16 == 0, TP_ESHAPE, "row bytes must be a multiple of 16");
  ::tp::count_launch();
  TP_CUDA(launch_pdl(rows_gather_multi_kernel, dim3(max_rows, g.count), dim3(256), 0, st, g));
  return TP_OK;
}

int kv_compact(tp_stage* s, const int32_t* d_src_rows, int n_keep, int first, cudaStream_t st) {
  const int nl = s->hi - s->lo;
  const KvView v = kv_view(s);
  TP_CHECK(v.row_bytes % 16 == 0, TP_ESHAPE, "KV row bytes must be a multiple of 16");
  TP_CHECK(v.row_bytes <= kMoveChunkBytes, TP_ESHAPE, "KV row too large for the compaction kernel");
  if (n_keep == 0 || nl == 0) return TP_OK;
  ::tp::count_launch();
  TP_CUDA(launch_pdl(kv_move_kernel, dim3(2 * nl, s->kv_heads), dim3(kMoveThreads), 0, st, v, d_src_rows, n_keep,
                     first));
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

__global__ void rows_gather_kernel(const char* __restrict__ src, char* __restrict__ dst, int row_bytes,
                                   const int32_t* __restrict__ idx) {
  pdl_wait();
  pdl_trigger();
  const uint4* s = reinterpret_cast<const uint4*>(src + (int64_t)idx[blockIdx.x] * row_bytes);
  uint4* d = reinterpret_cast<uint4*>(dst + (int64_t)blockIdx.x * row_bytes);
  for (int e = threadIdx.x; e < row_bytes / 16; e += blockDim.x) d[e] = s[e];
}

int rows_compact(const void* src, void* dst, int64_t row_bytes, const int32_t* d_idx, int n_out,
                 cudaStream_t st) {
  TP_CHECK(row_bytes % 16 == 0, TP_ESHAPE, "row bytes must be a multiple of 16");
  if (n_out == 0) return TP_OK;
  ::tp::count_launch();
  TP_CUDA(launch_pdl(rows_gather_kernel, dim3(n_out), dim3(256), 0, st, (const char*)src, (char*)dst, (int)row_bytes,
                     d_idx));
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

template <typename T>
__device__ __forceinline__ bool better(T a, int ia, T b, int ib) {
  bool na = a != a, nb = b != b;  // NaN ranks highest, first NaN wins
  if (na || nb) return na && (!nb || ia < ib);
  return a > b || (a == b && ia < ib);
}

// Per-thread best of a row: 16 independent loads per round trip (`better` is a
// strict total order, so the visiting order cannot change the winner).
template <typename T>
__device__ __forceinline__ void scan_best(const T* __restrict__ row, int V, T& best, int& bi) {
  constexpr int U = 16;
  for (int base = threadIdx.x; base < V; base += blockDim.x * U) {
    T xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = base + u * (int)blockDim.x;
      xv[u] = v < V ? row[v] : row[0];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int v = base + u * (int)blockDim.x;
      if (v < V && better(xv[u], v, best, bi)) {
        best = xv[u];
        bi = v;
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(1024) argmax_match_kernel(const T* __restrict__ logits, int V,
                                                            const int32_t* __restrict__ children,
                                                            int n_children, int32_t* __restrict__ result) {
  pdl_wait();
  pdl_trigger();
  __shared__ T sv[32];
  __shared__ int si[32];
  __shared__ int s_ib, s_child;
  // the candidate children, one per thread, loaded alongside the scan (not in a serial loop at the end)
  const int my_child = (int)threadIdx.x < n_children ? children[threadIdx.x] : -1;
  T best = logits[0];
  int bi = 0;
  scan_best(logits, V, best, bi);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T ov = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(ov, oi, best, bi)) {
      best = ov;
      bi = oi;
    }
  }
  int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sv[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    T b = sv[0];
    int ib = si[0];
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (better(sv[k], si[k], b, ib)) {
        b = sv[k];
        ib = si[k];
      }
    s_ib = ib;
    s_child = 0x7fffffff;
  }
  __syncthreads();
  const int ib = s_ib;
  if (my_child == ib) atomicMin(&s_child, (int)threadIdx.x);  // first matching child (BFS order)
  for (int c = threadIdx.x + blockDim.x; c < n_children; c += blockDim.x)
    if (children[c] == ib) atomicMin(&s_child, c);
  __syncthreads();
  if (threadIdx.x == 0) {
    result[0] = ib;
    result[1] = s_child == 0x7fffffff ? -1 : s_child;
  }
}

int argmax_match(const void* logits, int is_f64, int vocab, const int32_t* d_children, int n_children,
                 int32_t* d_result, cudaStream_t st) {
  ::tp::count_launch();
  if (is_f64)
    TP_CUDA(launch_pdl(argmax_match_kernel<double>, dim3(1), dim3(1024), 0, st, (const double*)logits, vocab, d_children,
                       n_children, d_result));
  else
    TP_CUDA(launch_pdl(argmax_match_kernel<float>, dim3(1), dim3(1024), 0, st, (const float*)logits, vocab, d_children,
                       n_children, d_result));
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

// One CTA per row: first argmax (lowest id wins ties) of n rows of fp32 logits.
__global__ void __launch_bounds__(1024) argmax_rows_kernel(const float* __restrict__ logits, int V,
                                                           int32_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sv[32];
  __shared__ int si[32];
  const float* row = logits + (size_t)blockIdx.x * V;
  float best = row[0];
  int bi = 0;
  scan_best(row, V, best, bi);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(ov, oi, best, bi)) {
      best = ov;
      bi = oi;
    }
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sv[w] = best;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float b = sv[0];
    int ib = si[0];
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (better(sv[k], si[k], b, ib)) {
        b = sv[k];
        ib = si[k];
      }
    out[blockIdx.x] = ib;
  }
}

int argmax_rows(const void* logits_f32, int vocab, int n, int32_t* d_out, cudaStream_t st) {
  ::tp::count_launch();
  TP_CUDA(launch_pdl(argmax_rows_kernel, dim3(n), dim3(1024), 0, st, (const float*)logits_f32, vocab, d_out));
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

}  // namespace tp

namespace tp {

// Top-K of n rows of fp32 logits (the draft model's proposal candidates): one CTA
// of 32 warps per row.  Each warp keeps its K best (value desc, lowest id first on
// ties, `better`) as a sorted list spread over its lanes (lane r = rank r) and
// scans coalesced batches of 32 logits: a batch costs one compare + ballot against
// the list's K-th entry, and the rare candidates are inserted by a ballot rank +
// shfl_up shift.  The warps' lists are then merged pairwise (5 levels).
__device__ __forceinline__ void topk_insert(float& lv, int& li, float cv, int ci, int K, int lane) {
  const unsigned ahead = __ballot_sync(0xffffffffu, lane < K && better(lv, li, cv, ci));
  const int p = __popc(ahead);
  const float pv = __shfl_up_sync(0xffffffffu, lv, 1);
  const int pi = __shfl_up_sync(0xffffffffu, li, 1);
  if (p < K) {
    if (lane == p) {
      lv = cv;
      li = ci;
    } else if (lane > p && lane < K) {
      lv = pv;
      li = pi;
    }
  }
}

// Merge two descending K-lists (K <= 16) held by one warp: lanes 0-15 its own
// list, lanes 16-31 the partner's reversed (a bitonic sequence of 32); five
// compare-exchange steps leave the best 16 in lanes 0-15, descending.
__device__ __forceinline__ void topk_bitonic16(float& lv, int& li, float pv, int pi, int lane) {
  if (lane >= 16) {
    lv = pv;
    li = pi;
  }
#pragma unroll
  for (int st = 16; st >= 1; st >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, lv, st);
    const int oi = __shfl_xor_sync(0xffffffffu, li, st);
    const bool lower = (lane & st) == 0;
    const bool other_better = better(ov, oi, lv, li);
    if (lower == other_better) {
      lv = ov;
      li = oi;
    }
  }
}

template <int K>
__global__ void __launch_bounds__(1024) topk_rows_kernel(const float* __restrict__ logits, int V, int k,
                                                         int32_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  constexpr int W = 32, U = 8;  // warps; batches loaded per round trip
  __shared__ float sv[W][32];
  __shared__ int si[W][32];
  __shared__ float smax[W];
  const float* row = logits + (size_t)blockIdx.x * V;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float lv = -INFINITY;
  int li = 0x7fffffff;
  // A lower bound T on the row's K-th value: the K-th largest of the 32 warps'
  // first-batch maxima (K distinct row elements are >= it).  Elements below T
  // are never candidates, which keeps the insertions per warp to a few.
  float T = -INFINITY;
  {
    const int j = w * 32 + lane;
    const float x = j < V ? __ldg(row + j) : -INFINITY;
    float m = x != x ? INFINITY : x;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) smax[w] = m;
    __syncthreads();
    if (V >= W * 32) {
      const float mine = smax[lane];
      int above = 0;
      for (int q = 0; q < W; ++q) above += smax[q] > mine || (smax[q] == mine && q < lane);
      const unsigned sel = __ballot_sync(0xffffffffu, above == K - 1);
      T = __shfl_sync(0xffffffffu, mine, __ffs(sel) - 1);
    }
  }
  // candidates: !(x < thr) — NaN, ties and larger values; topk_insert then
  // applies the exact order (a tie or a stale threshold only costs a no-op insert)
  float thr = T;
  for (int base0 = w * 32; base0 < V; base0 += U * W * 32) {
    float xs[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = base0 + u * W * 32 + lane;
      xs[u] = j < V ? __ldg(row + j) : -INFINITY;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = base0 + u * W * 32 + lane;
      const float x = xs[u];
      unsigned m = __ballot_sync(0xffffffffu, !(x < thr) && j < V);
      if (m) {
        do {
          const int src = __ffs(m) - 1;
          m &= m - 1;
          const float cv = __shfl_sync(0xffffffffu, x, src);
          const int ci = __shfl_sync(0xffffffffu, j, src);
          topk_insert(lv, li, cv, ci, K, lane);
        } while (m);
        const float kth = __shfl_sync(0xffffffffu, lv, K - 1);
        thr = kth != kth ? kth : fmaxf(T, kth);  // a NaN K-th entry: every element stays a candidate
      }
    }
  }
  // tree merge: at each level warp w < half takes in warp w + half's list
  for (int half = W / 2; half >= 1; half >>= 1) {
    if (w >= half && w < 2 * half) {
      sv[w][lane] = lv;
      si[w][lane] = li;
    }
    __syncthreads();
    if (w < half) {
      if (K <= 16) {
        topk_bitonic16(lv, li, sv[w + half][31 - lane], si[w + half][31 - lane], lane);
        if (lane >= K) {
          lv = -INFINITY;
          li = 0x7fffffff;
        }
      } else {
        for (int r = 0; r < K; ++r) {
          const float cv = sv[w + half][r];
          const int ci = si[w + half][r];
          if (ci == 0x7fffffff) break;  // the partner's list is shorter
          topk_insert(lv, li, cv, ci, K, lane);
        }
      }
    }
    __syncthreads();
  }
  if (w == 0 && lane < k) out[(size_t)blockIdx.x * k + lane] = li;
}

int topk_rows(const float* logits, int vocab, int n, int k, int32_t* d_out, cudaStream_t st) {
  TP_CHECK(n >= 1 && k >= 1 && k <= 32 && k <= vocab, TP_ESHAPE, "top-k: need 1 <= k <= min(32, vocab)");
  ::tp::count_launch();
  if (k <= 4)
    TP_CUDA(launch_pdl(topk_rows_kernel<4>, dim3(n), dim3(1024), 0, st, logits, vocab, k, d_out));
  else if (k <= 8)
    TP_CUDA(launch_pdl(topk_rows_kernel<8>, dim3(n), dim3(1024), 0, st, logits, vocab, k, d_out));
  else if (k <= 16)
    TP_CUDA(launch_pdl(topk_rows_kernel<16>, dim3(n), dim3(1024), 0, st, logits, vocab, k, d_out));
  else
    TP_CUDA(launch_pdl(topk_rows_kernel<32>, dim3(n), dim3(1024), 0, st, logits, vocab, k, d_out));
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

}  // namespace tp

// Draft-model proposals: the k best token ids of each of n logit rows (fp32, device).
extern "C" int tp_topk_rows(int32_t device, const void* logits_dev, int32_t vocab, int32_t n_rows, int32_t k,
                            void* out_dev, void* stream) {
  TP_CUDA(cudaSetDevice(device));
  return tp::topk_rows(static_cast<const float*>(logits_dev), vocab, n_rows, k, static_cast<int32_t*>(out_dev),
                       (cudaStream_t)stream);
}
