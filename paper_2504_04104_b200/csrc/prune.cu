// K3, device-driven: pruning propagation from the DEVICE-resident verification
// result (reference `pipeline.py:333-400`, `model.py:169-194`).
//
// K4 (tp_model_verify_async) leaves the greedy token tau in the verify stage's
// result word.  Without any host round trip:
//   prune_plan_kernel  one CTA per stage: finds the first level-1 child carrying
//                      tau (pipeline.py:333-339) from the uploaded level-1 tokens,
//                      then evaluates, per speculative cache row (tree node j, I2)
//                      keep = hit ? row(c)[j] | col(c)[j] : j == root (flush keeps the
//                      promoted root), and per in-flight hidden row of the stage's
//                      resident level keep = hit & col(c)[j] — bit tests on the
//                      packed tree rows — and turns each mask into a stable source
//                      list with a ballot + warp prefix sum (warp totals scanned in
//                      shared memory);
//   prune_move_kernel  moves the kept K/V rows of every layer / kv-head plane down
//                      behind the prefix (kept rows only move to lower rows, chunks
//                      staged in shared memory) and gathers the surviving hidden
//                      rows into the next stage's input buffer (hidden_src may be a
//                      peer device's buffer: the receiver-side compaction of the
//                      send-before-verify hand-off).
// The host reads tau only for its own tree update, after both are enqueued.
#include <mutex>
#include <set>
#include <utility>

#include "internal.h"

namespace tp {

constexpr int kPrunePlanThreads = 1024;
constexpr int kPruneMax = 16;  // stages per launch
constexpr int kPruneMoveThreads = 256;
constexpr int kPruneChunkBytes = 32 * 1024;

struct PruneItem {
  KvView kv;              // the stage's K/V storage (paged Llama cache or flat toy planes)
  int layers;
  int P, S, off;          // prefix rows, speculative rows = tree nodes [off, off + S)
  int lvl_lo, lvl_n;      // in-flight level
  const char* hsrc;
  char* hdst;
  int32_t* plan;          // device scratch: [0] kept spec rows, [1] kept hidden rows, [2..2+S) src rows, then hidden idx
  int32_t* keep_out;      // optional copy of the plan (tests)
  int cta_kv, cta_h;      // first CTA of this item in the move launch
};

struct PruneGroup {
  PruneItem m[kPruneMax];
  int count;
  int words, n1;
  const int32_t* verify;    // [0] = tau
  const uint64_t* bits;     // tree rows [tree_n][words]
  const int32_t* lvl1_tok;  // level-1 tokens (tree nodes 1 .. n1)
  int64_t hrow_bytes;
};

__device__ __forceinline__ bool bit_at(const uint64_t* __restrict__ bits, int words, int row, int col) {
  return (bits[(size_t)row * words + (col >> 6)] >> (col & 63)) & 1ull;
}

// Block-wide stable compaction of flags over [0, n): out[k] = base + index of the
// k-th set flag; returns the count.  n may exceed the block (strided passes).
template <typename Pred>
__device__ int block_compact(int n, Pred pred, int base, int32_t* __restrict__ out, int* warp_tot, int* carry) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) *carry = 0;
  __syncthreads();
  for (int r0 = 0; r0 < n; r0 += blockDim.x) {
    const int r = r0 + threadIdx.x;
    const bool k = r < n && pred(r);
    const unsigned bal = __ballot_sync(0xffffffffu, k);
    if (lane == 0) warp_tot[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the warp totals
      int t = lane < nw ? warp_tot[lane] : 0;
      int incl = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane < nw) warp_tot[lane] = incl - t;
      if (lane == 31) warp_tot[32] = incl;  // pass total
    }
    __syncthreads();
    if (k) out[*carry + warp_tot[warp] + __popc(bal & ((1u << lane) - 1u))] = base + r;
    __syncthreads();
    if (threadIdx.x == 0) *carry += warp_tot[32];
    __syncthreads();
  }
  return *carry;
}

__global__ void __launch_bounds__(kPrunePlanThreads) prune_plan_kernel(const __grid_constant__ PruneGroup G) {
  pdl_wait();
  pdl_trigger();
  __shared__ int warp_tot[33];
  __shared__ int carry, s_child;
  const PruneItem& M = G.m[blockIdx.x];
  const int tau = G.verify[0];
  if (threadIdx.x == 0) s_child = 0x7fffffff;
  __syncthreads();
  for (int i = threadIdx.x; i < G.n1; i += blockDim.x)
    if (G.lvl1_tok[i] == tau) atomicMin(&s_child, i);  // first matching child (BFS order)
  __syncthreads();
  const bool hit = s_child != 0x7fffffff;
  const int c = hit ? 1 + s_child : -1;  // tree index (level 1 starts right after the root)
  const uint64_t* bits = G.bits;
  const int words = G.words;
  const int ns = block_compact(
      M.S,
      [&](int r) {
        const int j = M.off + r;
        return hit ? (bit_at(bits, words, c, j) || bit_at(bits, words, j, c)) : j == 0;
      },
      M.P, M.plan + 2, warp_tot, &carry);
  const int nh = block_compact(
      M.lvl_n, [&](int i) { return hit && bit_at(bits, words, M.lvl_lo + i, c); }, 0, M.plan + 2 + M.S, warp_tot,
      &carry);
  if (threadIdx.x == 0) {
    M.plan[0] = ns;
    M.plan[1] = nh;
  }
  if (M.keep_out) {
    __syncthreads();
    for (int i = threadIdx.x; i < 2 + M.S + M.lvl_n; i += blockDim.x) M.keep_out[i] = M.plan[i];
  }
}

__global__ void __launch_bounds__(kPruneMoveThreads) prune_move_kernel(const __grid_constant__ PruneGroup G) {
  pdl_wait();
  pdl_trigger();
  __shared__ __align__(16) uint4 stage[kPruneChunkBytes / 16];
  int it = 0;
  while (it + 1 < G.count && (int)blockIdx.x >= G.m[it + 1].cta_kv) ++it;
  const PruneItem& M = G.m[it];
  const int local = blockIdx.x - M.cta_kv;
  const int n_kv = 2 * M.layers * M.kv.heads;
  if (local >= n_kv) {  // hidden-row gather: one CTA per possible survivor
    const int r = local - n_kv;
    if (r >= M.plan[1]) return;
    const int src = M.plan[2 + M.S + r];
    const uint4* s = reinterpret_cast<const uint4*>(M.hsrc + (int64_t)src * G.hrow_bytes);
    uint4* d = reinterpret_cast<uint4*>(M.hdst + (int64_t)r * G.hrow_bytes);
    for (int e = threadIdx.x; e < G.hrow_bytes / 16; e += blockDim.x) d[e] = s[e];
    return;
  }
  const int plane = local / M.kv.heads, head = local % M.kv.heads;
  kv_move_plane<kPruneChunkBytes>(M.kv, plane >> 1, plane & 1, head, M.plan + 2, M.plan[0], M.P, stage);
}

}  // namespace tp

using namespace tp;

extern "C" int tp_prune_device(int32_t count, const tp_prune_stage* stages, const tp_stage* verify_ws,
                               const uint64_t* tree_bits, int32_t tree_n, int32_t words, const int32_t* level1_tokens,
                               int32_t n_level1, int64_t hidden_row_bytes, void* stream) {
  TP_CHECK(count >= 0 && (count == 0 || stages) && verify_ws, TP_ECONFIG, "null argument");
  if (count == 0) return TP_OK;
  TP_CHECK(tree_n >= 1 && words >= (tree_n + 63) / 64 && tree_bits, TP_ESHAPE, "tree rows missing or too narrow");
  TP_CHECK(n_level1 >= 0 && n_level1 < tree_n && (n_level1 == 0 || level1_tokens), TP_ESHAPE, "bad level 1");
  TP_CHECK(hidden_row_bytes % 16 == 0, TP_ESHAPE, "hidden row bytes must be a multiple of 16");
  tp_model* m0 = verify_ws->m;  // the device of this call (stage-less entries: hand-off receivers)
  TP_CUDA(cudaSetDevice(m0->cfg.device));
  cudaStream_t st = (cudaStream_t)stream;
  // per-model plan scratch (device), grown on demand
  auto* ext = reinterpret_cast<int32_t**>(&m0->prune_plan);
  size_t need = 0;
  for (int i = 0; i < count; ++i) {
    const tp_prune_stage& d = stages[i];
    TP_CHECK(!d.stage || d.stage->m->cfg.device == m0->cfg.device, TP_ECONFIG,
             "stages of one prune call share the verification result's device (tp_result_mirror)");
    TP_CHECK(d.stage || (d.prefix_rows == 0 && d.spec_rows == 0), TP_ECONTRACT, "a stage-less entry has no K/V rows");
    TP_CHECK(!d.stage || (d.prefix_rows >= 0 && d.spec_rows >= 0 && d.prefix_rows + d.spec_rows == d.stage->rows),
             TP_ECONTRACT, "prefix + speculative rows must cover the cache (invariant I1)");
    TP_CHECK(d.spec_rows == 0 || (d.tree_off >= 0 && d.tree_off + d.spec_rows <= tree_n), TP_ECONTRACT,
             "speculative rows outside the tree (invariant I2)");
    TP_CHECK(d.level_n == 0 || (d.level_lo >= 0 && d.level_lo + d.level_n <= tree_n && d.hidden_src && d.hidden_dst),
             TP_ECONTRACT, "in-flight level outside the tree");
    TP_CHECK(!d.stage || ((d.stage->head_dim * d.stage->esize) % 16 == 0 &&
                           d.stage->head_dim * d.stage->esize <= kPruneChunkBytes),
             TP_ESHAPE, "KV row size unsupported");
    need += 2 + (size_t)d.spec_rows + d.level_n;
  }
  if (need > m0->prune_plan_ints) {
    if (*ext) {
      TP_CUDA(cudaStreamSynchronize(st));
      cudaFree(*ext);
    }
    m0->prune_plan_ints = std::max<size_t>(need * 2, 4096);
    TP_CUDA(cudaMalloc((void**)ext, m0->prune_plan_ints * 4));
  }
  int32_t* plan = *ext;
  // tree rows + level-1 tokens: one upload through the model's call ring
  const size_t bits_bytes = (size_t)tree_n * words * 8;
  const size_t tok_bytes = ((size_t)n_level1 * 4 + 15) & ~(size_t)15;
  char *h, *dm;
  int slot;
  TP_TRY(call_slot(m0, bits_bytes + tok_bytes, &h, &dm, &slot));
  std::memcpy(h, tree_bits, bits_bytes);
  if (n_level1) std::memcpy(h + bits_bytes, level1_tokens, 4 * (size_t)n_level1);
  TP_TRY(call_push(m0, slot, bits_bytes + tok_bytes, st));
  for (int c0 = 0; c0 < count; c0 += kPruneMax) {
    const int c1 = std::min(count, c0 + kPruneMax);
    PruneGroup g;
    g.count = c1 - c0;
    g.words = words;
    g.n1 = n_level1;
    g.verify = verify_ws->d_result;
    g.bits = reinterpret_cast<const uint64_t*>(dm);
    g.lvl1_tok = reinterpret_cast<const int32_t*>(dm + bits_bytes);
    g.hrow_bytes = hidden_row_bytes;
    int ctas = 0;
    for (int i = c0; i < c1; ++i) {
      const tp_prune_stage& d = stages[i];
      tp_stage* s = d.stage;
      PruneItem& it = g.m[i - c0];
      it.kv = s ? kv_view(s) : KvView{};
      it.kv.heads = s ? it.kv.heads : 1;
      it.layers = s ? s->hi - s->lo : 0;
      it.P = d.prefix_rows;
      it.S = d.spec_rows;
      it.off = d.tree_off;
      it.lvl_lo = d.level_lo;
      it.lvl_n = d.level_n;
      it.hsrc = static_cast<const char*>(d.hidden_src);
      it.hdst = static_cast<char*>(d.hidden_dst);
      it.plan = plan;
      it.keep_out = d.keep_out;
      plan += 2 + d.spec_rows + d.level_n;
      it.cta_kv = ctas;
      ctas += 2 * it.layers * it.kv.heads + d.level_n;
      it.cta_h = ctas - d.level_n;
    }
    ::tp::count_launch();
    TP_CUDA(launch_pdl(prune_plan_kernel, dim3(g.count), dim3(kPrunePlanThreads), 0, st, g));
    if (ctas) {
      ::tp::count_launch();
      TP_CUDA(launch_pdl(prune_move_kernel, dim3(ctas), dim3(kPruneMoveThreads), 0, st, g));
    }
    TP_CUDA(cudaGetLastError());
  }
  // host-side row bookkeeping of the stages is the caller's (it knows tau after
  // tp_model_verify_wait); the device rows are final once the move kernel ran
  timeline_mark("prune_device", st);
  return TP_OK;
}

extern "C" int tp_result_mirror(tp_stage* dst_ws, const tp_stage* src_ws, void* stream) {
  TP_CHECK(dst_ws && src_ws, TP_ECONFIG, "null argument");
  TP_CUDA(cudaSetDevice(dst_ws->m->cfg.device));
  TP_CUDA(cudaMemcpyPeerAsync(dst_ws->d_result, dst_ws->m->cfg.device, src_ws->d_result, src_ws->m->cfg.device, 16,
                              (cudaStream_t)stream));
  timeline_mark("verify_mirror", (cudaStream_t)stream);
  return TP_OK;
}

extern "C" int tp_peer_copy(void* dst, int32_t dst_device, const void* src, int32_t src_device, int64_t bytes,
                            void* stream) {
  TP_CHECK(bytes >= 0 && (bytes == 0 || (dst && src)), TP_ECONFIG, "null argument");
  if (bytes == 0) return TP_OK;
  TP_CUDA(cudaSetDevice(src_device));
  if (dst_device != src_device) {  // NVLink P2P between the two GPUs, enabled once per ordered pair
    static std::mutex mu;
    static std::set<std::pair<int, int>> done;
    std::lock_guard<std::mutex> lk(mu);
    if (done.insert({src_device, dst_device}).second) {
      int can = 0;
      TP_CUDA(cudaDeviceCanAccessPeer(&can, src_device, dst_device));
      if (can) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(dst_device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) TP_CUDA(e);
        cudaGetLastError();  // clear an "already enabled"
      }
    }
  }
  TP_CUDA(cudaMemcpyPeerAsync(dst, dst_device, src, src_device, (size_t)bytes, (cudaStream_t)stream));
  return TP_OK;
}
