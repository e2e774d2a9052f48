// K1: tree-masked attention of a level's nodes against one stage's KV cache
// (Llama path; replaces the gather + softmax + PV of the reference
// layer_step, `/root/reference/pkg/src/treepipe/model.py:157-167,265-276`).
//
// Node i attends its *logical* key sequence of T_i = P_i + A_i + 1 slots: cache
// rows [0, P_i) (verified prefix), its A_i speculative ancestors in row order
// (the set bits of its packed ancestor row), then itself (self last).  The
// sequence is split at a fixed distance from its end:
//
//   * chunked part, slots [0, T_i - W) (W = kSuffix = 16): with A_i < W these
//     are prefix rows only — cache row = slot — so every node of a tree level
//     shares them.  Cut into canonical 64-slot chunks (chunk c = slots
//     [64c, 64c + 64), the last one partial) and runs of kRun chunks.  A chunk
//     yields a partial (max, sum, unnormalised P.V) from one m16n8k16 bf16
//     tensor-core pass over a padded shared-memory tile; a run's state is the
//     in-order merge of its chunks from the empty state.
//       attn_chunks_kernel  one CTA per (member, KV head, run, block of 64
//                           (query head, node) rows): the run's K/V chunks are
//                           staged ONCE for all rows by bulk TMA copies
//                           (cp.async.bulk, one per 256-byte row, mbarrier
//                           completion, double buffered) and the run states
//                           written; members with few rows take the run's
//                           chunks in parallel across warps instead.
//   * suffix, the last W slots (prefix tail, ancestors, self): node-specific.
//       attn_tail_kernel    one warp per (node, query head): decodes the
//                           node's ancestor rows from its packed bit-row in
//                           registers (word popcounts + a warp scan, then
//                           the rank-th set bit), computes the suffix partial
//                           on the FMA pipes in a fixed order (lane l owns
//                           dims 4l..4l+3, dot products by a butterfly sum),
//                           merges the run states in order and the suffix
//                           last, and writes the bf16 output row.  The suffix
//                           is computed before griddepcontrol.wait, while the
//                           chunk kernel still runs.
//
// Batch invariance: every boundary above depends only on T_i, which is the
// node's position + 1 whether it sits in a tree level or is decoded alone, and
// a chunk partial depends only on the node's query and the chunk's key rows
// (tensor-core rows and columns are independent; merges use explicitly
// rounded ops).  A node computed inside a 64-node tree level is therefore
// bit-identical to the same position decoded alone (GPU pipeline == GPU greedy
// decode), whatever its launch-mates.
#include <cstdlib>
#include <type_traits>

#include "attn.h"
#include "gemm_tc.h"
#include "sm100.cuh"

namespace tp {

constexpr int kPad = 136;  // bf16 per staged row: 128 + 8 pad (conflict-free ldmatrix)
constexpr int kWarps = 4;
constexpr int kTileElems = kAttnChunk * kPad;
constexpr int kRowBytes = kAttnHeadDim * 2;

__device__ __forceinline__ uint32_t ld_b32(const __nv_bfloat16* p) {
  return *reinterpret_cast<const uint32_t*>(p);
}
__device__ __forceinline__ uint32_t pack_bf16(__nv_bfloat16 lo, __nv_bfloat16 hi) {
  return (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
}
__device__ __forceinline__ uint32_t pack_f32(float lo, float hi) {
  return pack_bf16(__float2bfloat16_rn(lo), __float2bfloat16_rn(hi));
}
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// exp(x) as one MUFU op: 2^(x*log2 e) with ex2.approx (flush-to-zero; every
// attention path — shared chunks, per-node tail, tile, merges — uses this same
// function, so batch invariance is unaffected).
__device__ __forceinline__ float fast_exp(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(__fmul_rn(x, 1.4426950408889634f)));
  return y;
}
__device__ __forceinline__ void mma16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// 16-byte async copy global -> shared; src_bytes = 0 writes zeros.
__device__ __forceinline__ void cp16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// wait until at most `ahead` (0..3) committed groups are still pending
__device__ __forceinline__ void cp_wait_ahead(int ahead) {
  switch (ahead) {
    case 0: cp_wait_group<0>(); break;
    case 1: cp_wait_group<1>(); break;
    case 2: cp_wait_group<2>(); break;
    default: cp_wait_group<3>(); break;
  }
}

__device__ __forceinline__ void ldsm4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm4t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

// Scores + chunk softmax of one canonical 64-slot chunk for the 16-row tile
// this warp holds, K staged in sK[slot][kPad]:
//   qa   : Q A-fragments (8 k-steps over head_dim)
//   lim  : rows g / g+8 see slots [0, lim) of this chunk
// Returns the chunk max m, sum l and the bf16 P A-fragments.
// Raw scores s = Q.K^T of one 64-slot chunk for the warp's 16-row tile, K
// staged in sK[slot][kPad].
__device__ __forceinline__ void tile_qk(const uint32_t (&qa)[8][4], const __nv_bfloat16* sK, float (&s)[8][4],
                                        int lane) {
  const int mi = lane >> 3, mr = lane & 7;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
      uint32_t b[4];  // b0/b1 of k-steps 2*k2 and 2*k2+1
      ldsm4(su32(sK + (nt * 8 + mr) * kPad + 32 * k2 + 8 * mi), b);
      mma16816(s[nt], qa[2 * k2], b[0], b[1]);
      mma16816(s[nt], qa[2 * k2 + 1], b[2], b[3]);
    }
  }
}

// Chunk softmax of the raw scores: rows g / g+8 see slots [0, lim); returns the
// chunk max m, sum l and the bf16 P A-fragments.
__device__ __forceinline__ void chunk_softmax(float (&s)[8][4], const int (&lim)[2], float scale, float (&m)[2],
                                              float (&l)[2], uint32_t (&pa)[4][4], int lane) {
  const int tig = lane & 3;
  float mc[2] = {-INFINITY, -INFINITY};
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int slot = nt * 8 + 2 * tig + (e & 1);
      const float v = slot < lim[e >> 1] ? __fmul_rn(s[nt][e], scale) : -INFINITY;
      s[nt][e] = v;
      mc[e >> 1] = fmaxf(mc[e >> 1], v);
    }
  float rs[2] = {0.f, 0.f};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    mc[h] = fmaxf(mc[h], __shfl_xor_sync(0xffffffffu, mc[h], 1));
    mc[h] = fmaxf(mc[h], __shfl_xor_sync(0xffffffffu, mc[h], 2));
  }
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int h = e >> 1;
      const float p = s[nt][e] == -INFINITY ? 0.f : fast_exp(__fsub_rn(s[nt][e], mc[h]));
      s[nt][e] = p;
      rs[h] = __fadd_rn(rs[h], p);
    }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    rs[h] = __fadd_rn(rs[h], __shfl_xor_sync(0xffffffffu, rs[h], 1));
    rs[h] = __fadd_rn(rs[h], __shfl_xor_sync(0xffffffffu, rs[h], 2));
    l[h] = rs[h];
    m[h] = mc[h];
  }
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    pa[kk][0] = pack_f32(s[2 * kk][0], s[2 * kk][1]);
    pa[kk][1] = pack_f32(s[2 * kk][2], s[2 * kk][3]);
    pa[kk][2] = pack_f32(s[2 * kk + 1][0], s[2 * kk + 1][1]);
    pa[kk][3] = pack_f32(s[2 * kk + 1][2], s[2 * kk + 1][3]);
  }
}

__device__ __forceinline__ void chunk_scores(const uint32_t (&qa)[8][4], const __nv_bfloat16* sK,
                                             const int (&lim)[2], float scale, float (&m)[2], float (&l)[2],
                                             uint32_t (&pa)[4][4], int lane) {
  float s[8][4];
  tile_qk(qa, sK, s, lane);
  chunk_softmax(s, lim, scale, m, l, pa, lane);
}

// Online merge of a chunk partial (mc, lc, oc) into the running (M, L, O).
__device__ __forceinline__ void merge_scale(float& M, float& L, float mc, float lc, float& sa, float& sb) {
  const float mn = fmaxf(M, mc);
  sa = M == -INFINITY ? 0.f : fast_exp(__fsub_rn(M, mn));
  sb = fast_exp(__fsub_rn(mc, mn));
  L = __fmaf_rn(L, sa, __fmul_rn(lc, sb));
  M = mn;
}
__device__ __forceinline__ float merge_val(float O, float oc, float sa, float sb) {
  return __fmaf_rn(O, sa, __fmul_rn(oc, sb));
}

__device__ __forceinline__ size_t part_idx(const AttnArgs& a, int node, int h, int c) {
  return ((size_t)node * a.H + h) * a.max_chunks + c;
}

// kind: 0 shared, 1 per-node tail, 2 GQA tail
__device__ __forceinline__ int member_of(const AttnGroup& G, int b, int kind) {
  auto start = [&](int g) { return kind == 0 ? G.m[g].cta_shared : kind == 1 ? G.m[g].cta_tail : G.m[g].cta_gqa; };
  int gi = 0;
  while (gi + 1 < G.count && b >= start(gi + 1)) ++gi;
  return gi;
}

// o = P . V over the dims [128 / NP * PART, 128 / NP * (PART + 1)) — n-tiles of
// the full P . V in the same k order (the same MMAs per output element), with
// 1/NP of the accumulators live.
template <int PART, int NP>
__device__ __forceinline__ void chunk_pv_part(const uint32_t (&pa)[4][4], const __nv_bfloat16* sV,
                                              float (&o)[16 / NP][4], int lane) {
  const int mi = lane >> 3, mr = lane & 7;
#pragma unroll
  for (int nd = 0; nd < 16 / NP; ++nd) o[nd][0] = o[nd][1] = o[nd][2] = o[nd][3] = 0.f;
#pragma unroll
  for (int n2l = 0; n2l < 8 / NP; ++n2l)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int n2 = (8 / NP) * PART + n2l;
      uint32_t b[4];
      ldsm4t(su32(sV + (16 * kk + 8 * (mi & 1) + mr) * kPad + 16 * n2 + 8 * (mi >> 1)), b);
      mma16816(o[2 * n2l], pa[kk], b[0], b[1]);
      mma16816(o[2 * n2l + 1], pa[kk], b[2], b[3]);
    }
}
template <int HALF>
__device__ __forceinline__ void chunk_pv_half(const uint32_t (&pa)[4][4], const __nv_bfloat16* sV, float (&o)[8][4],
                                              int lane) {
  chunk_pv_part<HALF, 2>(pa, sV, o, lane);
}

// Merge a partial (mc, lc, oc) into a lane-layout state (M, L, O).
__device__ __forceinline__ void merge_lane(float& M, float& L, float4& O, float mc, float lc, float4 oc) {
  float sa, sb;
  merge_scale(M, L, mc, lc, sa, sb);
  O.x = merge_val(O.x, oc.x, sa, sb);
  O.y = merge_val(O.y, oc.y, sa, sb);
  O.z = merge_val(O.z, oc.z, sa, sb);
  O.w = merge_val(O.w, oc.w, sa, sb);
}


// Canonical chunks per run: a fixed property of the numerics (every launch of a
// process must use the same value for batch invariance); knob 1 for tuning.
static int g_attn_run = 4;
constexpr int kCtaRows = 64;  // (query head, node) rows per chunk CTA: one 16-row MMA tile per warp
constexpr int kSmallRows = 32;
constexpr int kXsLd = 132;  // floats per hand-over row
constexpr size_t kChunksSmem = (size_t)4 * kTileElems * 2 + 64;  // 2 x (K, V) chunk tiles + mbarriers

__device__ __forceinline__ void bulk_row(void* smem_dst, const void* gsrc, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(smem_dst)),
               "l"(gsrc), "r"(kRowBytes), "r"(su32(bar))
               : "memory");
}

// Slots of node i's chunked part (T_i - W, >= 0).
__device__ __forceinline__ int chunked_slots(const LevelDev& lv, int i) {
  return max(0, __ldg(lv.prefix_rows + i) + __ldg(lv.anc_cnt + i) + 1 - kAttnSuffix);
}

// Empty-partial guard of a merge: a row with no slot in the chunk keeps its state.
__device__ __forceinline__ void merge_scale_live(float& M, float& L, float mc, float lc, bool live, float& sa,
                                                 float& sb) {
  if (live) {
    merge_scale(M, L, mc, lc, sa, sb);
  } else {
    sa = 1.f;
    sb = 0.f;
  }
}

// Stage rows [j0, j0 + nrows) of one kv-head plane into a tile by bulk copies
// issued by the calling warp (completion counted on `bar`); with zero_tail the
// rows beyond nrows are zeroed (V of a partial chunk: their P is 0, and
// 0 x stale bits must not be NaN).
__device__ __forceinline__ void stage_rows(const __nv_bfloat16* plane, const AttnArgs& a, int kh, int j0, int nrows,
                                           __nv_bfloat16* tile, uint64_t* bar, bool zero_tail, int lane) {
  const __nv_bfloat16* src = plane + ((size_t)kh * a.cap + (size_t)j0) * kAttnHeadDim;
  // the tile's previous generic-proxy reads / zero stores are ordered before these async-proxy writes
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  for (int r = lane; r < nrows; r += 32) bulk_row(tile + r * kPad, src + (size_t)r * kAttnHeadDim, bar);
  if (zero_tail) {
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    for (int e = nrows * 16 + lane; e < kAttnChunk * 16; e += 32)
      *reinterpret_cast<uint4*>(tile + (e >> 4) * kPad + (e & 15) * 8) = z;
  }
}

// K and V of one chunk into a (K, V) tile pair, one mbarrier phase.
__device__ __forceinline__ void stage_chunk(const AttnArgs& a, int kh, int j0, int nrows, __nv_bfloat16* sK,
                                            __nv_bfloat16* sV, uint64_t* bar, int lane) {
  if (lane == 0) sm100::mbar_expect_tx(bar, (uint32_t)(2 * nrows * kRowBytes));
  __syncwarp();
  stage_rows(a.k, a, kh, j0, nrows, sK, bar, false, lane);
  stage_rows(a.v, a, kh, j0, nrows, sV, bar, true, lane);
}

// Few rows (<= kSmallRows (query head, node) pairs, e.g. the lone verification
// node): one CTA per (member, KV head, run, 16-row tile), warp w computing chunk
// w of the run (run <= kWarps) on its own tile, partials handed over through
// smem and merged in chunk order — the same chunk arithmetic and merge sequence
// as the row-parallel path, the run's chunks in parallel.
__device__ __forceinline__ void chunks_small(const AttnGroup& G, int gi, int local, uint8_t* dsm) {
  const AttnArgs& a = G.m[gi].a;
  const LevelDev& lv = G.m[gi].lv;
  const int c_hi = G.m[gi].c_shared, R = G.run;
  const int runs = (c_hi + R - 1) / R;
  const int kh = local % a.KV;
  local /= a.KV;
  const int r = local % runs, t = local / runs;
  const int grp = a.H / a.KV;
  const int n = lv.n, rows = n * grp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int nw = min(R, c_hi - r * R);
  __nv_bfloat16* buf = reinterpret_cast<__nv_bfloat16*>(dsm) + (size_t)warp * kTileElems;  // K, then V
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<__nv_bfloat16*>(dsm) + (size_t)kWarps * kTileElems);
  float* xs = reinterpret_cast<float*>(buf);  // [16][kXsLd] partial, then 16 max + 16 sum + 16 live
  const int c = r * R + warp;
  const int ra = 16 * t + g, rb = ra + 8;
  const bool va = ra < rows, vb = rb < rows;
  const int ia = va ? ra % n : 0, ib = vb ? rb % n : 0;
  const int ha = kh * grp + (va ? ra / n : 0), hb = kh * grp + (vb ? rb / n : 0);
  const int Ca = va ? chunked_slots(lv, ia) : 0, Cb = vb ? chunked_slots(lv, ib) : 0;
  if (threadIdx.x < kWarps) sm100::mbar_init(bars + threadIdx.x, 1);
  sm100::fence_barrier_init();
  __syncthreads();
  if (warp < nw) {
    const int j0 = c * kAttnChunk;
    const int nrows = min(kAttnChunk, max(0, G.m[gi].max_c - j0));
    if (lane == 0) sm100::mbar_expect_tx(bars + warp, (uint32_t)(nrows * kRowBytes));
    __syncwarp();
    stage_rows(a.k, a, kh, j0, nrows, buf, bars + warp, false, lane);
    uint32_t qa[8][4];
    const __nv_bfloat16* qra = a.q + (size_t)ia * a.q_stride + ha * kAttnHeadDim;
    const __nv_bfloat16* qrb = a.q + (size_t)ib * a.q_stride + hb * kAttnHeadDim;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      qa[kk][0] = va ? ld_b32(qra + 16 * kk + 2 * tig) : 0u;
      qa[kk][1] = vb ? ld_b32(qrb + 16 * kk + 2 * tig) : 0u;
      qa[kk][2] = va ? ld_b32(qra + 16 * kk + 8 + 2 * tig) : 0u;
      qa[kk][3] = vb ? ld_b32(qrb + 16 * kk + 8 + 2 * tig) : 0u;
    }
    const int lim[2] = {min(kAttnChunk, max(0, Ca - j0)), min(kAttnChunk, max(0, Cb - j0))};
    sm100::mbar_wait(bars + warp, 0);
    float m[2], l[2];
    uint32_t pa[4][4];
    chunk_scores(qa, buf, lim, a.scale, m, l, pa, lane);
    __syncwarp();  // every lane is done reading K: the tile takes V
    if (lane == 0) sm100::mbar_expect_tx(bars + warp, (uint32_t)(nrows * kRowBytes));
    __syncwarp();
    stage_rows(a.v, a, kh, j0, nrows, buf, bars + warp, true, lane);
    __syncwarp();
    sm100::mbar_wait(bars + warp, 1);
    float o0[8][4], o1[8][4];
    chunk_pv_half<0>(pa, buf, o0, lane);
    chunk_pv_half<1>(pa, buf, o1, lane);
    __syncwarp();  // the tile becomes the hand-over buffer
#pragma unroll
    for (int nd = 0; nd < 8; ++nd) {
      *reinterpret_cast<float2*>(xs + g * kXsLd + nd * 8 + 2 * tig) = make_float2(o0[nd][0], o0[nd][1]);
      *reinterpret_cast<float2*>(xs + (g + 8) * kXsLd + nd * 8 + 2 * tig) = make_float2(o0[nd][2], o0[nd][3]);
      *reinterpret_cast<float2*>(xs + g * kXsLd + 64 + nd * 8 + 2 * tig) = make_float2(o1[nd][0], o1[nd][1]);
      *reinterpret_cast<float2*>(xs + (g + 8) * kXsLd + 64 + nd * 8 + 2 * tig) = make_float2(o1[nd][2], o1[nd][3]);
    }
    if (tig == 0) {
      xs[16 * kXsLd + g] = m[0];
      xs[16 * kXsLd + g + 8] = m[1];
      xs[16 * kXsLd + 16 + g] = l[0];
      xs[16 * kXsLd + 16 + g + 8] = l[1];
      xs[16 * kXsLd + 32 + g] = lim[0] > 0 ? 1.f : 0.f;
      xs[16 * kXsLd + 32 + g + 8] = lim[1] > 0 ? 1.f : 0.f;
    }
  }
  __syncthreads();
  const int row = threadIdx.x >> 3, d0 = (threadIdx.x & 7) * 16;  // 8 threads per row, 16 dims each
  const int rr = 16 * t + row;
  if (rr >= rows) return;
  float M = -INFINITY, L = 0.f, O[16];
#pragma unroll
  for (int d = 0; d < 16; ++d) O[d] = 0.f;
  for (int w = 0; w < nw; ++w) {
    const float* xw = reinterpret_cast<const float*>(reinterpret_cast<const __nv_bfloat16*>(dsm) +
                                                     (size_t)w * kTileElems);
    float sa, sb;
    merge_scale_live(M, L, xw[16 * kXsLd + row], xw[16 * kXsLd + 16 + row], xw[16 * kXsLd + 32 + row] != 0.f, sa,
                     sb);
#pragma unroll
    for (int d = 0; d < 16; ++d) O[d] = merge_val(O[d], xw[row * kXsLd + d0 + d], sa, sb);
  }
  const size_t idx = part_idx(a, rr % n, kh * grp + rr / n, r);
  float* po = a.po + idx * kAttnHeadDim + d0;
#pragma unroll
  for (int d = 0; d < 16; d += 4) *reinterpret_cast<float4*>(po + d) = make_float4(O[d], O[d + 1], O[d + 2], O[d + 3]);
  if ((threadIdx.x & 7) == 0) {
    a.pm[idx] = M;
    a.pl[idx] = L;
  }
}

// One CTA per (member, KV head, run, block of kCtaRows (query head, node) rows):
// streams the run's chunks (chunk c + 1 in flight by bulk TMA while chunk c
// computes), each K/V chunk staged once for every row, merges them in order
// into the rows' run states (fragment layout, the same scalar merge ops as
// merge_lane) and writes the states.
__global__ void __launch_bounds__(kWarps * 32, 3) attn_chunks_kernel(const __grid_constant__ AttnGroup G) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t dsm[];
  const int gi = member_of(G, blockIdx.x, 0);
  if (G.m[gi].small) {
    chunks_small(G, gi, blockIdx.x - G.m[gi].cta_shared, dsm);
    return;
  }
  const AttnArgs& a = G.m[gi].a;
  const LevelDev& lv = G.m[gi].lv;
  const int c_hi = G.m[gi].c_shared;
  const int kRun = G.run;
  const int runs = (c_hi + kRun - 1) / kRun;
  int local = blockIdx.x - G.m[gi].cta_shared;
  const int kh = local % a.KV;
  local /= a.KV;
  const int r = local % runs, blk = local / runs;
  const int grp = a.H / a.KV;
  const int npc = kCtaRows / grp;  // nodes per CTA
  const int base = blk * npc;
  const int c0 = r * kRun, c1 = min(c_hi, c0 + kRun);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int nreal = min(npc, lv.n - base);
  const int rows = nreal * grp;  // (query head, node) pairs, head-major
  __nv_bfloat16* smt = reinterpret_cast<__nv_bfloat16*>(dsm);  // [2][K | V][kTileElems]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smt + 4 * kTileElems);
  if (threadIdx.x < 2) sm100::mbar_init(bars + threadIdx.x, 1);
  sm100::fence_barrier_init();
  __syncthreads();
  const int max_c = G.m[gi].max_c;
  auto stage = [&](int c, int buf) {  // warp 0 issues; everyone waits on the buffer's mbarrier
    if (warp == 0) {
      __nv_bfloat16* sK = smt + (size_t)buf * 2 * kTileElems;
      stage_chunk(a, kh, c * kAttnChunk, min(kAttnChunk, max(0, max_c - c * kAttnChunk)), sK, sK + kTileElems,
                  bars + buf, lane);
    }
  };
  stage(c0, 0);
  const int ra = 16 * warp + g, rb = ra + 8;
  const bool busy = 16 * warp < rows;
  const bool va = ra < rows, vb = rb < rows;
  const int ia = base + (va ? ra % nreal : 0), ib = base + (vb ? rb % nreal : 0);
  const int ha = kh * grp + (va ? ra / nreal : 0), hb = kh * grp + (vb ? rb / nreal : 0);
  const int Ca = va ? chunked_slots(lv, ia) : 0, Cb = vb ? chunked_slots(lv, ib) : 0;
  uint32_t qa[8][4];
  {
    const __nv_bfloat16* qra = a.q + (size_t)ia * a.q_stride + ha * kAttnHeadDim;
    const __nv_bfloat16* qrb = a.q + (size_t)ib * a.q_stride + hb * kAttnHeadDim;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      qa[kk][0] = va ? ld_b32(qra + 16 * kk + 2 * tig) : 0u;
      qa[kk][1] = vb ? ld_b32(qrb + 16 * kk + 2 * tig) : 0u;
      qa[kk][2] = va ? ld_b32(qra + 16 * kk + 8 + 2 * tig) : 0u;
      qa[kk][3] = vb ? ld_b32(qrb + 16 * kk + 8 + 2 * tig) : 0u;
    }
  }
  float M[2] = {-INFINITY, -INFINITY}, L[2] = {0.f, 0.f};
  float O[16][4];
#pragma unroll
  for (int nd = 0; nd < 16; ++nd) O[nd][0] = O[nd][1] = O[nd][2] = O[nd][3] = 0.f;
  for (int c = c0; c < c1; ++c) {
    const int buf = (c - c0) & 1;
    if (c + 1 < c1) stage(c + 1, buf ^ 1);
#ifdef TP_ATTN_PRINTF
    if (threadIdx.x == 0) printf("blk %d c %d c0 %d c1 %d max_c %d rows %d\n", blockIdx.x, c, c0, c1, max_c, rows);
#endif
    sm100::mbar_wait(bars + buf, ((c - c0) >> 1) & 1);
#ifdef TP_ATTN_PRINTF
    if (threadIdx.x == 0) printf("blk %d c %d waited\n", blockIdx.x, c);
#endif
    __syncthreads();  // the zero-filled V rows of a partial chunk are visible too
    const int j0 = c * kAttnChunk;
    const int lim[2] = {min(kAttnChunk, max(0, Ca - j0)), min(kAttnChunk, max(0, Cb - j0))};
    // warp-uniform: the MMAs and shuffles below need every lane of the warp
    if (busy && __any_sync(0xffffffffu, lim[0] > 0 || lim[1] > 0)) {
      const __nv_bfloat16* sK = smt + (size_t)buf * 2 * kTileElems;
      float m[2], l[2], sa[2], sb[2];
      uint32_t pa[4][4];
      chunk_scores(qa, sK, lim, a.scale, m, l, pa, lane);
      merge_scale_live(M[0], L[0], m[0], l[0], lim[0] > 0, sa[0], sb[0]);
      merge_scale_live(M[1], L[1], m[1], l[1], lim[1] > 0, sa[1], sb[1]);
      auto merge_part = [&](auto part_tag) {  // PV a quarter of the dims at a time, merged at once
        constexpr int PT = decltype(part_tag)::value;
        float o[4][4];
        chunk_pv_part<PT, 4>(pa, sK + kTileElems, o, lane);
#pragma unroll
        for (int nd = 0; nd < 4; ++nd)
#pragma unroll
          for (int e = 0; e < 4; ++e)
            O[4 * PT + nd][e] = merge_val(O[4 * PT + nd][e], o[nd][e], sa[e >> 1], sb[e >> 1]);
      };
      merge_part(std::integral_constant<int, 0>{});
      merge_part(std::integral_constant<int, 1>{});
      merge_part(std::integral_constant<int, 2>{});
      merge_part(std::integral_constant<int, 3>{});
    }
    __syncthreads();  // buffer `buf` is restaged for chunk c + 2
  }
  if (!busy) return;
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    if (!(hh ? vb : va)) continue;
    const size_t idx = part_idx(a, hh ? ib : ia, hh ? hb : ha, r);
    float* po = a.po + idx * kAttnHeadDim;
#pragma unroll
    for (int nd = 0; nd < 16; ++nd)
      *reinterpret_cast<float2*>(po + nd * 8 + 2 * tig) = make_float2(O[nd][2 * hh], O[nd][2 * hh + 1]);
    if (tig == 0) {
      a.pm[idx] = M[hh];
      a.pl[idx] = L[hh];
    }
  }
}

// The cache row of the rank-th (0-based) speculative ancestor of a node: its
// packed ancestor bit-row is walked word by word in registers (popcount to skip
// whole words, __fns for the bit inside the word) — no host-side decode.
__device__ __forceinline__ int ancestor_row(const uint64_t* __restrict__ bits, int rank, int bits_base) {
  for (int w = 0;; ++w) {
    const uint64_t x = __ldg(bits + w);
    const int pc = __popcll(x);
    if (rank < pc) {
      const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
      const int plo = __popc(lo);
      const int bit = rank < plo ? (int)__fns(lo, 0, rank + 1) : 32 + (int)__fns(hi, 0, rank - plo + 1);
      return bits_base + 64 * w + bit;
    }
    rank -= pc;
  }
}

// One warp per (node, query head): suffix partial of the last kSuffix slots on the
// FMA pipes (before griddepcontrol.wait when `early`), then the ordered merge of
// the chunk kernel's run states, the suffix last, and the bf16 output row.
__global__ void __launch_bounds__(kWarps * 32) attn_tail_kernel(const __grid_constant__ AttnGroup G, int early) {
  if (!early) pdl_wait();
  pdl_trigger();  // the O-projection GEMM may start streaming its weights
  const int gi = member_of(G, blockIdx.x, 1);
  const AttnArgs& a = G.m[gi].a;
  const LevelDev& lv = G.m[gi].lv;
  const int local = blockIdx.x - G.m[gi].cta_tail;
  const int h = local % a.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = (local / a.H) * kWarps + warp;
  if (i >= lv.n) {
    if (early) pdl_wait();
    return;
  }
  const int kh = h / (a.H / a.KV);
  const __nv_bfloat16* Kh = a.k + (size_t)kh * a.cap * kAttnHeadDim;
  const __nv_bfloat16* Vh = a.v + (size_t)kh * a.cap * kAttnHeadDim;
  const int P = __ldg(lv.prefix_rows + i);
  const int A = __ldg(lv.anc_cnt + i);
  const int T = P + A + 1;
  const int s0 = max(0, T - kAttnSuffix), ns = T - s0;
  // lane j < ns: the cache row of suffix slot s0 + j (-1 = self)
  int my_row = -1;
  if (lane < ns) {
    const int slot = s0 + lane;
    if (slot < P)
      my_row = slot;
    else if (slot < P + A)
      my_row = ancestor_row(lv.anc + (size_t)i * lv.words, slot - P, lv.bits_base);
  }
  const __nv_bfloat16* kself = a.kself ? a.kself + ((size_t)i * a.KV + kh) * kAttnHeadDim
                                       : Kh + (size_t)(lv.row0 + i) * kAttnHeadDim;
  const __nv_bfloat16* vself = a.vself ? a.vself + ((size_t)i * a.KV + kh) * kAttnHeadDim
                                       : Vh + (size_t)(lv.row0 + i) * kAttnHeadDim;
  const uint2 qv = *reinterpret_cast<const uint2*>(a.q + (size_t)i * a.q_stride + h * kAttnHeadDim + 4 * lane);
  const float q0 = __uint_as_float(qv.x << 16), q1 = __uint_as_float(qv.x & 0xffff0000u);
  const float q2 = __uint_as_float(qv.y << 16), q3 = __uint_as_float(qv.y & 0xffff0000u);
  // scores of the suffix slots (all loads first)
  uint2 kr[kAttnSuffix];
#pragma unroll
  for (int j = 0; j < kAttnSuffix; ++j) {
    const int row = __shfl_sync(0xffffffffu, my_row, j);
    const __nv_bfloat16* kp = row >= 0 ? Kh + (size_t)row * kAttnHeadDim : kself;
    kr[j] = j < ns ? __ldcg(reinterpret_cast<const uint2*>(kp + 4 * lane)) : make_uint2(0u, 0u);
  }
  float sc[kAttnSuffix];
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < kAttnSuffix; ++j) {
    float d = __fmul_rn(q0, __uint_as_float(kr[j].x << 16));
    d = __fmaf_rn(q1, __uint_as_float(kr[j].x & 0xffff0000u), d);
    d = __fmaf_rn(q2, __uint_as_float(kr[j].y << 16), d);
    d = __fmaf_rn(q3, __uint_as_float(kr[j].y & 0xffff0000u), d);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d = __fadd_rn(d, __shfl_xor_sync(0xffffffffu, d, o));
    sc[j] = j < ns ? __fmul_rn(d, a.scale) : -INFINITY;
    mx = fmaxf(mx, sc[j]);
  }
  uint2 vr[kAttnSuffix];
#pragma unroll
  for (int j = 0; j < kAttnSuffix; ++j) {
    const int row = __shfl_sync(0xffffffffu, my_row, j);
    const __nv_bfloat16* vp = row >= 0 ? Vh + (size_t)row * kAttnHeadDim : vself;
    vr[j] = j < ns ? __ldcg(reinterpret_cast<const uint2*>(vp + 4 * lane)) : make_uint2(0u, 0u);
  }
  float ls = 0.f;
  float4 os = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int j = 0; j < kAttnSuffix; ++j) {
    if (j >= ns) break;
    const float p = fast_exp(__fsub_rn(sc[j], mx));
    ls = __fadd_rn(ls, p);
    const float pb = __bfloat162float(__float2bfloat16_rn(p));  // P rounded to bf16, as the chunk path
    os.x = __fmaf_rn(pb, __uint_as_float(vr[j].x << 16), os.x);
    os.y = __fmaf_rn(pb, __uint_as_float(vr[j].x & 0xffff0000u), os.y);
    os.z = __fmaf_rn(pb, __uint_as_float(vr[j].y << 16), os.z);
    os.w = __fmaf_rn(pb, __uint_as_float(vr[j].y & 0xffff0000u), os.w);
  }
  if (early) pdl_wait();  // the chunk kernel's run states are complete from here on
  // ordered merge: runs of the chunked part, then the suffix
  float M = -INFINITY, L = 0.f;
  float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
  const int C = max(0, T - kAttnSuffix);
  const int nruns = ((C + kAttnChunk - 1) / kAttnChunk + G.run - 1) / G.run;
  const size_t pbase = part_idx(a, i, h, 0);
  const float4* po = reinterpret_cast<const float4*>(a.po + pbase * kAttnHeadDim) + lane;
  for (int r0 = 0; r0 < nruns; r0 += 8) {
    float4 blk[8];
    float pm[8], pl[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const bool ok = r0 + j < nruns;
      blk[j] = ok ? __ldcg(po + (size_t)(r0 + j) * (kAttnHeadDim / 4)) : O;
      pm[j] = ok ? __ldcg(a.pm + pbase + r0 + j) : -INFINITY;
      pl[j] = ok ? __ldcg(a.pl + pbase + r0 + j) : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (r0 + j < nruns) merge_lane(M, L, O, pm[j], pl[j], blk[j]);
  }
  merge_lane(M, L, O, mx, ls, os);
  __nv_bfloat16* out = a.out + (size_t)i * a.out_stride + h * kAttnHeadDim + 4 * lane;
  uint2 u;
  u.x = pack_f32(__fdiv_rn(O.x, L), __fdiv_rn(O.y, L));
  u.y = pack_f32(__fdiv_rn(O.z, L), __fdiv_rn(O.w, L));
  *reinterpret_cast<uint2*>(out) = u;
}

int attn_tree_group(const AttnArgs* a, const LevelDev* lv, int count, cudaStream_t st) {
  TP_CHECK(count >= 1 && count <= kAttnMaxGroup, TP_ECONFIG, "attention group size outside [1, 64]");
  AttnGroup G;
  G.count = count;
  G.run = g_attn_run;
  const int kRun = G.run;
  int cs = 0, ct = 0;
  for (int g = 0; g < count; ++g) {
    AttnMember& m = G.m[g];
    m.a = a[g];
    m.lv = lv[g];
    const int grp = a[g].H / a[g].KV;
    TP_CHECK(grp >= 1 && kCtaRows % grp == 0, TP_ESHAPE, "query group size must divide 64");
    m.max_c = std::max(0, lv[g].max_t - kAttnSuffix);  // longest chunked part of the member
    m.c_shared = (m.max_c + kAttnChunk - 1) / kAttnChunk;
    m.small = kRun <= kWarps && lv[g].n * grp <= kSmallRows;
    m.zt = m.small ? (lv[g].n * grp + 15) / 16 : (lv[g].n + kCtaRows / grp - 1) / (kCtaRows / grp);
    TP_CHECK(m.c_shared <= a[g].max_chunks, TP_ESHAPE, "attention chunks exceed scratch");
    m.cta_shared = cs;
    m.cta_tail = ct;
    m.cta_gqa = 0;
    cs += a[g].KV * ((m.c_shared + kRun - 1) / kRun) * m.zt;
    ct += a[g].H * ((lv[g].n + kWarps - 1) / kWarps);
  }
  static bool attr_set[64] = {false};  // per device
  int dev = 0;
  TP_CUDA(cudaGetDevice(&dev));
  if (!attr_set[dev & 63]) {
    TP_CUDA(cudaFuncSetAttribute(attn_chunks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kChunksSmem));
    attr_set[dev & 63] = true;
  }
  static const int dbg = getenv("TP_ATTN_DEBUG") ? atoi(getenv("TP_ATTN_DEBUG")) : 0;  // diagnostics: 1 skip tail, 2 skip chunks
  if (dbg & 2) cs = 0;
  if (dbg & 1) ct = 0;
  if (cs > 0) {
    ::tp::count_launch();
    TP_CUDA(launch_pdl(attn_chunks_kernel, dim3(cs), dim3(kWarps * 32), kChunksSmem, st, G));
    TP_CUDA(cudaGetLastError());
    timeline_mark("attn_shared", st);
  }
  if (ct > 0) {
    ::tp::count_launch();
    TP_CUDA(launch_pdl(attn_tail_kernel, dim3(ct), dim3(kWarps * 32), 0, st, G, cs > 0 ? 1 : 0));
    TP_CUDA(cudaGetLastError());
    timeline_mark("attn_tail", st);
  }
  return TP_OK;
}

int attn_tree(const AttnArgs& a, const LevelDev& lv, cudaStream_t st) { return attn_tree_group(&a, &lv, 1, st); }

int attn_set_run(int run) {
  TP_CHECK(run >= 1 && run <= 64, TP_ECONFIG, "attention run length outside [1, 64]");
  g_attn_run = run;
  return TP_OK;
}

}  // namespace tp
