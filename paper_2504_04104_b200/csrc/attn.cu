// K1: tree-masked attention of a level's nodes against one stage's KV cache
// (Llama path; replaces the gather + softmax + PV of the reference
// layer_step, `/root/reference/pkg/src/treepipe/model.py:157-167,265-276`).
//
// Node i attends its *logical* key sequence: cache rows [0, P_i) (verified
// prefix), then its speculative ancestors in row order (the set bits of its
// packed ancestor row, decoded in registers), then itself.  The sequence is
// cut into canonical 64-slot chunks (slot = logical position mod 64).  Each
// chunk yields a partial (max, sum, unnormalised P.V) from one m16n8k16 bf16
// tensor-core pass over a padded shared-memory tile (ldmatrix fragments), and
// the partials are merged in chunk order.  Two launches per layer slot, each
// covering every stage of the group:
//   attn_shared_kernel  chunks entirely inside every node's verified prefix
//                       (c < floor(min_i P_i / 64)): the K/V chunk is staged
//                       once in shared memory for 4 warps x 16 nodes;
//   attn_tail_kernel    one warp per (node, head): merges the shared chunks'
//                       partials in order, then stages each remaining chunk
//                       (prefix tail, ancestors, self) in shared memory, runs
//                       it with the node in row 0 of the MMA tile, merges, and
//                       writes the bf16 output.
//
// Batch invariance: the arithmetic applied to a node depends only on its own
// logical key sequence — never on its launch-mates, on where its keys live
// (prefix vs speculative rows) or on which kernel handled a chunk (both
// kernels run the same chunk code on the same smem tile layout; tensor-core
// rows are independent; merges use explicitly rounded ops so the compiler
// cannot contract them differently at the two merge sites).  A node computed
// inside a 64-node tree level is therefore bit-identical to the same position
// decoded alone (GPU pipeline == GPU greedy decode).
#include "attn.h"
#include "gemm_tc.h"

namespace tp {

#ifndef TP_TAIL_MINB
#define TP_TAIL_MINB 3
#endif
#ifndef TP_SHARED_MINB
#define TP_SHARED_MINB 4
#endif
constexpr int kPad = 136;  // bf16 per staged row: 128 + 8 pad (conflict-free ldmatrix)
constexpr int kCtaNodes = 64;
constexpr int kWarps = 4;
constexpr int kTileElems = kAttnChunk * kPad;
static bool g_attn_tail2 = false;  // shared-prefix tail for uniform levels (knob 2): bit-exact, measured no faster
static bool g_attn_tile = false;  // measured slower than the per-node tail on the bench workload  // tp_debug_attn_tile(0) forces the per-node path (tests)
constexpr size_t kTailSmem = (size_t)kWarps * kTileElems * 2;

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

// The same MMA sequences with per-slot row pointers (rows gathered from a CTA
// tile, a per-warp own-row buffer and a zero row): identical fragments, so
// identical results.
template <typename RowK>
__device__ __forceinline__ void tile_qk_rows(const uint32_t (&qa)[8][4], RowK rowK, float (&s)[8][4], int lane) {
  const int mi = lane >> 3, mr = lane & 7;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
    const __nv_bfloat16* rp = rowK(nt * 8 + mr);
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
      uint32_t b[4];
      ldsm4(su32(rp + 32 * k2 + 8 * mi), b);
      mma16816(s[nt], qa[2 * k2], b[0], b[1]);
      mma16816(s[nt], qa[2 * k2 + 1], b[2], b[3]);
    }
  }
}

template <typename RowV>
__device__ __forceinline__ void chunk_pv_rows(const uint32_t (&pa)[4][4], RowV rowV, float (&o)[16][4], int lane) {
  const int mi = lane >> 3, mr = lane & 7;
#pragma unroll
  for (int nd = 0; nd < 16; ++nd) o[nd][0] = o[nd][1] = o[nd][2] = o[nd][3] = 0.f;
#pragma unroll
  for (int n2 = 0; n2 < 8; ++n2)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t b[4];
      ldsm4t(su32(rowV(16 * kk + 8 * (mi & 1) + mr) + 16 * n2 + 8 * (mi >> 1)), b);
      mma16816(o[2 * n2], pa[kk], b[0], b[1]);
      mma16816(o[2 * n2 + 1], pa[kk], b[2], b[3]);
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

// o = P . V for the chunk, V staged in sV[slot][kPad] (ldmatrix.trans B fragments).
__device__ __forceinline__ void chunk_pv(const uint32_t (&pa)[4][4], const __nv_bfloat16* sV, float (&o)[16][4],
                                         int lane) {
  const int mi = lane >> 3, mr = lane & 7;
#pragma unroll
  for (int nd = 0; nd < 16; ++nd) o[nd][0] = o[nd][1] = o[nd][2] = o[nd][3] = 0.f;
#pragma unroll
  for (int n2 = 0; n2 < 8; ++n2)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t b[4];  // b0/b1 of n-tiles 2*n2 and 2*n2+1
      ldsm4t(su32(sV + (16 * kk + 8 * (mi & 1) + mr) * kPad + 16 * n2 + 8 * (mi >> 1)), b);
      mma16816(o[2 * n2], pa[kk], b[0], b[1]);
      mma16816(o[2 * n2 + 1], pa[kk], b[2], b[3]);
    }
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

// kind: 0 shared, 1 per-node tail, 2 tile
__device__ __forceinline__ int member_of(const AttnGroup& G, int b, int kind) {
  auto start = [&](int g) {
    return kind == 0   ? G.m[g].cta_shared
           : kind == 1 ? G.m[g].cta_tail
           : kind == 2 ? G.m[g].cta_tile
           : kind == 3 ? G.m[g].cta_tail2
                       : G.m[g].cta_gqa;
  };
  int gi = 0;
  while (gi + 1 < G.count && b >= start(gi + 1)) ++gi;
  return gi;
}

// Chunks inside every node's verified prefix: rows [64c, 64c+64) for all nodes.
// A CTA walks kSharedRun consecutive chunks of one (member, head, 64-node
// block), staging chunk c+1 (cp.async, double-buffered) while chunk c computes;
// every chunk's partial is stored separately, exactly as one CTA per chunk.
constexpr int kSharedRunMax = 4;
constexpr size_t kSharedSmem = (size_t)4 * kTileElems * 2;  // 2 x (K, V) chunk tiles
static int g_shared_run = 1;  // chunks per CTA (tp_debug_attn_knob 1)

__global__ void __launch_bounds__(kWarps * 32, TP_SHARED_MINB) attn_shared_kernel(const __grid_constant__ AttnGroup G, int run_len) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t dsm[];
  const int gi = member_of(G, blockIdx.x, 0);
  const AttnArgs& a = G.m[gi].a;
  const LevelDev& lv = G.m[gi].lv;
  const int runs = (G.m[gi].c_shared + run_len - 1) / run_len;
  // one CTA per (member, KV head, run of chunks, 64-node block): the K/V chunk is
  // staged once for every query head of the GQA group (MHA: group of 1)
  int local = blockIdx.x - G.m[gi].cta_shared;
  const int kh = local % a.KV;
  local /= a.KV;
  const int run = local % runs, base = (local / runs) * kCtaNodes;
  const int c0 = run * run_len, c1 = min(G.m[gi].c_shared, c0 + run_len);
  const int grp = a.H / a.KV;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int nreal = min(kCtaNodes, lv.n - base);
  const int rows = nreal * grp;  // (query head, node) pairs, head-major
  const int tiles = (rows + 15) / 16;
  __nv_bfloat16* smt = reinterpret_cast<__nv_bfloat16*>(dsm);  // [2][K | V][kTileElems]
  auto stage = [&](int c, int buf) {
    const __nv_bfloat16* Kh = a.k + ((size_t)kh * a.cap + (size_t)c * kAttnChunk) * kAttnHeadDim;
    const __nv_bfloat16* Vh = a.v + ((size_t)kh * a.cap + (size_t)c * kAttnChunk) * kAttnHeadDim;
    __nv_bfloat16* sK = smt + (size_t)buf * 2 * kTileElems;
    __nv_bfloat16* sV = sK + kTileElems;
#pragma unroll
    for (int e = threadIdx.x; e < kAttnChunk * 16; e += kWarps * 32) {
      const int row = e >> 4, part = e & 15;
      cp16(sK + row * kPad + part * 8, Kh + row * kAttnHeadDim + part * 8, 16);
      cp16(sV + row * kPad + part * 8, Vh + row * kAttnHeadDim + part * 8, 16);
    }
    cp_commit();
  };
  stage(c0, 0);
  for (int c = c0; c < c1; ++c) {
    const int buf = (c - c0) & 1;
    if (c + 1 < c1) {
      stage(c + 1, buf ^ 1);
      cp_wait_group<1>();
    } else {
      cp_wait_group<0>();
    }
    __syncthreads();
    const __nv_bfloat16* sK = smt + (size_t)buf * 2 * kTileElems;
    for (int t = warp; t < tiles; t += kWarps) {
      const int ra = 16 * t + g, rb = ra + 8;
      const bool va = ra < rows, vb = rb < rows;
      const int ia = base + (va ? ra % nreal : 0), ib = base + (vb ? rb % nreal : 0);
      const int ha = kh * grp + (va ? ra / nreal : 0), hb = kh * grp + (vb ? rb / nreal : 0);
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
      const int lim[2] = {va ? kAttnChunk : 0, vb ? kAttnChunk : 0};
      float m[2], l[2], o[16][4];
      uint32_t pa[4][4];
      chunk_scores(qa, sK, lim, a.scale, m, l, pa, lane);
      chunk_pv(pa, sK + kTileElems, o, lane);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        if (!(hh ? vb : va)) continue;
        const size_t idx = part_idx(a, hh ? ib : ia, hh ? hb : ha, c);
        float* po = a.po + idx * kAttnHeadDim;
#pragma unroll
        for (int nd = 0; nd < 16; ++nd)
          *reinterpret_cast<float2*>(po + nd * 8 + 2 * tig) = make_float2(o[nd][2 * hh], o[nd][2 * hh + 1]);
        if (tig == 0) {
          a.pm[idx] = m[hh];
          a.pl[idx] = l[hh];
        }
      }
    }
    __syncthreads();  // buffer `buf` is restaged for chunk c + 2
  }
}

// One warp per (node, head): the node's own chunks (prefix tail, ancestors,
// self), then the ordered merge of the shared chunks' partials followed by its
// own chunks' partials, then the bf16 output row.  The running state lives in
// "lane layout" (lane l owns dims 4l..4l+3); a chunk computed on the tensor
// cores (row 0 of the tile, fragment layout) is handed over through smem.
//
// `early` (an attention kernel precedes this one in the stream, so the QKV
// GEMM has completed before this grid is launched): up to kEarly own chunks
// are computed BEFORE griddepcontrol.wait, i.e. while the shared-prefix kernel
// is still running; only the merge waits for its partials.  Loads issued
// before the wait bypass L1 (.cg).  The merge order — shared chunks, then own
// chunks, each in chunk order — and every chunk's arithmetic are unchanged.
constexpr int kEarly = 2;
__global__ void __launch_bounds__(kWarps * 32, TP_TAIL_MINB)
    attn_tail_kernel(const __grid_constant__ AttnGroup G, int early) {
  if (!early) pdl_wait();
  pdl_trigger();  // the O-projection GEMM may start streaming its weights
  extern __shared__ __align__(16) uint8_t dsm[];
  const int gi = member_of(G, blockIdx.x, 1);
  const AttnArgs& a = G.m[gi].a;
  const LevelDev& lv = G.m[gi].lv;
  int local = blockIdx.x - G.m[gi].cta_tail;
  const int h = local % a.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int i = (local / a.H) * kWarps + warp;
  const bool live = i < lv.n;
  __nv_bfloat16* buf = reinterpret_cast<__nv_bfloat16*>(dsm) + (size_t)warp * kTileElems;
  float* xo = reinterpret_cast<float*>(buf);  // 128-float hand-over row (aliases the tile between chunks)
  const int kh = h / (a.H / a.KV);
  const __nv_bfloat16* Kh = a.k + (size_t)kh * a.cap * kAttnHeadDim;
  const __nv_bfloat16* Vh = a.v + (size_t)kh * a.cap * kAttnHeadDim;
  const int c_start = G.m[gi].c_shared;
  const int ii = live ? i : 0;
  const int A = __ldcg(lv.anc_cnt + ii);
  const int32_t* anc = lv.anc_rows + (size_t)ii * lv.anc_stride;  // decoded on the host, row order
  const int anc_l = lane < A ? __ldcg(anc + lane) : 0;            // first 32 ancestors in lane registers
  const int P = __ldcg(lv.prefix_rows + ii);
  const int T = P + A + 1;
  const __nv_bfloat16* kself = a.kself ? a.kself + ((size_t)ii * a.KV + kh) * kAttnHeadDim
                                       : Kh + (size_t)(lv.row0 + ii) * kAttnHeadDim;
  const __nv_bfloat16* vself = a.vself ? a.vself + ((size_t)ii * a.KV + kh) * kAttnHeadDim
                                       : Vh + (size_t)(lv.row0 + ii) * kAttnHeadDim;
  uint32_t q1[8][4];
  {
    const uint32_t* qr = reinterpret_cast<const uint32_t*>(a.q + (size_t)ii * a.q_stride + h * kAttnHeadDim);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      q1[kk][0] = g == 0 ? __ldcg(qr + 8 * kk + tig) : 0u;
      q1[kk][1] = 0u;
      q1[kk][2] = g == 0 ? __ldcg(qr + 8 * kk + 4 + tig) : 0u;
      q1[kk][3] = 0u;
    }
  }
  const int c_end = (T + kAttnChunk - 1) / kAttnChunk;
  const int part = lane & 15, rsub = lane >> 4;  // this lane stages 16-byte piece `part` of rows rsub, rsub+2, ...
  // stage the chunk's rows of one plane: prefix rows (affine), own rows (gathered), zeros beyond T
  auto stage = [&](const __nv_bfloat16* plane, const __nv_bfloat16* self, int j0) {
    const int np = min(max(P - j0, 0), kAttnChunk);   // prefix rows in this chunk
    const int nt = min(T - j0, kAttnChunk);           // rows holding keys
    const __nv_bfloat16* pre = plane + (size_t)j0 * kAttnHeadDim + part * 8;
    for (int row = rsub; row < np; row += 2) cp16(buf + row * kPad + part * 8, pre + (size_t)row * kAttnHeadDim, 16);
    for (int r0 = np; r0 < nt; r0 += 2) {  // warp-uniform trip count (the shuffle below)
      const int row = r0 + rsub;
      const int ai = j0 + row - P;  // ancestor index, A = self
      const int av = __shfl_sync(0xffffffffu, anc_l, ai & 31);
      if (row < nt) {
        const __nv_bfloat16* src =
            ai < A ? plane + (size_t)(ai < 32 ? av : __ldcg(anc + ai)) * kAttnHeadDim : self;
        cp16(buf + row * kPad + part * 8, src + part * 8, 16);
      }
    }
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    for (int row = max(nt, 0) + rsub; row < kAttnChunk; row += 2)
      *reinterpret_cast<uint4*>(buf + row * kPad + part * 8) = z;
    cp_wait_all();
    __syncwarp();
  };
  // one own chunk -> its partial (mc, lc warp-uniform; oc in lane layout)
  auto run_chunk = [&](int c, float& mc, float& lc, float4& oc) {
    const int j0 = c * kAttnChunk;
    __syncwarp();  // previous chunk's hand-over row has been read
    stage(Kh, kself, j0);
    const int lim[2] = {g == 0 ? min(T - j0, kAttnChunk) : 0, 0};
    float m[2], l[2], o[16][4];
    uint32_t pa[4][4];
    chunk_scores(q1, buf, lim, a.scale, m, l, pa, lane);
    __syncwarp();
    stage(Vh, vself, j0);
    chunk_pv(pa, buf, o, lane);
    __syncwarp();  // every lane is done reading the tile: reuse it for the hand-over row
    if (g == 0) {
#pragma unroll
      for (int nd = 0; nd < 16; ++nd)
        *reinterpret_cast<float2*>(xo + nd * 8 + 2 * tig) = make_float2(o[nd][0], o[nd][1]);
    }
    __syncwarp();
    oc = *reinterpret_cast<const float4*>(xo + 4 * lane);
    mc = __shfl_sync(0xffffffffu, m[0], 0);
    lc = __shfl_sync(0xffffffffu, l[0], 0);
  };
  // running state, lane layout: dims 4*lane .. 4*lane+3
  float M = -INFINITY, L = 0.f;
  float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
  auto merge_in = [&](float mc, float lc, float4 oc) {
    float sa, sb;
    merge_scale(M, L, mc, lc, sa, sb);
    O.x = merge_val(O.x, oc.x, sa, sb);
    O.y = merge_val(O.y, oc.y, sa, sb);
    O.z = merge_val(O.z, oc.z, sa, sb);
    O.w = merge_val(O.w, oc.w, sa, sb);
  };
  const int n_early = early && live ? min(c_end - c_start, kEarly) : 0;
  float em[kEarly], el[kEarly];
  float4 eo[kEarly];
#pragma unroll
  for (int k = 0; k < kEarly; ++k)
    if (k < n_early) run_chunk(c_start + k, em[k], el[k], eo[k]);
  if (early) pdl_wait();  // the shared-prefix partials are complete from here on
  if (!live) return;
  {  // shared chunks' partials, 8 chunk rows in flight per batch (one L2 round trip per batch)
    constexpr int kPre = 8;
    const size_t pbase = part_idx(a, i, h, 0);
    const float4* po = reinterpret_cast<const float4*>(a.po + pbase * kAttnHeadDim) + lane;
    float pm_l = -INFINITY, pl_l = 0.f;  // lane c holds chunk c0 + c's (max, sum)
    for (int c0 = 0; c0 < c_start; c0 += kPre) {
      if ((c0 & 31) == 0) {
        pm_l = c0 + lane < c_start ? __ldcg(a.pm + pbase + c0 + lane) : -INFINITY;
        pl_l = c0 + lane < c_start ? __ldcg(a.pl + pbase + c0 + lane) : 0.f;
      }
      float4 blk[kPre];
#pragma unroll
      for (int j = 0; j < kPre; ++j)
        blk[j] = c0 + j < c_start ? __ldcg(po + (size_t)(c0 + j) * (kAttnHeadDim / 4)) : O;
#pragma unroll
      for (int j = 0; j < kPre; ++j) {
        const int c = c0 + j;
        if (c >= c_start) break;
        merge_in(__shfl_sync(0xffffffffu, pm_l, c & 31), __shfl_sync(0xffffffffu, pl_l, c & 31), blk[j]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kEarly; ++k)
    if (k < n_early) merge_in(em[k], el[k], eo[k]);
  for (int c = c_start + n_early; c < c_end; ++c) {
    float mc, lc;
    float4 oc;
    run_chunk(c, mc, lc, oc);
    merge_in(mc, lc, oc);
  }
  __nv_bfloat16* out = a.out + (size_t)i * a.out_stride + h * kAttnHeadDim + 4 * lane;
  uint2 u;
  u.x = pack_f32(__fdiv_rn(O.x, L), __fdiv_rn(O.y, L));
  u.y = pack_f32(__fdiv_rn(O.z, L), __fdiv_rn(O.w, L));
  *reinterpret_cast<uint2*>(out) = u;
}

// ---------------------------------------------------------------------------
// Tree levels (every node has the same prefix P and the same number A of
// speculative ancestors — the common case, `uniform_a` >= 0): one warp per
// 16-node tile.  A tail chunk's slots below P are the same K/V rows for every
// node: they are staged once per CTA and run as ordinary tile MMAs.  Only the
// node's own slots [P, P+A] (ancestors + self, <= kTileOwn) differ: for those
// n-tiles / k-groups the node runs alone in row 0 of an MMA (the per-lane
// ldmatrix addresses mix shared and own rows), exactly the arithmetic of the
// per-node path, with its accumulator moved to row 0 and back by shuffles.
// Per element the operations and their order are those of attn_tail_kernel,
// so the result is bit-identical to it (and to sequential decode).
constexpr int kTileOwn = 16;
constexpr int kOwnElems = kTileOwn * kPad;
constexpr int kOwnRing = 4;  // per-warp ring of staged own-row tiles: nodes r+1..r+3 load while r computes
constexpr size_t kTileWarpBytes = (size_t)kOwnRing * kOwnElems * 2 + (size_t)16 * kTileOwn * 4;
constexpr size_t kTileSmem = (size_t)2 * kTileElems * 2 + (size_t)kPad * 2 + kWarps * kTileWarpBytes;

__global__ void __launch_bounds__(kWarps * 32) attn_tile_kernel(const __grid_constant__ AttnGroup G) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t dsm[];
  const int gi = member_of(G, blockIdx.x, 2);
  const AttnArgs& a = G.m[gi].a;
  const LevelDev& lv = G.m[gi].lv;
  const int local = blockIdx.x - G.m[gi].cta_tile;
  const int h = local % a.H, base = (local / a.H) * kCtaNodes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3, mi = lane >> 3, mr = lane & 7;
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(dsm);
  __nv_bfloat16* sV = sK + kTileElems;
  __nv_bfloat16* zrow = sV + kTileElems;
  uint8_t* wb = reinterpret_cast<uint8_t*>(zrow + kPad) + warp * kTileWarpBytes;
  __nv_bfloat16* ring = reinterpret_cast<__nv_bfloat16*>(wb);
  int* extra = reinterpret_cast<int*>(ring + kOwnRing * kOwnElems);  // [16][kTileOwn]
  const int kh = h / (a.H / a.KV);
  const __nv_bfloat16* Kh = a.k + (size_t)kh * a.cap * kAttnHeadDim;
  const __nv_bfloat16* Vh = a.v + (size_t)kh * a.cap * kAttnHeadDim;
  const int P = lv.min_p, A = lv.uniform_a, T = P + A + 1;
  const int t0 = base + warp * 16;
  const int nv = min(16, lv.n - t0);
  for (int e = threadIdx.x; e < kPad; e += blockDim.x) zrow[e] = __float2bfloat16_rn(0.f);
  if (lane < nv) {  // lane r decodes node t0 + r's ancestor rows (A of them, in row order)
    int cnt = 0;
    for (int w = 0; w < lv.words && cnt < A; ++w) {
      uint64_t bits = lv.anc[(size_t)(t0 + lane) * lv.words + w];
      while (bits && cnt < A) {
        extra[lane * kTileOwn + cnt++] = lv.bits_base + w * 64 + (__ffsll((long long)bits) - 1);
        bits &= bits - 1;
      }
    }
  }
  const bool va = g < nv, vb = g + 8 < nv;
  const __nv_bfloat16* qra = a.q + (size_t)(t0 + g) * a.q_stride + h * kAttnHeadDim;
  const __nv_bfloat16* qrb = a.q + (size_t)(t0 + g + 8) * a.q_stride + h * kAttnHeadDim;
  // running state of rows g / g+8 (fragment layout)
  float M[2] = {-INFINITY, -INFINITY}, L[2] = {0.f, 0.f}, O[16][4];
#pragma unroll
  for (int nd = 0; nd < 16; ++nd) O[nd][0] = O[nd][1] = O[nd][2] = O[nd][3] = 0.f;
  const int c_start = G.m[gi].c_shared;
  for (int c = 0; c < c_start; ++c) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int r = g + 8 * hh;
      if (r >= nv) continue;
      const size_t idx = part_idx(a, t0 + r, h, c);
      float sa, sb;
      merge_scale(M[hh], L[hh], __ldcg(a.pm + idx), __ldcg(a.pl + idx), sa, sb);
      const float* po = a.po + idx * kAttnHeadDim + 2 * tig;
#pragma unroll
      for (int nd = 0; nd < 16; ++nd) {
        const float2 v = __ldcg(reinterpret_cast<const float2*>(po + nd * 8));
        O[nd][2 * hh] = merge_val(O[nd][2 * hh], v.x, sa, sb);
        O[nd][2 * hh + 1] = merge_val(O[nd][2 * hh + 1], v.y, sa, sb);
      }
    }
  }
  __syncwarp();
  // own row o (0..A-1 ancestors, A self) of node t0 + r; nullptr beyond
  auto own_src = [&](int r, int o, bool isv) -> const __nv_bfloat16* {
    if (o < A) return (isv ? Vh : Kh) + (size_t)extra[r * kTileOwn + o] * kAttnHeadDim;
    if (o == A) {
      const int i = t0 + r;
      const __nv_bfloat16* self = isv ? a.vself : a.kself;
      return self ? self + ((size_t)i * a.KV + kh) * kAttnHeadDim
                  : (isv ? Vh : Kh) + (size_t)(lv.row0 + i) * kAttnHeadDim;
    }
    return nullptr;
  };
  auto stage_own = [&](int r, __nv_bfloat16* dst, bool isv) {  // only the A+1 rows ever read
#pragma unroll 4
    for (int e = lane; e < (A + 1) * 16; e += 32) {
      const int o = e >> 4, part = e & 15;
      const __nv_bfloat16* src = own_src(r, o, isv);
      cp16(dst + o * kPad + part * 8, (src ? src : Kh) + part * 8, src ? 16 : 0);
    }
    cp_commit();
  };
  const int c_end = (T + kAttnChunk - 1) / kAttnChunk;
  for (int c = c_start; c < c_end; ++c) {
    const int j0 = c * kAttnChunk;
    __syncthreads();  // every warp is done with the previous chunk's shared rows
#pragma unroll
    for (int e = threadIdx.x; e < kAttnChunk * 16; e += kWarps * 32) {
      const int row = e >> 4, part = e & 15, j = j0 + row;
      const bool ok = j < P;
      cp16(sK + row * kPad + part * 8, Kh + (size_t)(ok ? j : 0) * kAttnHeadDim + part * 8, ok ? 16 : 0);
      cp16(sV + row * kPad + part * 8, Vh + (size_t)(ok ? j : 0) * kAttnHeadDim + part * 8, ok ? 16 : 0);
    }
    cp_wait_all();
    __syncthreads();
    if (nv <= 0) continue;
    const int lo_slot = max(P - j0, 0), hi_slot = min(T - j0, kAttnChunk);  // own slots of this chunk
    auto rowp = [&](const __nv_bfloat16* shared_tile, const __nv_bfloat16* own, int slot) {
      const int ja = j0 + slot;
      return ja < P ? shared_tile + slot * kPad : (ja < T ? own + (ja - P) * kPad : zrow);
    };
    uint32_t qa[8][4];  // reloaded per chunk (L2): keeps registers free for the P.V phase
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      qa[kk][0] = va ? ld_b32(qra + 16 * kk + 2 * tig) : 0u;
      qa[kk][1] = vb ? ld_b32(qrb + 16 * kk + 2 * tig) : 0u;
      qa[kk][2] = va ? ld_b32(qra + 16 * kk + 8 + 2 * tig) : 0u;
      qa[kk][3] = vb ? ld_b32(qrb + 16 * kk + 8 + 2 * tig) : 0u;
    }
    float s[8][4];
    tile_qk(qa, sK, s, lane);
    if (lo_slot < hi_slot) {
      const int nt0 = lo_slot >> 3, nt1 = (hi_slot - 1) >> 3;
      for (int p = 0; p < min(kOwnRing - 1, nv); ++p) stage_own(p, ring + (p % kOwnRing) * kOwnElems, false);
      for (int r = 0; r < nv; ++r) {
        __nv_bfloat16* own = ring + (r % kOwnRing) * kOwnElems;
        if (r + kOwnRing - 1 < nv)
          stage_own(r + kOwnRing - 1, ring + ((r + kOwnRing - 1) % kOwnRing) * kOwnElems, false);
        cp_wait_ahead(min(kOwnRing - 1, nv - 1 - r));
        __syncwarp();
        const int src_lane = (r & 7) * 4 + tig, hr = r >> 3;
        uint32_t q1[8][4];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t v0 = __shfl_sync(0xffffffffu, hr ? qa[kk][1] : qa[kk][0], src_lane);
          const uint32_t v2 = __shfl_sync(0xffffffffu, hr ? qa[kk][3] : qa[kk][2], src_lane);
          q1[kk][0] = g == 0 ? v0 : 0u;
          q1[kk][1] = 0u;
          q1[kk][2] = g == 0 ? v2 : 0u;
          q1[kk][3] = 0u;
        }
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
          if (nt < nt0 || nt > nt1) continue;
          float s1[4] = {0.f, 0.f, 0.f, 0.f};
          const __nv_bfloat16* rp = rowp(sK, own, nt * 8 + mr);
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2) {
            uint32_t b[4];
            ldsm4(su32(rp + 32 * k2 + 8 * mi), b);
            mma16816(s1, q1[2 * k2], b[0], b[1]);
            mma16816(s1, q1[2 * k2 + 1], b[2], b[3]);
          }
          const float e0 = __shfl_sync(0xffffffffu, s1[0], tig), e1 = __shfl_sync(0xffffffffu, s1[1], tig);
          if (g == (r & 7)) {
            if (hr) {
              s[nt][2] = e0;
              s[nt][3] = e1;
            } else {
              s[nt][0] = e0;
              s[nt][1] = e1;
            }
          }
        }
        __syncwarp();  // buffer `own` may be restaged for node r + 2
      }
    }
    const int lim[2] = {g < nv ? min(T - j0, kAttnChunk) : 0, g + 8 < nv ? min(T - j0, kAttnChunk) : 0};
    float m[2], l[2];
    uint32_t pa[4][4];
    chunk_softmax(s, lim, a.scale, m, l, pa, lane);
    float o[16][4];
#pragma unroll
    for (int nd = 0; nd < 16; ++nd) o[nd][0] = o[nd][1] = o[nd][2] = o[nd][3] = 0.f;
    const bool any_own = lo_slot < hi_slot;
    const int kk_lo = any_own ? lo_slot >> 4 : 4, kk_hi = any_own ? (hi_slot - 1) >> 4 : 3;
    auto tile_group = [&](int kk) {
#pragma unroll
      for (int n2 = 0; n2 < 8; ++n2) {
        uint32_t b[4];
        ldsm4t(su32(sV + (16 * kk + 8 * (mi & 1) + mr) * kPad + 16 * n2 + 8 * (mi >> 1)), b);
        mma16816(o[2 * n2], pa[kk], b[0], b[1]);
        mma16816(o[2 * n2 + 1], pa[kk], b[2], b[3]);
      }
    };
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
      if (kk < kk_lo) tile_group(kk);
    if (any_own) {
      for (int p = 0; p < min(kOwnRing - 1, nv); ++p) stage_own(p, ring + (p % kOwnRing) * kOwnElems, true);
      for (int r = 0; r < nv; ++r) {
        __nv_bfloat16* own = ring + (r % kOwnRing) * kOwnElems;
        if (r + kOwnRing - 1 < nv)
          stage_own(r + kOwnRing - 1, ring + ((r + kOwnRing - 1) % kOwnRing) * kOwnElems, true);
        cp_wait_ahead(min(kOwnRing - 1, nv - 1 - r));
        __syncwarp();
        const int src_lane = (r & 7) * 4 + tig, hr = r >> 3;
#pragma unroll
        for (int half = 0; half < 2; ++half) {  // n-tiles 8*half .. 8*half+7 (accumulators independent per n-tile)
          float acc[8][4];
#pragma unroll
          for (int q8 = 0; q8 < 8; ++q8) {
            const int nd = 8 * half + q8;
            const float c0 = __shfl_sync(0xffffffffu, hr ? o[nd][2] : o[nd][0], src_lane);
            const float c1 = __shfl_sync(0xffffffffu, hr ? o[nd][3] : o[nd][1], src_lane);
            acc[q8][0] = g == 0 ? c0 : 0.f;
            acc[q8][1] = g == 0 ? c1 : 0.f;
            acc[q8][2] = acc[q8][3] = 0.f;
          }
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            if (kk < kk_lo || kk > kk_hi) continue;
            uint32_t p1[4];
            const uint32_t v0 = __shfl_sync(0xffffffffu, hr ? pa[kk][1] : pa[kk][0], src_lane);
            const uint32_t v2 = __shfl_sync(0xffffffffu, hr ? pa[kk][3] : pa[kk][2], src_lane);
            p1[0] = g == 0 ? v0 : 0u;
            p1[1] = 0u;
            p1[2] = g == 0 ? v2 : 0u;
            p1[3] = 0u;
            const __nv_bfloat16* rp = rowp(sV, own, 16 * kk + 8 * (mi & 1) + mr);
#pragma unroll
            for (int n4 = 0; n4 < 4; ++n4) {
              const int n2 = 4 * half + n4;
              uint32_t b[4];
              ldsm4t(su32(rp + 16 * n2 + 8 * (mi >> 1)), b);
              mma16816(acc[2 * n4], p1, b[0], b[1]);
              mma16816(acc[2 * n4 + 1], p1, b[2], b[3]);
            }
          }
#pragma unroll
          for (int q8 = 0; q8 < 8; ++q8) {
            const int nd = 8 * half + q8;
            const float e0 = __shfl_sync(0xffffffffu, acc[q8][0], tig);
            const float e1 = __shfl_sync(0xffffffffu, acc[q8][1], tig);
            if (g == (r & 7)) {
              if (hr) {
                o[nd][2] = e0;
                o[nd][3] = e1;
              } else {
                o[nd][0] = e0;
                o[nd][1] = e1;
              }
            }
          }
        }
        __syncwarp();
      }
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
      if (kk > kk_hi) tile_group(kk);
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      float sa, sb;
      merge_scale(M[hh], L[hh], m[hh], l[hh], sa, sb);
#pragma unroll
      for (int nd = 0; nd < 16; ++nd) {
        O[nd][2 * hh] = merge_val(O[nd][2 * hh], o[nd][2 * hh], sa, sb);
        O[nd][2 * hh + 1] = merge_val(O[nd][2 * hh + 1], o[nd][2 * hh + 1], sa, sb);
      }
    }
  }
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    const int r = g + 8 * hh;
    if (r >= nv) continue;
    __nv_bfloat16* out = a.out + (size_t)(t0 + r) * a.out_stride + h * kAttnHeadDim + 2 * tig;
#pragma unroll
    for (int nd = 0; nd < 16; ++nd)
      *reinterpret_cast<uint32_t*>(out + nd * 8) =
          pack_f32(__fdiv_rn(O[nd][2 * hh], L[hh]), __fdiv_rn(O[nd][2 * hh + 1], L[hh]));
  }
}


// ---------------------------------------------------------------------------
// Per-node tail for uniform tree levels (every node: prefix P, A ancestors):
// a CTA's 4 warps are 4 nodes of one (member, head), so the tail chunk's
// prefix rows [64c, P) are staged ONCE per CTA; each warp stages only its own
// <= kOwnMax rows (ancestors + self).  The chunk math reads fragments through
// per-slot row pointers — the same bytes in the same MMA order as the per-node
// path, hence the same bits.
constexpr int kOwnMax = 16;
constexpr size_t kTail2Smem = (size_t)2 * kTileElems * 2 + (size_t)kWarps * 2 * kOwnMax * kPad * 2 +
                              (size_t)kPad * 2 + (size_t)kWarps * 128 * 4;

__global__ void __launch_bounds__(kWarps * 32, 3) attn_tail2_kernel(const __grid_constant__ AttnGroup G) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t dsm[];
  const int gi = member_of(G, blockIdx.x, 3);
  const AttnArgs& a = G.m[gi].a;
  const LevelDev& lv = G.m[gi].lv;
  const int local = blockIdx.x - G.m[gi].cta_tail2;
  const int h = local % a.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int i = (local / a.H) * kWarps + warp;
  const bool valid = i < lv.n;
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(dsm);
  __nv_bfloat16* sV = sK + kTileElems;
  __nv_bfloat16* oK = sV + kTileElems + (size_t)warp * 2 * kOwnMax * kPad;
  __nv_bfloat16* oV = oK + kOwnMax * kPad;
  __nv_bfloat16* zrow = sV + kTileElems + (size_t)kWarps * 2 * kOwnMax * kPad;
  float* xo = reinterpret_cast<float*>(zrow + kPad) + warp * 128;
  for (int e = threadIdx.x; e < kPad; e += blockDim.x) zrow[e] = __float2bfloat16_rn(0.f);
  const int kh = h / (a.H / a.KV);
  const __nv_bfloat16* Kh = a.k + (size_t)kh * a.cap * kAttnHeadDim;
  const __nv_bfloat16* Vh = a.v + (size_t)kh * a.cap * kAttnHeadDim;
  const int c_start = G.m[gi].c_shared;
  const int P = lv.min_p, A = lv.uniform_a, T = P + A + 1;
  const int ic = valid ? i : 0;
  const size_t pbase = part_idx(a, ic, h, 0);
  float pm_l = -INFINITY, pl_l = 0.f;
  if (valid && lane < c_start) {
    pm_l = __ldcg(a.pm + pbase + lane);
    pl_l = __ldcg(a.pl + pbase + lane);
  }
  const int32_t* anc = lv.anc_rows + (size_t)ic * lv.anc_stride;
  const __nv_bfloat16* kself = a.kself ? a.kself + ((size_t)ic * a.KV + kh) * kAttnHeadDim
                                       : Kh + (size_t)(lv.row0 + ic) * kAttnHeadDim;
  const __nv_bfloat16* vself = a.vself ? a.vself + ((size_t)ic * a.KV + kh) * kAttnHeadDim
                                       : Vh + (size_t)(lv.row0 + ic) * kAttnHeadDim;
  uint32_t q1[8][4];
  const __nv_bfloat16* qr = a.q + (size_t)ic * a.q_stride + h * kAttnHeadDim;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    q1[kk][0] = (valid && g == 0) ? ld_b32(qr + 16 * kk + 2 * tig) : 0u;
    q1[kk][1] = 0u;
    q1[kk][2] = (valid && g == 0) ? ld_b32(qr + 16 * kk + 8 + 2 * tig) : 0u;
    q1[kk][3] = 0u;
  }
  float M = -INFINITY, L = 0.f;
  float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
  if (valid) {
    const float* po = a.po + pbase * kAttnHeadDim + 4 * lane;
    float4 nxt = c_start > 0 ? __ldcg(reinterpret_cast<const float4*>(po)) : O;
    for (int c = 0; c < c_start; ++c) {
      if (c > 0 && (c & 31) == 0) {
        pm_l = c + lane < c_start ? __ldcg(a.pm + pbase + c + lane) : -INFINITY;
        pl_l = c + lane < c_start ? __ldcg(a.pl + pbase + c + lane) : 0.f;
      }
      const float4 cur = nxt;
      if (c + 1 < c_start) nxt = __ldcg(reinterpret_cast<const float4*>(po + (size_t)(c + 1) * kAttnHeadDim));
      float sa, sb;
      merge_scale(M, L, __shfl_sync(0xffffffffu, pm_l, c & 31), __shfl_sync(0xffffffffu, pl_l, c & 31), sa, sb);
      O.x = merge_val(O.x, cur.x, sa, sb);
      O.y = merge_val(O.y, cur.y, sa, sb);
      O.z = merge_val(O.z, cur.z, sa, sb);
      O.w = merge_val(O.w, cur.w, sa, sb);
    }
  }
  const int c_end = (T + kAttnChunk - 1) / kAttnChunk;
  const int part = lane & 15, rsub = lane >> 4;
  for (int c = c_start; c < c_end; ++c) {
    const int j0 = c * kAttnChunk;
    const int np = min(max(P - j0, 0), kAttnChunk);  // prefix rows of this chunk (shared by the CTA)
    const int nt = min(T - j0, kAttnChunk);
    __syncthreads();  // everybody is done with the previous chunk's rows
    for (int e = threadIdx.x; e < np * 16; e += kWarps * 32) {
      const int row = e >> 4, pt = e & 15;
      cp16(sK + row * kPad + pt * 8, Kh + (size_t)(j0 + row) * kAttnHeadDim + pt * 8, 16);
      cp16(sV + row * kPad + pt * 8, Vh + (size_t)(j0 + row) * kAttnHeadDim + pt * 8, 16);
    }
    if (valid) {
      for (int row = np + rsub; row < nt; row += 2) {  // own rows: ancestors, then self
        const int j = j0 + row, o = j - P;
        const bool is_anc = j < P + A;
        const __nv_bfloat16* ks = is_anc ? Kh + (size_t)anc[o] * kAttnHeadDim : kself;
        const __nv_bfloat16* vs = is_anc ? Vh + (size_t)anc[o] * kAttnHeadDim : vself;
        cp16(oK + o * kPad + part * 8, ks + part * 8, 16);
        cp16(oV + o * kPad + part * 8, vs + part * 8, 16);
      }
    }
    cp_wait_all();
    __syncthreads();
    if (!valid) continue;
    auto rowK = [&](int slot) -> const __nv_bfloat16* {
      const int j = j0 + slot;
      return j < P ? sK + slot * kPad : (j < T ? oK + (j - P) * kPad : zrow);
    };
    auto rowV = [&](int slot) -> const __nv_bfloat16* {
      const int j = j0 + slot;
      return j < P ? sV + slot * kPad : (j < T ? oV + (j - P) * kPad : zrow);
    };
    const int lim[2] = {g == 0 ? nt : 0, 0};
    float s[8][4], m[2], l[2], o[16][4];
    uint32_t pa[4][4];
    tile_qk_rows(q1, rowK, s, lane);
    chunk_softmax(s, lim, a.scale, m, l, pa, lane);
    chunk_pv_rows(pa, rowV, o, lane);
    if (g == 0) {
#pragma unroll
      for (int nd = 0; nd < 16; ++nd)
        *reinterpret_cast<float2*>(xo + nd * 8 + 2 * tig) = make_float2(o[nd][0], o[nd][1]);
    }
    __syncwarp();
    const float4 oc = *reinterpret_cast<const float4*>(xo + 4 * lane);
    __syncwarp();
    float sa, sb;
    merge_scale(M, L, __shfl_sync(0xffffffffu, m[0], 0), __shfl_sync(0xffffffffu, l[0], 0), sa, sb);
    O.x = merge_val(O.x, oc.x, sa, sb);
    O.y = merge_val(O.y, oc.y, sa, sb);
    O.z = merge_val(O.z, oc.z, sa, sb);
    O.w = merge_val(O.w, oc.w, sa, sb);
  }
  if (!valid) return;
  __nv_bfloat16* out = a.out + (size_t)i * a.out_stride + h * kAttnHeadDim + 4 * lane;
  uint2 u;
  u.x = pack_f32(__fdiv_rn(O.x, L), __fdiv_rn(O.y, L));
  u.y = pack_f32(__fdiv_rn(O.z, L), __fdiv_rn(O.w, L));
  *reinterpret_cast<uint2*>(out) = u;
}


// ---------------------------------------------------------------------------
// Per-node tail for GQA (H/KV >= 4, e.g. the 70B shape): one CTA per (node, KV
// head) with one warp per query head of the group.  The node's chunk rows
// (prefix tail, ancestors, self, zeros) are staged ONCE for the whole group;
// each warp runs the node's row-0 MMAs with its own query — the same
// fragments and order as the per-node kernel, hence the same bits.
constexpr int kGqaWarps = 8;
constexpr size_t kTailGqaSmem = (size_t)2 * kTileElems * 2 + (size_t)kGqaWarps * 128 * 4;

__global__ void __launch_bounds__(kGqaWarps * 32, 2) attn_tail_gqa_kernel(const __grid_constant__ AttnGroup G) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t dsm[];
  const int gi = member_of(G, blockIdx.x, 4);
  const AttnArgs& a = G.m[gi].a;
  const LevelDev& lv = G.m[gi].lv;
  const int local = blockIdx.x - G.m[gi].cta_gqa;
  const int kh = local % a.KV, i = local / a.KV;
  const int grp = a.H / a.KV;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const bool active = warp < grp;
  const int h = kh * grp + (active ? warp : 0);
  __nv_bfloat16* sK = reinterpret_cast<__nv_bfloat16*>(dsm);
  __nv_bfloat16* sV = sK + kTileElems;
  float* xo = reinterpret_cast<float*>(sV + kTileElems) + warp * 128;
  const __nv_bfloat16* Kh = a.k + (size_t)kh * a.cap * kAttnHeadDim;
  const __nv_bfloat16* Vh = a.v + (size_t)kh * a.cap * kAttnHeadDim;
  const int c_start = G.m[gi].c_shared;
  const size_t pbase = part_idx(a, i, h, 0);
  float pm_l = -INFINITY, pl_l = 0.f;
  if (active && lane < c_start) {
    pm_l = __ldcg(a.pm + pbase + lane);
    pl_l = __ldcg(a.pl + pbase + lane);
  }
  const int A = lv.anc_cnt[i];
  const int32_t* anc = lv.anc_rows + (size_t)i * lv.anc_stride;
  const int P = lv.prefix_rows[i];
  const int T = P + A + 1;
  const __nv_bfloat16* kself = a.kself ? a.kself + ((size_t)i * a.KV + kh) * kAttnHeadDim
                                       : Kh + (size_t)(lv.row0 + i) * kAttnHeadDim;
  const __nv_bfloat16* vself = a.vself ? a.vself + ((size_t)i * a.KV + kh) * kAttnHeadDim
                                       : Vh + (size_t)(lv.row0 + i) * kAttnHeadDim;
  uint32_t q1[8][4];
  const __nv_bfloat16* qr = a.q + (size_t)i * a.q_stride + h * kAttnHeadDim;
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    q1[kk][0] = (active && g == 0) ? ld_b32(qr + 16 * kk + 2 * tig) : 0u;
    q1[kk][1] = 0u;
    q1[kk][2] = (active && g == 0) ? ld_b32(qr + 16 * kk + 8 + 2 * tig) : 0u;
    q1[kk][3] = 0u;
  }
  float M = -INFINITY, L = 0.f;
  float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
  if (active) {
    const float* po = a.po + pbase * kAttnHeadDim + 4 * lane;
    float4 nxt = c_start > 0 ? __ldcg(reinterpret_cast<const float4*>(po)) : O;
    for (int c = 0; c < c_start; ++c) {
      if (c > 0 && (c & 31) == 0) {
        pm_l = c + lane < c_start ? __ldcg(a.pm + pbase + c + lane) : -INFINITY;
        pl_l = c + lane < c_start ? __ldcg(a.pl + pbase + c + lane) : 0.f;
      }
      const float4 cur = nxt;
      if (c + 1 < c_start) nxt = __ldcg(reinterpret_cast<const float4*>(po + (size_t)(c + 1) * kAttnHeadDim));
      float sa, sb;
      merge_scale(M, L, __shfl_sync(0xffffffffu, pm_l, c & 31), __shfl_sync(0xffffffffu, pl_l, c & 31), sa, sb);
      O.x = merge_val(O.x, cur.x, sa, sb);
      O.y = merge_val(O.y, cur.y, sa, sb);
      O.z = merge_val(O.z, cur.z, sa, sb);
      O.w = merge_val(O.w, cur.w, sa, sb);
    }
  }
  const int c_end = (T + kAttnChunk - 1) / kAttnChunk;
  for (int c = c_start; c < c_end; ++c) {
    const int j0 = c * kAttnChunk;
    __syncthreads();  // every warp is done with the previous chunk's rows
    for (int e = threadIdx.x; e < kAttnChunk * 16; e += kGqaWarps * 32) {
      const int row = e >> 4, part = e & 15, j = j0 + row;
      const __nv_bfloat16* ks = j < P ? Kh + (size_t)j * kAttnHeadDim
                                      : (j < P + A ? Kh + (size_t)anc[j - P] * kAttnHeadDim : kself);
      const __nv_bfloat16* vs = j < P ? Vh + (size_t)j * kAttnHeadDim
                                      : (j < P + A ? Vh + (size_t)anc[j - P] * kAttnHeadDim : vself);
      const int nb = j < T ? 16 : 0;
      cp16(sK + row * kPad + part * 8, (nb ? ks : Kh) + part * 8, nb);
      cp16(sV + row * kPad + part * 8, (nb ? vs : Vh) + part * 8, nb);
    }
    cp_wait_all();
    __syncthreads();
    if (!active) continue;
    const int lim[2] = {g == 0 ? min(T - j0, kAttnChunk) : 0, 0};
    float m[2], l[2], o[16][4];
    uint32_t pa[4][4];
    chunk_scores(q1, sK, lim, a.scale, m, l, pa, lane);
    chunk_pv(pa, sV, o, lane);
    if (g == 0) {
#pragma unroll
      for (int nd = 0; nd < 16; ++nd)
        *reinterpret_cast<float2*>(xo + nd * 8 + 2 * tig) = make_float2(o[nd][0], o[nd][1]);
    }
    __syncwarp();
    const float4 oc = *reinterpret_cast<const float4*>(xo + 4 * lane);
    __syncwarp();
    float sa, sb;
    merge_scale(M, L, __shfl_sync(0xffffffffu, m[0], 0), __shfl_sync(0xffffffffu, l[0], 0), sa, sb);
    O.x = merge_val(O.x, oc.x, sa, sb);
    O.y = merge_val(O.y, oc.y, sa, sb);
    O.z = merge_val(O.z, oc.z, sa, sb);
    O.w = merge_val(O.w, oc.w, sa, sb);
  }
  if (!active) return;
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
  int cs = 0, ct = 0, cg = 0, c2 = 0, cq = 0;
  for (int g = 0; g < count; ++g) {
    AttnMember& m = G.m[g];
    m.a = a[g];
    m.lv = lv[g];
    m.c_shared = lv[g].min_p / kAttnChunk;
    m.zt = (lv[g].n + kCtaNodes - 1) / kCtaNodes;
    const int c_max = (lv[g].max_t + kAttnChunk - 1) / kAttnChunk;
    TP_CHECK(c_max <= a[g].max_chunks, TP_ESHAPE, "attention chunks exceed scratch");
    const bool tiled = g_attn_tile && lv[g].uniform_a >= 0 && lv[g].uniform_a + 1 <= kTileOwn && lv[g].n >= 4;
    const bool tail2 = !tiled && g_attn_tail2 && lv[g].uniform_a >= 0 && lv[g].uniform_a + 1 <= kOwnMax &&
                       lv[g].n >= 2;
    m.cta_shared = cs;
    m.cta_tail = ct;
    m.cta_tile = cg;
    m.cta_tail2 = c2;
    m.cta_gqa = cq;
    const int grp = a[g].H / a[g].KV;
    const bool gqa = !tiled && !tail2 && grp >= 4 && grp <= kGqaWarps;
    cs += a[g].KV * ((m.c_shared + g_shared_run - 1) / g_shared_run) * m.zt;
    if (tiled)
      cg += a[g].H * m.zt;
    else if (tail2)
      c2 += a[g].H * ((lv[g].n + kWarps - 1) / kWarps);
    else if (gqa)
      cq += a[g].KV * lv[g].n;
    else
      ct += a[g].H * ((lv[g].n + kWarps - 1) / kWarps);
  }
  G.ctas_shared = cs;
  G.ctas_tail = ct;
  G.ctas_tile = cg;
  G.ctas_tail2 = c2;
  static bool attr_set[64] = {false};  // per device
  int dev = 0;
  TP_CUDA(cudaGetDevice(&dev));
  if (!attr_set[dev & 63]) {
    TP_CUDA(cudaFuncSetAttribute(attn_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTailSmem));
    TP_CUDA(cudaFuncSetAttribute(attn_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTileSmem));
    TP_CUDA(cudaFuncSetAttribute(attn_shared_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSharedSmem));
    TP_CUDA(cudaFuncSetAttribute(attn_tail2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTail2Smem));
    TP_CUDA(cudaFuncSetAttribute(attn_tail_gqa_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kTailGqaSmem));
    attr_set[dev & 63] = true;
  }
  if (cs > 0) {
    const size_t smem = (g_shared_run > 1 ? 2 : 1) * (size_t)2 * kTileElems * 2;
    ::tp::count_launch();
    TP_CUDA(launch_pdl(attn_shared_kernel, dim3(cs), dim3(kWarps * 32), smem, st, G, g_shared_run));
    TP_CUDA(cudaGetLastError());
    timeline_mark("attn_shared", st);
  }
  if (cg > 0) {
    ::tp::count_launch();
    TP_CUDA(launch_pdl(attn_tile_kernel, dim3(cg), dim3(kWarps * 32), kTileSmem, st, G));
    TP_CUDA(cudaGetLastError());
    timeline_mark("attn_tile", st);
  }
  if (cq > 0) {
    ::tp::count_launch();
    TP_CUDA(launch_pdl(attn_tail_gqa_kernel, dim3(cq), dim3(kGqaWarps * 32), kTailGqaSmem, st, G));
    TP_CUDA(cudaGetLastError());
    timeline_mark("attn_tail_gqa", st);
  }
  if (c2 > 0) {
    ::tp::count_launch();
    TP_CUDA(launch_pdl(attn_tail2_kernel, dim3(c2), dim3(kWarps * 32), kTail2Smem, st, G));
    TP_CUDA(cudaGetLastError());
    timeline_mark("attn_tail2", st);
  }
  if (ct > 0) {
    ::tp::count_launch();
    TP_CUDA(launch_pdl(attn_tail_kernel, dim3(ct), dim3(kWarps * 32), kTailSmem, st, G,
                       (cs + cg + cq + c2) > 0 ? 1 : 0));
    TP_CUDA(cudaGetLastError());
    timeline_mark("attn_tail", st);
  }
  return TP_OK;
}

int attn_tree(const AttnArgs& a, const LevelDev& lv, cudaStream_t st) { return attn_tree_group(&a, &lv, 1, st); }

void attn_set_tile(bool on) { g_attn_tile = on; }
void attn_set_tail2(bool on) { g_attn_tail2 = on; }
void attn_set_shared_run(int n) { g_shared_run = n < 1 ? 1 : (n > kSharedRunMax ? kSharedRunMax : n); }

}  // namespace tp
