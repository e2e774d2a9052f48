// K1: tree-masked attention of a level's nodes against one stage's KV cache
// (Llama path; replaces the gather + softmax + PV of the reference
// layer_step, `/root/reference/pkg/src/treepipe/model.py:157-167,265-276`).
//
// Node i attends its *logical* key sequence: cache rows [0, P_i) (verified
// prefix), then its speculative ancestors in row order (the set bits of its
// packed ancestor row, decoded on the host), then itself.  The sequence is cut
// into canonical 64-slot chunks (slot = logical position mod 64) and the
// chunks into canonical runs of kRun chunks (run = chunk / kRun).  Each chunk
// yields a partial (max, sum, unnormalised P.V) from one m16n8k16 bf16
// tensor-core pass over a padded shared-memory tile (ldmatrix fragments); a
// run's state is the in-order online merge of its chunks' partials starting
// from the empty state, and the node's result the in-order merge of its runs'
// states.  Two launches per layer slot, each covering every stage of the group:
//   attn_shared_kernel  chunks inside every node's verified prefix
//                       (c < c_shared = floor(min_i P_i / 64)): one CTA per
//                       (member, KV head, run, block of 64 (query head, node)
//                       rows) streams the run's K/V chunks (cp.async double
//                       buffer), each staged once for all rows, and writes the
//                       run state (for the run holding c_shared, the state
//                       after chunk c_shared - 1);
//   attn_tail_kernel    one warp per (node, head): its own chunks (prefix tail,
//                       ancestors, self) in row 0 of the MMA tile — the ones
//                       it can, before griddepcontrol.wait — then the ordered
//                       merge of the shared runs' states and its own chunks;
//   attn_tail_gqa_kernel the tail for GQA (H/KV >= 4): one CTA per (node, KV
//                       head), the chunk rows staged once for the query group.
//
// Batch invariance: the arithmetic applied to a node depends only on its own
// logical key sequence — never on its launch-mates, on where its keys live
// (prefix vs speculative rows) or on which kernel handled a chunk (both run
// the same chunk code on the same smem tile layout; tensor-core rows are
// independent; merges use explicitly rounded ops so the compiler cannot
// contract them differently at the merge sites; a run started in the shared
// kernel and continued in the tail goes through the same merge sequence).  A
// node computed inside a 64-node tree level is therefore bit-identical to the
// same position decoded alone (GPU pipeline == GPU greedy decode).
#include <type_traits>

#include "attn.h"
#include "gemm_tc.h"

namespace tp {

#ifndef TP_TAIL_MINB
#define TP_TAIL_MINB 3
#endif
#ifndef TP_SHARED_MINB
#define TP_SHARED_MINB 3
#endif
constexpr int kPad = 136;  // bf16 per staged row: 128 + 8 pad (conflict-free ldmatrix)
constexpr int kWarps = 4;
constexpr int kTileElems = kAttnChunk * kPad;
constexpr size_t kTailSmem = (size_t)kWarps * (kTileElems * 2 + 128 * 4);  // per warp: chunk tile + hand-over row

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
constexpr int kCtaRows = 64;   // (query head, node) rows per shared CTA: one 16-row MMA tile per warp
constexpr size_t kSharedSmem = (size_t)4 * kTileElems * 2;  // 2 x (K, V) chunk tiles

// Ordered merge of the shared kernel's run states for (node i, head h) into the
// lane-layout state (M, L, O): runs wholly below c_start are merged; the state
// of the run holding c_start (the shared kernel's state after chunk
// c_start - 1; empty when c_start is a run boundary) is returned in (PM, PL, PO)
// for the caller to continue with the node's own chunks.  States are loaded 8
// per L2 round trip.
__device__ __forceinline__ void merge_shared_runs(const AttnArgs& a, int i, int h, int c_start, int kRun, int lane,
                                                  float& M, float& L, float4& O, float& PM, float& PL, float4& PO) {
  constexpr int kPre = 8;
  const int nfull = c_start / kRun;
  const int nst = nfull + (c_start % kRun ? 1 : 0);
  const size_t pbase = part_idx(a, i, h, 0);
  const float4* po = reinterpret_cast<const float4*>(a.po + pbase * kAttnHeadDim) + lane;
  PM = -INFINITY;
  PL = 0.f;
  PO = make_float4(0.f, 0.f, 0.f, 0.f);
  float pm_l = -INFINITY, pl_l = 0.f;  // lane r holds run r0 + r's (max, sum)
  for (int r0 = 0; r0 < nst; r0 += kPre) {
    if ((r0 & 31) == 0) {
      pm_l = r0 + lane < nst ? __ldcg(a.pm + pbase + r0 + lane) : -INFINITY;
      pl_l = r0 + lane < nst ? __ldcg(a.pl + pbase + r0 + lane) : 0.f;
    }
    float4 blk[kPre];
#pragma unroll
    for (int j = 0; j < kPre; ++j) blk[j] = r0 + j < nst ? __ldcg(po + (size_t)(r0 + j) * (kAttnHeadDim / 4)) : PO;
#pragma unroll
    for (int j = 0; j < kPre; ++j) {
      const int r = r0 + j;
      if (r >= nst) break;
      const float mr = __shfl_sync(0xffffffffu, pm_l, r & 31), lr = __shfl_sync(0xffffffffu, pl_l, r & 31);
      if (r < nfull) {
        merge_lane(M, L, O, mr, lr, blk[j]);
      } else {
        PM = mr;
        PL = lr;
        PO = blk[j];
      }
    }
  }
}

// A node's own chunks continue the run holding c_start, then open new runs;
// each finished run is merged into the node state.
struct OwnRuns {
  float CM, CL;
  float4 CO;
  int cur, run;
  __device__ __forceinline__ void add(int c, float mc, float lc, float4 oc, float& M, float& L, float4& O) {
    if (c / run != cur) {
      merge_lane(M, L, O, CM, CL, CO);
      CM = -INFINITY;
      CL = 0.f;
      CO = make_float4(0.f, 0.f, 0.f, 0.f);
      cur = c / run;
    }
    merge_lane(CM, CL, CO, mc, lc, oc);
  }
};

// Shared runs of a member with few rows (<= kSmallRows (query head, node)
// pairs, e.g. the lone verification node): one CTA per (member, KV head, run,
// 16-row tile) with warp w computing chunk w of the run (run <= kWarps), its
// partial handed over through smem and the run state merged in chunk order —
// the same chunk arithmetic and merge sequence as the row-parallel path, with
// the run's chunks in parallel instead of one after another.
constexpr int kSmallRows = 32;
constexpr int kXsLd = 132;  // floats per hand-over row

__device__ __forceinline__ void shared_small(const AttnGroup& G, int gi, int local, uint8_t* dsm) {
  const AttnArgs& a = G.m[gi].a;
  const LevelDev& lv = G.m[gi].lv;
  const int c_shared = G.m[gi].c_shared, R = G.run;
  const int runs = (c_shared + R - 1) / R;
  const int kh = local % a.KV;
  local /= a.KV;
  const int r = local % runs, t = local / runs;
  const int grp = a.H / a.KV;
  const int n = lv.n, rows = n * grp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int nw = min(R, c_shared - r * R);  // chunks of this run below c_shared
  __nv_bfloat16* buf = reinterpret_cast<__nv_bfloat16*>(dsm) + (size_t)warp * kTileElems;
  float* xs = reinterpret_cast<float*>(buf);  // [16][kXsLd] partial, then 16 max + 16 sum
  if (warp < nw) {
    const int c = r * R + warp;
    const int ra = 16 * t + g, rb = ra + 8;
    const bool va = ra < rows, vb = rb < rows;
    const int ia = va ? ra % n : 0, ib = vb ? rb % n : 0;
    const int ha = kh * grp + (va ? ra / n : 0), hb = kh * grp + (vb ? rb / n : 0);
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
    auto stage = [&](const __nv_bfloat16* plane) {
      const __nv_bfloat16* src = plane + ((size_t)kh * a.cap + (size_t)c * kAttnChunk) * kAttnHeadDim;
      for (int e = lane; e < kAttnChunk * 16; e += 32) {
        const int row = e >> 4, part = e & 15;
        cp16(buf + row * kPad + part * 8, src + row * kAttnHeadDim + part * 8, 16);
      }
      cp_wait_all();
      __syncwarp();
    };
    stage(a.k);
    const int lim[2] = {va ? kAttnChunk : 0, vb ? kAttnChunk : 0};
    float m[2], l[2];
    uint32_t pa[4][4];
    chunk_scores(qa, buf, lim, a.scale, m, l, pa, lane);
    __syncwarp();
    stage(a.v);
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
    const float* xw = reinterpret_cast<const float*>(reinterpret_cast<const __nv_bfloat16*>(dsm) + (size_t)w * kTileElems);
    float sa, sb;
    merge_scale(M, L, xw[16 * kXsLd + row], xw[16 * kXsLd + 16 + row], sa, sb);
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
// streams the run's chunks below c_shared (chunk c + 1 staged by cp.async while
// chunk c computes), each K/V chunk staged once for every row, merges them in
// order into the rows' run states (fragment layout, the same scalar merge ops
// as merge_lane) and writes the states.
__global__ void __launch_bounds__(kWarps * 32, TP_SHARED_MINB) attn_shared_kernel(const __grid_constant__ AttnGroup G) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) uint8_t dsm[];
  const int gi = member_of(G, blockIdx.x, 0);
  if (G.m[gi].small) {
    shared_small(G, gi, blockIdx.x - G.m[gi].cta_shared, dsm);
    return;
  }
  const AttnArgs& a = G.m[gi].a;
  const LevelDev& lv = G.m[gi].lv;
  const int c_shared = G.m[gi].c_shared;
  const int kRun = G.run;
  const int runs = (c_shared + kRun - 1) / kRun;
  int local = blockIdx.x - G.m[gi].cta_shared;
  const int kh = local % a.KV;
  local /= a.KV;
  const int r = local % runs, blk = local / runs;
  const int grp = a.H / a.KV;
  const int npc = kCtaRows / grp;  // nodes per CTA
  const int base = blk * npc;
  const int c0 = r * kRun, c1 = min(c_shared, c0 + kRun);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int nreal = min(npc, lv.n - base);
  const int rows = nreal * grp;  // (query head, node) pairs, head-major
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
  const int ra = 16 * warp + g, rb = ra + 8;
  const bool busy = 16 * warp < rows;
  const bool va = ra < rows, vb = rb < rows;
  const int ia = base + (va ? ra % nreal : 0), ib = base + (vb ? rb % nreal : 0);
  const int ha = kh * grp + (va ? ra / nreal : 0), hb = kh * grp + (vb ? rb / nreal : 0);
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
  const int lim[2] = {va ? kAttnChunk : 0, vb ? kAttnChunk : 0};
  float M[2] = {-INFINITY, -INFINITY}, L[2] = {0.f, 0.f};
  float O[16][4];
#pragma unroll
  for (int nd = 0; nd < 16; ++nd) O[nd][0] = O[nd][1] = O[nd][2] = O[nd][3] = 0.f;
  for (int c = c0; c < c1; ++c) {
    const int buf = (c - c0) & 1;
    if (c + 1 < c1) {
      stage(c + 1, buf ^ 1);
      cp_wait_group<1>();
    } else {
      cp_wait_group<0>();
    }
    __syncthreads();
    if (busy) {
      const __nv_bfloat16* sK = smt + (size_t)buf * 2 * kTileElems;
      float m[2], l[2], sa[2], sb[2];
      uint32_t pa[4][4];
      chunk_scores(qa, sK, lim, a.scale, m, l, pa, lane);
      merge_scale(M[0], L[0], m[0], l[0], sa[0], sb[0]);
      merge_scale(M[1], L[1], m[1], l[1], sa[1], sb[1]);
      auto merge_part = [&](auto part_tag) {  // PV a quarter of the dims at a time, merged at once
        constexpr int P = decltype(part_tag)::value;
        float o[4][4];
        chunk_pv_part<P, 4>(pa, sK + kTileElems, o, lane);
#pragma unroll
        for (int nd = 0; nd < 4; ++nd)
#pragma unroll
          for (int e = 0; e < 4; ++e)
            O[4 * P + nd][e] = merge_val(O[4 * P + nd][e], o[nd][e], sa[e >> 1], sb[e >> 1]);
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

// One warp per (node, head): the node's own chunks (prefix tail, ancestors,
// self), then the ordered merge of the shared runs' states and its own
// chunks, then the bf16 output row.  The running state lives in "lane layout"
// (lane l owns dims 4l..4l+3); a chunk computed on the tensor cores (row 0 of
// the tile, fragment layout) is handed over through smem.
//
// `early` (an attention kernel precedes this one in the stream, so the QKV
// GEMM has completed before this grid is launched): up to kEarly own chunks
// are computed BEFORE griddepcontrol.wait, i.e. while the shared-prefix kernel
// is still running; only the merge waits for its run states.  Loads issued
// before the wait bypass L1 (.cg).  Merge order and chunk arithmetic are
// unchanged by it.
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
  float* xo = reinterpret_cast<float*>(reinterpret_cast<__nv_bfloat16*>(dsm) + (size_t)kWarps * kTileElems) +
              warp * 128;  // 128-float hand-over row (its own: PV halves are handed over one at a time)
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
    const int np = min(max(P - j0, 0), kAttnChunk);  // prefix rows in this chunk
    const int nt = min(T - j0, kAttnChunk);          // rows holding keys
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
    float m[2], l[2];
    uint32_t pa[4][4];
    chunk_scores(q1, buf, lim, a.scale, m, l, pa, lane);
    __syncwarp();
    stage(Vh, vself, j0);
    {
      float o[8][4];
      chunk_pv_half<0>(pa, buf, o, lane);
      if (g == 0) {
#pragma unroll
        for (int nd = 0; nd < 8; ++nd) *reinterpret_cast<float2*>(xo + nd * 8 + 2 * tig) = make_float2(o[nd][0], o[nd][1]);
      }
    }
    {
      float o[8][4];
      chunk_pv_half<1>(pa, buf, o, lane);
      if (g == 0) {
#pragma unroll
        for (int nd = 0; nd < 8; ++nd)
          *reinterpret_cast<float2*>(xo + 64 + nd * 8 + 2 * tig) = make_float2(o[nd][0], o[nd][1]);
      }
    }
    __syncwarp();
    oc = *reinterpret_cast<const float4*>(xo + 4 * lane);
    mc = __shfl_sync(0xffffffffu, m[0], 0);
    lc = __shfl_sync(0xffffffffu, l[0], 0);
  };
  const int n_early = early && live ? min(c_end - c_start, kEarly) : 0;
  float em[kEarly], el[kEarly];
  float4 eo[kEarly];
#pragma unroll
  for (int k = 0; k < kEarly; ++k)
    if (k < n_early) run_chunk(c_start + k, em[k], el[k], eo[k]);
  if (early) pdl_wait();  // the shared runs' states are complete from here on
  if (!live) return;
  float M = -INFINITY, L = 0.f;
  float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
  OwnRuns own;
  merge_shared_runs(a, i, h, c_start, G.run, lane, M, L, O, own.CM, own.CL, own.CO);
  own.cur = c_start / G.run;
  own.run = G.run;
#pragma unroll
  for (int k = 0; k < kEarly; ++k)
    if (k < n_early) own.add(c_start + k, em[k], el[k], eo[k], M, L, O);
  for (int c = c_start + n_early; c < c_end; ++c) {
    float mc, lc;
    float4 oc;
    run_chunk(c, mc, lc, oc);
    own.add(c, mc, lc, oc, M, L, O);
  }
  merge_lane(M, L, O, own.CM, own.CL, own.CO);
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
  const int gi = member_of(G, blockIdx.x, 2);
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
  OwnRuns own{-INFINITY, 0.f, make_float4(0.f, 0.f, 0.f, 0.f), c_start / G.run, G.run};
  if (active) merge_shared_runs(a, i, h, c_start, G.run, lane, M, L, O, own.CM, own.CL, own.CO);
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
    float m[2], l[2];
    uint32_t pa[4][4];
    chunk_scores(q1, sK, lim, a.scale, m, l, pa, lane);
    {
      float o[8][4];
      chunk_pv_half<0>(pa, sV, o, lane);
      if (g == 0) {
#pragma unroll
        for (int nd = 0; nd < 8; ++nd) *reinterpret_cast<float2*>(xo + nd * 8 + 2 * tig) = make_float2(o[nd][0], o[nd][1]);
      }
    }
    {
      float o[8][4];
      chunk_pv_half<1>(pa, sV, o, lane);
      if (g == 0) {
#pragma unroll
        for (int nd = 0; nd < 8; ++nd)
          *reinterpret_cast<float2*>(xo + 64 + nd * 8 + 2 * tig) = make_float2(o[nd][0], o[nd][1]);
      }
    }
    __syncwarp();
    const float4 oc = *reinterpret_cast<const float4*>(xo + 4 * lane);
    __syncwarp();
    own.add(c, __shfl_sync(0xffffffffu, m[0], 0), __shfl_sync(0xffffffffu, l[0], 0), oc, M, L, O);
  }
  if (!active) return;
  merge_lane(M, L, O, own.CM, own.CL, own.CO);
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
  int cs = 0, ct = 0, cq = 0;
  for (int g = 0; g < count; ++g) {
    AttnMember& m = G.m[g];
    m.a = a[g];
    m.lv = lv[g];
    const int grp = a[g].H / a[g].KV;
    TP_CHECK(grp >= 1 && kCtaRows % grp == 0, TP_ESHAPE, "query group size must divide 64");
    m.c_shared = lv[g].min_p / kAttnChunk;
    m.small = kRun <= kWarps && lv[g].n * grp <= kSmallRows;
    m.zt = m.small ? (lv[g].n * grp + 15) / 16 : (lv[g].n + kCtaRows / grp - 1) / (kCtaRows / grp);
    const int c_max = (lv[g].max_t + kAttnChunk - 1) / kAttnChunk;
    TP_CHECK(c_max <= a[g].max_chunks, TP_ESHAPE, "attention chunks exceed scratch");
    m.cta_shared = cs;
    m.cta_tail = ct;
    m.cta_gqa = cq;
    cs += a[g].KV * ((m.c_shared + kRun - 1) / kRun) * m.zt;
    if (grp >= 4 && grp <= kGqaWarps)
      cq += a[g].KV * lv[g].n;
    else
      ct += a[g].H * ((lv[g].n + kWarps - 1) / kWarps);
  }
  static bool attr_set[64] = {false};  // per device
  int dev = 0;
  TP_CUDA(cudaGetDevice(&dev));
  if (!attr_set[dev & 63]) {
    TP_CUDA(cudaFuncSetAttribute(attn_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTailSmem));
    TP_CUDA(cudaFuncSetAttribute(attn_shared_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSharedSmem));
    TP_CUDA(cudaFuncSetAttribute(attn_tail_gqa_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kTailGqaSmem));
    attr_set[dev & 63] = true;
  }
  if (cs > 0) {
    ::tp::count_launch();
    TP_CUDA(launch_pdl(attn_shared_kernel, dim3(cs), dim3(kWarps * 32), kSharedSmem, st, G));
    TP_CUDA(cudaGetLastError());
    timeline_mark("attn_shared", st);
  }
  if (cq > 0) {
    ::tp::count_launch();
    TP_CUDA(launch_pdl(attn_tail_gqa_kernel, dim3(cq), dim3(kGqaWarps * 32), kTailGqaSmem, st, G));
    TP_CUDA(cudaGetLastError());
    timeline_mark("attn_tail_gqa", st);
  }
  if (ct > 0) {
    ::tp::count_launch();
    TP_CUDA(launch_pdl(attn_tail_kernel, dim3(ct), dim3(kWarps * 32), kTailSmem, st, G, (cs + cq) > 0 ? 1 : 0));
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
