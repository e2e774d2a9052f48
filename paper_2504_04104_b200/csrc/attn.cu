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

constexpr int kPad = 136;  // bf16 per staged row: 128 + 8 pad (conflict-free ldmatrix)
constexpr int kCtaNodes = 64;
constexpr int kWarps = 4;
constexpr int kTileElems = kAttnChunk * kPad;
constexpr size_t kTailSmem = (size_t)kWarps * kTileElems * 2 + (size_t)kWarps * (kAttnChunk + kAttnMaxExtra) * 4;

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
__device__ __forceinline__ void chunk_scores(const uint32_t (&qa)[8][4], const __nv_bfloat16* sK,
                                             const int (&lim)[2], float scale, float (&m)[2], float (&l)[2],
                                             uint32_t (&pa)[4][4], int lane) {
  const int tig = lane & 3, mi = lane >> 3, mr = lane & 7;
  float s[8][4];
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
      const float p = s[nt][e] == -INFINITY ? 0.f : expf(__fsub_rn(s[nt][e], mc[h]));
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
  sa = M == -INFINITY ? 0.f : expf(__fsub_rn(M, mn));
  sb = expf(__fsub_rn(mc, mn));
  L = __fmaf_rn(L, sa, __fmul_rn(lc, sb));
  M = mn;
}
__device__ __forceinline__ float merge_val(float O, float oc, float sa, float sb) {
  return __fmaf_rn(O, sa, __fmul_rn(oc, sb));
}

__device__ __forceinline__ size_t part_idx(const AttnArgs& a, int node, int h, int c) {
  return ((size_t)node * a.H + h) * a.max_chunks + c;
}

__device__ __forceinline__ int member_of(const AttnGroup& G, int b, bool tail) {
  int gi = 0;
  while (gi + 1 < G.count && b >= (tail ? G.m[gi + 1].cta_tail : G.m[gi + 1].cta_shared)) ++gi;
  return gi;
}

// Chunks inside every node's verified prefix: rows [64c, 64c+64) for all nodes.
__global__ void __launch_bounds__(kWarps * 32) attn_shared_kernel(const __grid_constant__ AttnGroup G) {
  __shared__ __align__(16) __nv_bfloat16 sK[kTileElems];
  __shared__ __align__(16) __nv_bfloat16 sV[kTileElems];
  const int gi = member_of(G, blockIdx.x, false);
  const AttnArgs& a = G.m[gi].a;
  const LevelDev& lv = G.m[gi].lv;
  int local = blockIdx.x - G.m[gi].cta_shared;
  const int h = local % a.H;
  local /= a.H;
  const int c = local % G.m[gi].c_shared, base = (local / G.m[gi].c_shared) * kCtaNodes;
  const int kh = h / (a.H / a.KV);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int nreal = min(kCtaNodes, lv.n - base);
  const int j0 = c * kAttnChunk;
  const __nv_bfloat16* Kh = a.k + ((size_t)kh * a.cap + j0) * kAttnHeadDim;
  const __nv_bfloat16* Vh = a.v + ((size_t)kh * a.cap + j0) * kAttnHeadDim;
#pragma unroll
  for (int e = threadIdx.x; e < kAttnChunk * 16; e += kWarps * 32) {
    const int row = e >> 4, part = e & 15;
    cp16(sK + row * kPad + part * 8, Kh + row * kAttnHeadDim + part * 8, 16);
    cp16(sV + row * kPad + part * 8, Vh + row * kAttnHeadDim + part * 8, 16);
  }
  cp_wait_all();
  __syncthreads();
  const int r0 = warp * 16;
  if (r0 >= nreal) return;
  const int ia = base + r0 + g, ib = ia + 8;
  const bool va = r0 + g < nreal, vb = r0 + g + 8 < nreal;
  uint32_t qa[8][4];
  {
    const __nv_bfloat16* qra = a.q + (size_t)ia * a.q_stride + h * kAttnHeadDim;
    const __nv_bfloat16* qrb = a.q + (size_t)ib * a.q_stride + h * kAttnHeadDim;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      qa[kk][0] = va ? ld_b32(qra + 16 * kk + 2 * tig) : 0u;
      qa[kk][1] = vb ? ld_b32(qrb + 16 * kk + 2 * tig) : 0u;
      qa[kk][2] = va ? ld_b32(qra + 16 * kk + 8 + 2 * tig) : 0u;
      qa[kk][3] = vb ? ld_b32(qrb + 16 * kk + 8 + 2 * tig) : 0u;
    }
  }
  const int lim[2] = {va ? kAttnChunk : 0, vb ? kAttnChunk : 0};
  float m[2], l[2], o[16][4];
  uint32_t pa[4][4];
  chunk_scores(qa, sK, lim, a.scale, m, l, pa, lane);
  chunk_pv(pa, sV, o, lane);
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    if (!(hh ? vb : va)) continue;
    const size_t idx = part_idx(a, hh ? ib : ia, h, c);
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

// One warp per (node, head): ordered merge of the shared chunks, then the
// node's remaining chunks, then the bf16 output row.  The running state lives
// in "lane layout" (lane l owns dims 4l..4l+3); a chunk computed on the tensor
// cores (row 0 of the tile, fragment layout) is handed over through smem.
__global__ void __launch_bounds__(kWarps * 32) attn_tail_kernel(const __grid_constant__ AttnGroup G) {
  pdl_trigger();  // the O-projection GEMM may start streaming its weights
  extern __shared__ __align__(16) uint8_t dsm[];
  const int gi = member_of(G, blockIdx.x, true);
  const AttnArgs& a = G.m[gi].a;
  const LevelDev& lv = G.m[gi].lv;
  int local = blockIdx.x - G.m[gi].cta_tail;
  const int h = local % a.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int i = (local / a.H) * kWarps + warp;
  if (i >= lv.n) return;
  __nv_bfloat16* buf = reinterpret_cast<__nv_bfloat16*>(dsm) + (size_t)warp * kTileElems;
  int* src = reinterpret_cast<int*>(dsm + (size_t)kWarps * kTileElems * 2) + warp * (kAttnChunk + kAttnMaxExtra);
  int* extra = src + kAttnChunk;
  float* xo = reinterpret_cast<float*>(buf);  // 128-float hand-over row (aliases the tile between chunks)
  const int kh = h / (a.H / a.KV);
  const __nv_bfloat16* Kh = a.k + (size_t)kh * a.cap * kAttnHeadDim;
  const __nv_bfloat16* Vh = a.v + (size_t)kh * a.cap * kAttnHeadDim;
  const int c_start = G.m[gi].c_shared;
  // issue the loads of the first 32 shared chunks' (max, sum) early: lane c holds chunk c
  const size_t pbase = part_idx(a, i, h, 0);
  float pm_l = -INFINITY, pl_l = 0.f;
  if (lane < c_start) {
    pm_l = __ldcg(a.pm + pbase + lane);
    pl_l = __ldcg(a.pl + pbase + lane);
  }
  // ancestor bits -> ordered rows: lane w decodes word w, offsets by a warp scan
  int A = 0;
  for (int w0 = 0; w0 < lv.words; w0 += 32) {
    const int w = w0 + lane;
    const uint64_t bits = w < lv.words ? lv.anc[(size_t)i * lv.words + w] : 0ull;
    const int cnt = __popcll(bits);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int pos = A + incl - cnt;
    uint64_t b = bits;
    while (b && pos < kAttnMaxExtra) {
      extra[pos++] = lv.bits_base + w * 64 + (__ffsll((long long)b) - 1);
      b &= b - 1;
    }
    A += __shfl_sync(0xffffffffu, incl, 31);
  }
  A = min(A, kAttnMaxExtra);
  __syncwarp();
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
    q1[kk][0] = g == 0 ? ld_b32(qr + 16 * kk + 2 * tig) : 0u;
    q1[kk][1] = 0u;
    q1[kk][2] = g == 0 ? ld_b32(qr + 16 * kk + 8 + 2 * tig) : 0u;
    q1[kk][3] = 0u;
  }
  // running state, lane layout: dims 4*lane .. 4*lane+3
  float M = -INFINITY, L = 0.f;
  float4 O = make_float4(0.f, 0.f, 0.f, 0.f);
  {
    const float* po = a.po + pbase * kAttnHeadDim + 4 * lane;
    float4 nxt = c_start > 0 ? __ldcg(reinterpret_cast<const float4*>(po)) : O;
    for (int c = 0; c < c_start; ++c) {
      if (c > 0 && (c & 31) == 0) {  // next block of 32 chunk scalars
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
    __syncwarp();  // previous chunk's hand-over row has been read
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int slot = lane + 32 * u, j = j0 + slot;
      src[slot] = j >= T ? -1 : (j < P ? j : (j < P + A ? extra[j - P] : -2));
    }
    __syncwarp();
    // stage K rows of the chunk: every 16-byte piece in flight at once (empty slots: zeros)
#pragma unroll 8
    for (int e = lane; e < kAttnChunk * 16; e += 32) {
      const int row = e >> 4, part = e & 15, sr = src[row];
      const __nv_bfloat16* g_src = sr == -2 ? kself : Kh + (size_t)max(sr, 0) * kAttnHeadDim;
      cp16(buf + row * kPad + part * 8, g_src + part * 8, sr == -1 ? 0 : 16);
    }
    cp_wait_all();
    __syncwarp();
    const int lim[2] = {g == 0 ? min(T - j0, kAttnChunk) : 0, 0};
    float m[2], l[2], o[16][4];
    uint32_t pa[4][4];
    chunk_scores(q1, buf, lim, a.scale, m, l, pa, lane);
    __syncwarp();
#pragma unroll 8
    for (int e = lane; e < kAttnChunk * 16; e += 32) {
      const int row = e >> 4, part = e & 15, sr = src[row];
      const __nv_bfloat16* g_src = sr == -2 ? vself : Vh + (size_t)max(sr, 0) * kAttnHeadDim;
      cp16(buf + row * kPad + part * 8, g_src + part * 8, sr == -1 ? 0 : 16);
    }
    cp_wait_all();
    __syncwarp();
    chunk_pv(pa, buf, o, lane);
    __syncwarp();  // every lane is done reading the tile: reuse it for the hand-over row
    if (g == 0) {
#pragma unroll
      for (int nd = 0; nd < 16; ++nd)
        *reinterpret_cast<float2*>(xo + nd * 8 + 2 * tig) = make_float2(o[nd][0], o[nd][1]);
    }
    __syncwarp();
    const float4 oc = *reinterpret_cast<const float4*>(xo + 4 * lane);
    float sa, sb;
    merge_scale(M, L, __shfl_sync(0xffffffffu, m[0], 0), __shfl_sync(0xffffffffu, l[0], 0), sa, sb);
    O.x = merge_val(O.x, oc.x, sa, sb);
    O.y = merge_val(O.y, oc.y, sa, sb);
    O.z = merge_val(O.z, oc.z, sa, sb);
    O.w = merge_val(O.w, oc.w, sa, sb);
  }
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
  int cs = 0, ct = 0;
  for (int g = 0; g < count; ++g) {
    AttnMember& m = G.m[g];
    m.a = a[g];
    m.lv = lv[g];
    m.c_shared = lv[g].min_p / kAttnChunk;
    m.zt = (lv[g].n + kCtaNodes - 1) / kCtaNodes;
    const int c_max = (lv[g].max_t + kAttnChunk - 1) / kAttnChunk;
    TP_CHECK(c_max <= a[g].max_chunks, TP_ESHAPE, "attention chunks exceed scratch");
    m.cta_shared = cs;
    m.cta_tail = ct;
    cs += a[g].H * m.c_shared * m.zt;
    ct += a[g].H * ((lv[g].n + kWarps - 1) / kWarps);
  }
  G.ctas_shared = cs;
  G.ctas_tail = ct;
  static bool attr_set[64] = {false};  // per device
  int dev = 0;
  TP_CUDA(cudaGetDevice(&dev));
  if (!attr_set[dev & 63]) {
    TP_CUDA(cudaFuncSetAttribute(attn_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTailSmem));
    attr_set[dev & 63] = true;
  }
  if (cs > 0) {
    ::tp::count_launch(), attn_shared_kernel<<<cs, kWarps * 32, 0, st>>>(G);
    TP_CUDA(cudaGetLastError());
  }
  ::tp::count_launch(), attn_tail_kernel<<<ct, kWarps * 32, kTailSmem, st>>>(G);
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

int attn_tree(const AttnArgs& a, const LevelDev& lv, cudaStream_t st) { return attn_tree_group(&a, &lv, 1, st); }

}  // namespace tp
