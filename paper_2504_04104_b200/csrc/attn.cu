// K1: tree-masked attention of a level's nodes against one stage's KV cache
// (Llama path; replaces the gather + softmax + PV of the reference
// layer_step, `/root/reference/pkg/src/treepipe/model.py:157-167,265-276`).
//
// Node i attends its *logical* key sequence: cache rows [0, P_i) (verified
// prefix), then its speculative ancestors in row order (the set bits of its
// packed ancestor row, decoded in registers), then itself.  The sequence is
// cut into canonical 64-slot chunks (slot = logical position mod 64).  Each
// chunk yields a partial (max, sum, unnormalised P.V) from one m16n8k16 bf16
// tensor-core pass, and a combine kernel merges a node's chunk partials in
// order.  Three launches:
//   attn_shared_kernel  chunks entirely inside every node's verified prefix
//                       (c < floor(min_i P_i / 64)): K/V staged once in shared
//                       memory, 4 warps x 16 nodes per CTA, one chunk per CTA;
//   attn_tail_kernel    the remaining chunks of each node (prefix tail +
//                       ancestors + self), one warp per (node, head), the node
//                       in row 0 of the MMA tile, per-lane row pointers;
//   attn_combine_kernel ordered merge, bf16 output.
//
// Batch invariance: the arithmetic applied to a node depends only on its own
// logical key sequence — never on its launch-mates, on where its keys live
// (prefix vs speculative rows) or on which kernel handled a chunk — so a node
// computed inside a 64-node tree level is bit-identical to the same position
// decoded alone (GPU pipeline == GPU greedy decode).  Tensor-core tiles are
// used row-independently: other rows (other nodes or zeros) never change a
// row's result.
#include "attn.h"
#include "gemm_tc.h"

namespace tp {

constexpr int kPad = 136;  // bf16 per staged row: 128 + 8 pad (conflict-free fragment loads)
constexpr int kCtaNodes = 64;
constexpr int kWarps = 4;

__device__ __forceinline__ uint32_t ld_b32(const __nv_bfloat16* p) {
  return *reinterpret_cast<const uint32_t*>(p);
}
__device__ __forceinline__ uint32_t pack_bf16(__nv_bfloat16 lo, __nv_bfloat16 hi) {
  return (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
}
__device__ __forceinline__ uint32_t pack_f32(float lo, float hi) {
  return pack_bf16(__float2bfloat16_rn(lo), __float2bfloat16_rn(hi));
}
__device__ __forceinline__ void mma16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// One canonical 64-slot chunk for the 16-row tile this warp holds, from the
// empty state: returns the chunk max m, sum l and unnormalised o = P.V.
//   qa    : Q A-fragments (8 k-steps over head_dim)
//   krow  : K row of slot nt*8+g, per n-tile
//   vrow  : V rows of slots 16kk + 2tig + {0,1,8,9}
//   lim   : rows g / g+8 see slots [0, lim) of this chunk
__device__ __forceinline__ void chunk_partial(const uint32_t (&qa)[8][4], const __nv_bfloat16* const (&krow)[8],
                                              const __nv_bfloat16* const (&vrow)[4][4], const int (&lim)[2],
                                              float scale, float (&m)[2], float (&l)[2], float (&o)[16][4],
                                              int lane) {
  const int g = lane >> 2, tig = lane & 3;
  float s[8][4];
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t b0 = ld_b32(krow[nt] + 16 * kk + 2 * tig);
      const uint32_t b1 = ld_b32(krow[nt] + 16 * kk + 8 + 2 * tig);
      mma16816(s[nt], qa[kk], b0, b1);
    }
  }
  float mc[2] = {-INFINITY, -INFINITY};
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int slot = nt * 8 + 2 * tig + (e & 1);
      const float v = slot < lim[e >> 1] ? s[nt][e] * scale : -INFINITY;
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
      const float p = s[nt][e] == -INFINITY ? 0.f : expf(s[nt][e] - mc[h]);
      s[nt][e] = p;
      rs[h] += p;
    }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    rs[h] += __shfl_xor_sync(0xffffffffu, rs[h], 1);
    rs[h] += __shfl_xor_sync(0xffffffffu, rs[h], 2);
    l[h] = rs[h];
    m[h] = mc[h];
  }
  uint32_t pa[4][4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    pa[kk][0] = pack_f32(s[2 * kk][0], s[2 * kk][1]);
    pa[kk][1] = pack_f32(s[2 * kk][2], s[2 * kk][3]);
    pa[kk][2] = pack_f32(s[2 * kk + 1][0], s[2 * kk + 1][1]);
    pa[kk][3] = pack_f32(s[2 * kk + 1][2], s[2 * kk + 1][3]);
  }
#pragma unroll
  for (int nd = 0; nd < 16; ++nd) {
    o[nd][0] = o[nd][1] = o[nd][2] = o[nd][3] = 0.f;
    const int col = nd * 8 + g;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t b0 = pack_bf16(vrow[kk][0][col], vrow[kk][1][col]);
      const uint32_t b1 = pack_bf16(vrow[kk][2][col], vrow[kk][3][col]);
      mma16816(o[nd], pa[kk], b0, b1);
    }
  }
}

__device__ __forceinline__ size_t part_idx(const AttnArgs& a, int node, int h, int c) {
  return ((size_t)node * a.H + h) * a.max_chunks + c;
}

// Store one row's chunk partial held in fragment layout (row half `hh` of lanes with group g).
__device__ __forceinline__ void store_row(const AttnArgs& a, size_t idx, const float (&o)[16][4], int hh, float m,
                                          float l, int tig) {
  float* po = a.po + idx * kAttnHeadDim;
#pragma unroll
  for (int nd = 0; nd < 16; ++nd)
    *reinterpret_cast<float2*>(po + nd * 8 + 2 * tig) = make_float2(o[nd][2 * hh], o[nd][2 * hh + 1]);
  if (tig == 0) {
    a.pm[idx] = m;
    a.pl[idx] = l;
  }
}

struct SharedSmem {
  __nv_bfloat16 k[kAttnChunk][kPad];
  __nv_bfloat16 v[kAttnChunk][kPad];
};

// Chunks inside every node's verified prefix: rows [64c, 64c+64) for all nodes.
__global__ void __launch_bounds__(kWarps * 32) attn_shared_kernel(AttnArgs a, LevelDev lv) {
  __shared__ __align__(16) SharedSmem S;
  const int h = blockIdx.x, c = blockIdx.y, base = blockIdx.z * kCtaNodes;
  const int kh = h / (a.H / a.KV);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int nreal = min(kCtaNodes, lv.n - base);
  const int j0 = c * kAttnChunk;
  const __nv_bfloat16* Kh = a.k + ((size_t)kh * a.cap + j0) * kAttnHeadDim;
  const __nv_bfloat16* Vh = a.v + ((size_t)kh * a.cap + j0) * kAttnHeadDim;
  for (int e = threadIdx.x; e < kAttnChunk * 16; e += blockDim.x) {
    const int row = e >> 4, part = e & 15;
    reinterpret_cast<uint4*>(&S.k[row][0])[part] = reinterpret_cast<const uint4*>(Kh + row * kAttnHeadDim)[part];
    reinterpret_cast<uint4*>(&S.v[row][0])[part] = reinterpret_cast<const uint4*>(Vh + row * kAttnHeadDim)[part];
  }
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
  const __nv_bfloat16* krow[8];
  const __nv_bfloat16* vrow[4][4];
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) krow[nt] = &S.k[nt * 8 + g][0];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    vrow[kk][0] = &S.v[16 * kk + 2 * tig][0];
    vrow[kk][1] = &S.v[16 * kk + 2 * tig + 1][0];
    vrow[kk][2] = &S.v[16 * kk + 8 + 2 * tig][0];
    vrow[kk][3] = &S.v[16 * kk + 9 + 2 * tig][0];
  }
  const int lim[2] = {va ? kAttnChunk : 0, vb ? kAttnChunk : 0};
  float m[2], l[2], o[16][4];
  chunk_partial(qa, krow, vrow, lim, a.scale, m, l, o, lane);
  if (va) store_row(a, part_idx(a, ia, h, c), o, 0, m[0], l[0], tig);
  if (vb) store_row(a, part_idx(a, ib, h, c), o, 1, m[1], l[1], tig);
}

// Remaining chunks of one node (from the first non-shared chunk to its last).
__global__ void __launch_bounds__(kWarps * 32) attn_tail_kernel(AttnArgs a, LevelDev lv, int c_start) {
  __shared__ int extra[kWarps][kAttnMaxExtra];
  __shared__ __align__(16) __nv_bfloat16 zero[kPad];
  const int h = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int i = blockIdx.y * kWarps + warp;
  for (int e = threadIdx.x; e < kPad; e += blockDim.x) zero[e] = __float2bfloat16_rn(0.f);
  __syncthreads();
  if (i >= lv.n) return;
  const int kh = h / (a.H / a.KV);
  const __nv_bfloat16* Kh = a.k + (size_t)kh * a.cap * kAttnHeadDim;
  const __nv_bfloat16* Vh = a.v + (size_t)kh * a.cap * kAttnHeadDim;
  // ancestor bits -> ordered rows (lane 0 decodes; a handful of words)
  int A = 0;
  if (lane == 0) {
    for (int w = 0; w < lv.words; ++w) {
      uint64_t bits = lv.anc[(size_t)i * lv.words + w];
      while (bits && A < kAttnMaxExtra) {
        extra[warp][A++] = lv.bits_base + w * 64 + (__ffsll((long long)bits) - 1);
        bits &= bits - 1;
      }
    }
  }
  A = __shfl_sync(0xffffffffu, A, 0);
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
  const int c_end = (T + kAttnChunk - 1) / kAttnChunk;
  for (int c = c_start; c < c_end; ++c) {
    const int j0 = c * kAttnChunk;
    auto row = [&](bool is_k, int slot) -> const __nv_bfloat16* {
      const int j = j0 + slot;
      if (j >= T) return zero;
      if (j < P) return (is_k ? Kh : Vh) + (size_t)j * kAttnHeadDim;
      if (j < P + A) return (is_k ? Kh : Vh) + (size_t)extra[warp][j - P] * kAttnHeadDim;
      return is_k ? kself : vself;
    };
    const __nv_bfloat16* krow[8];
    const __nv_bfloat16* vrow[4][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) krow[nt] = row(true, nt * 8 + g);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      vrow[kk][0] = row(false, 16 * kk + 2 * tig);
      vrow[kk][1] = row(false, 16 * kk + 2 * tig + 1);
      vrow[kk][2] = row(false, 16 * kk + 8 + 2 * tig);
      vrow[kk][3] = row(false, 16 * kk + 9 + 2 * tig);
    }
    const int lim[2] = {g == 0 ? min(max(T - j0, 0), kAttnChunk) : 0, 0};
    float m[2], l[2], o[16][4];
    chunk_partial(q1, krow, vrow, lim, a.scale, m, l, o, lane);
    if (g == 0) store_row(a, part_idx(a, i, h, c), o, 0, m[0], l[0], tig);
  }
}

__global__ void attn_combine_kernel(AttnArgs a, LevelDev lv) {
  pdl_trigger();  // the O-projection GEMM may start streaming its weights
  const int i = blockIdx.x, h = blockIdx.y, d = threadIdx.x;
  int A = 0;
  for (int w = 0; w < lv.words; ++w) A += __popcll(lv.anc[(size_t)i * lv.words + w]);
  A = min(A, kAttnMaxExtra);
  const int T = lv.prefix_rows[i] + A + 1;
  const int chunks = (T + kAttnChunk - 1) / kAttnChunk;
  float M = -INFINITY, L = 0.f, O = 0.f;
  for (int c = 0; c < chunks; ++c) {
    const size_t idx = part_idx(a, i, h, c);
    const float mc = a.pm[idx];
    if (mc == -INFINITY) continue;
    const float mn = fmaxf(M, mc);
    const float sa = M == -INFINITY ? 0.f : expf(M - mn);
    const float sb = expf(mc - mn);
    L = L * sa + a.pl[idx] * sb;
    O = O * sa + a.po[idx * kAttnHeadDim + d] * sb;
    M = mn;
  }
  a.out[(size_t)i * a.out_stride + h * kAttnHeadDim + d] = __float2bfloat16_rn(O / L);
}

int attn_tree(const AttnArgs& a, const LevelDev& lv, cudaStream_t st) {
  const int c_shared = lv.min_p / kAttnChunk;
  const int c_max = (lv.max_t + kAttnChunk - 1) / kAttnChunk;
  TP_CHECK(c_max <= a.max_chunks, TP_ESHAPE, "attention chunks exceed scratch");
  if (c_shared > 0) {
    dim3 grid(a.H, c_shared, (lv.n + kCtaNodes - 1) / kCtaNodes);
    ::tp::count_launch(), attn_shared_kernel<<<grid, kWarps * 32, 0, st>>>(a, lv);
    TP_CUDA(cudaGetLastError());
  }
  ::tp::count_launch(), attn_tail_kernel<<<dim3(a.H, (lv.n + kWarps - 1) / kWarps), kWarps * 32, 0, st>>>(a, lv, c_shared);
  TP_CUDA(cudaGetLastError());
  ::tp::count_launch(), attn_combine_kernel<<<dim3(lv.n, a.H), kAttnHeadDim, 0, st>>>(a, lv);
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

}  // namespace tp
