// K1: tree-masked attention of a level's nodes against one stage's KV cache
// (Llama path; replaces the gather + softmax + PV of the reference
// layer_step, `/root/reference/pkg/src/treepipe/model.py:157-167,265-276`).
//
// Node i attends its *logical* key sequence: cache rows [0, P_i) (verified
// prefix), then its speculative ancestors in row order (the set bits of its
// packed ancestor row, evaluated in registers at kernel start), then itself.
// The sequence is cut into canonical 64-slot chunks (slot = logical position
// mod 64); each chunk is one m16n8k16 bf16 tensor-core tile pass
// (S = Q K^T, online softmax, O += P V) and chunks are merged in order, four
// per split (256 positions), splits merged in order by a small combine
// kernel.  K/V of a chunk are staged once in shared memory and shared by all
// (up to 64) nodes of the CTA; only ancestor / self rows past the common
// prefix are fetched per node.
//
// Batch invariance: the arithmetic applied to a node depends only on its own
// logical key sequence — never on its launch-mates, on where its ancestors
// live (prefix vs speculative rows) or on how many splits were launched — so a
// node computed inside a 64-node tree level is bit-identical to the same
// position decoded alone (the GPU pipeline is lossless w.r.t. the GPU greedy
// decode).  Tensor-core tiles are used row-independently: rows of other
// nodes (or zero rows) never change a row's result.
#include "attn.h"

namespace tp {

constexpr int kPad = 136;  // bf16 per staged row: 128 + 8 pad (conflict-free fragment loads)
constexpr int kCtaNodes = 64;
constexpr int kWarps = 4;
constexpr int kOPad = 132;

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

// One canonical 64-slot chunk for the 16-row tile this warp holds.
//   qa    : Q A-fragments (8 k-steps over head_dim)
//   krow  : K row of slot nt*8+g, per n-tile
//   vrow  : V rows of slots 16kk + 2tig + {0,1,8,9}
//   lim   : rows g / g+8 see slots [0, lim) of this chunk
__device__ __forceinline__ void chunk_step(const uint32_t (&qa)[8][4], const __nv_bfloat16* const (&krow)[8],
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
  float mn[2], alpha[2], rs[2] = {0.f, 0.f};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    mc[h] = fmaxf(mc[h], __shfl_xor_sync(0xffffffffu, mc[h], 1));
    mc[h] = fmaxf(mc[h], __shfl_xor_sync(0xffffffffu, mc[h], 2));
    mn[h] = fmaxf(m[h], mc[h]);
    alpha[h] = mn[h] == -INFINITY ? 1.f : expf(m[h] - mn[h]);
  }
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int h = e >> 1;
      const float p = s[nt][e] == -INFINITY ? 0.f : expf(s[nt][e] - mn[h]);
      s[nt][e] = p;
      rs[h] += p;
    }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    rs[h] += __shfl_xor_sync(0xffffffffu, rs[h], 1);
    rs[h] += __shfl_xor_sync(0xffffffffu, rs[h], 2);
    l[h] = l[h] * alpha[h] + rs[h];
    m[h] = mn[h];
  }
#pragma unroll
  for (int nd = 0; nd < 16; ++nd) {
    o[nd][0] *= alpha[0];
    o[nd][1] *= alpha[0];
    o[nd][2] *= alpha[1];
    o[nd][3] *= alpha[1];
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
    const int col = nd * 8 + g;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t b0 = pack_bf16(vrow[kk][0][col], vrow[kk][1][col]);
      const uint32_t b1 = pack_bf16(vrow[kk][2][col], vrow[kk][3][col]);
      mma16816(o[nd], pa[kk], b0, b1);
    }
  }
}

struct AttnSmem {
  __nv_bfloat16 k[kAttnChunk][kPad];
  __nv_bfloat16 v[kAttnChunk][kPad];
  __nv_bfloat16 zero[kPad];
  int P[kCtaNodes], A[kCtaNodes], T[kCtaNodes];
  int extra[kCtaNodes][kAttnMaxExtra];
  float sm[kCtaNodes], sl[kCtaNodes];
  float so[kCtaNodes][kOPad];
};

__global__ void __launch_bounds__(kWarps * 32) attn_tree_kernel(AttnArgs a, LevelDev lv) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  AttnSmem& S = *reinterpret_cast<AttnSmem*>(smem_raw);
  const int h = blockIdx.x, split = blockIdx.y, base = blockIdx.z * kCtaNodes;
  const int kh = h / (a.H / a.KV);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int nreal = min(kCtaNodes, lv.n - base);
  const __nv_bfloat16* Kh = a.k + (size_t)kh * a.cap * kAttnHeadDim;
  const __nv_bfloat16* Vh = a.v + (size_t)kh * a.cap * kAttnHeadDim;

  // ---- per-node metadata: ancestor bits -> ordered extra rows ---------------
  for (int r = threadIdx.x; r < kCtaNodes; r += blockDim.x) {
    S.sm[r] = -INFINITY;
    S.sl[r] = 0.f;
    if (r < nreal) {
      const int i = base + r;
      int cnt = 0;
      for (int w = 0; w < lv.words; ++w) {
        uint64_t bits = lv.anc[(size_t)i * lv.words + w];
        while (bits && cnt < kAttnMaxExtra) {
          S.extra[r][cnt++] = lv.bits_base + w * 64 + (__ffsll((long long)bits) - 1);
          bits &= bits - 1;
        }
      }
      S.P[r] = lv.prefix_rows[i];
      S.A[r] = cnt;
      S.T[r] = lv.prefix_rows[i] + cnt + 1;
    } else {
      S.P[r] = 0x3fffffff;
      S.A[r] = 0;
      S.T[r] = 0;
    }
  }
  for (int e = threadIdx.x; e < kCtaNodes * kOPad; e += blockDim.x) (&S.so[0][0])[e] = 0.f;
  for (int e = threadIdx.x; e < kPad; e += blockDim.x) S.zero[e] = __float2bfloat16_rn(0.f);
  __syncthreads();
  int pmin = 0x3fffffff, tmax = 0;
  for (int r = 0; r < nreal; ++r) {
    pmin = min(pmin, S.P[r]);
    tmax = max(tmax, S.T[r]);
  }
  const int ch0 = split * kAttnSplitChunks;
  const int ch1 = min(ch0 + kAttnSplitChunks, (tmax + kAttnChunk - 1) / kAttnChunk);

  // Q fragments of this warp's 16 rows (zero for padding rows)
  const int r0 = warp * 16;
  uint32_t qa[8][4];
  {
    const int ia = base + r0 + g, ib = ia + 8;
    const __nv_bfloat16* qra = a.q + (size_t)ia * a.q_stride + h * kAttnHeadDim;
    const __nv_bfloat16* qrb = a.q + (size_t)ib * a.q_stride + h * kAttnHeadDim;
    const bool va = r0 + g < nreal, vb = r0 + g + 8 < nreal;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      qa[kk][0] = va ? ld_b32(qra + 16 * kk + 2 * tig) : 0u;
      qa[kk][1] = vb ? ld_b32(qrb + 16 * kk + 2 * tig) : 0u;
      qa[kk][2] = va ? ld_b32(qra + 16 * kk + 8 + 2 * tig) : 0u;
      qa[kk][3] = vb ? ld_b32(qrb + 16 * kk + 8 + 2 * tig) : 0u;
    }
  }

  for (int ch = ch0; ch < ch1; ++ch) {
    const int j0 = ch * kAttnChunk;
    __syncthreads();
    // stage cache rows [j0, j0+64) of this kv head (zeros past capacity)
    for (int e = threadIdx.x; e < kAttnChunk * 16; e += blockDim.x) {
      const int row = e >> 4, part = e & 15;
      uint4 kv = make_uint4(0, 0, 0, 0), vv = make_uint4(0, 0, 0, 0);
      if (j0 + row < a.cap) {
        kv = reinterpret_cast<const uint4*>(Kh + (size_t)(j0 + row) * kAttnHeadDim)[part];
        vv = reinterpret_cast<const uint4*>(Vh + (size_t)(j0 + row) * kAttnHeadDim)[part];
      }
      reinterpret_cast<uint4*>(&S.k[row][0])[part] = kv;
      reinterpret_cast<uint4*>(&S.v[row][0])[part] = vv;
    }
    __syncthreads();
    if (j0 + kAttnChunk <= pmin) {
      // shared chunk: every slot is a verified-prefix row for every node
      if (r0 < nreal) {
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
        const int ra = r0 + g, rb = ra + 8;
        int lim[2] = {min(max(S.T[ra] - j0, 0), kAttnChunk), min(max(S.T[rb] - j0, 0), kAttnChunk)};
        float m[2] = {S.sm[ra], S.sm[rb]}, l[2] = {S.sl[ra], S.sl[rb]};
        float o[16][4];
#pragma unroll
        for (int nd = 0; nd < 16; ++nd) {
          o[nd][0] = S.so[ra][nd * 8 + 2 * tig];
          o[nd][1] = S.so[ra][nd * 8 + 2 * tig + 1];
          o[nd][2] = S.so[rb][nd * 8 + 2 * tig];
          o[nd][3] = S.so[rb][nd * 8 + 2 * tig + 1];
        }
        chunk_step(qa, krow, vrow, lim, a.scale, m, l, o, lane);
        __syncwarp();
        if (tig == 0) {
          S.sm[ra] = m[0];
          S.sl[ra] = l[0];
          S.sm[rb] = m[1];
          S.sl[rb] = l[1];
        }
#pragma unroll
        for (int nd = 0; nd < 16; ++nd) {
          S.so[ra][nd * 8 + 2 * tig] = o[nd][0];
          S.so[ra][nd * 8 + 2 * tig + 1] = o[nd][1];
          S.so[rb][nd * 8 + 2 * tig] = o[nd][2];
          S.so[rb][nd * 8 + 2 * tig + 1] = o[nd][3];
        }
      }
    } else {
      // tail chunk: per node, row 0 of the tile, own slot -> row map
      for (int rr = 0; rr < 16; ++rr) {
        const int r = r0 + rr;
        if (r >= nreal) break;
        const int i = base + r;
        const int P = S.P[r], A = S.A[r], T = S.T[r];
        auto kv_row = [&](bool is_k, int slot) -> const __nv_bfloat16* {
          const int j = j0 + slot;
          if (j >= T) return S.zero;
          if (j < P) return is_k ? &S.k[slot][0] : &S.v[slot][0];
          const __nv_bfloat16* cache = is_k ? Kh : Vh;
          if (j < P + A) return cache + (size_t)S.extra[r][j - P] * kAttnHeadDim;
          const __nv_bfloat16* self = is_k ? a.kself : a.vself;
          if (self) return self + ((size_t)i * a.KV + kh) * kAttnHeadDim;
          return cache + (size_t)(lv.row0 + i) * kAttnHeadDim;
        };
        uint32_t q1[8][4];
        const __nv_bfloat16* qr = a.q + (size_t)i * a.q_stride + h * kAttnHeadDim;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          q1[kk][0] = g == 0 ? ld_b32(qr + 16 * kk + 2 * tig) : 0u;
          q1[kk][1] = 0u;
          q1[kk][2] = g == 0 ? ld_b32(qr + 16 * kk + 8 + 2 * tig) : 0u;
          q1[kk][3] = 0u;
        }
        const __nv_bfloat16* krow[8];
        const __nv_bfloat16* vrow[4][4];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) krow[nt] = kv_row(true, nt * 8 + g);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          vrow[kk][0] = kv_row(false, 16 * kk + 2 * tig);
          vrow[kk][1] = kv_row(false, 16 * kk + 2 * tig + 1);
          vrow[kk][2] = kv_row(false, 16 * kk + 8 + 2 * tig);
          vrow[kk][3] = kv_row(false, 16 * kk + 9 + 2 * tig);
        }
        int lim[2] = {g == 0 ? min(max(T - j0, 0), kAttnChunk) : 0, 0};
        float m[2] = {g == 0 ? S.sm[r] : -INFINITY, -INFINITY}, l[2] = {g == 0 ? S.sl[r] : 0.f, 0.f};
        float o[16][4];
#pragma unroll
        for (int nd = 0; nd < 16; ++nd) {
          o[nd][0] = g == 0 ? S.so[r][nd * 8 + 2 * tig] : 0.f;
          o[nd][1] = g == 0 ? S.so[r][nd * 8 + 2 * tig + 1] : 0.f;
          o[nd][2] = o[nd][3] = 0.f;
        }
        chunk_step(q1, krow, vrow, lim, a.scale, m, l, o, lane);
        __syncwarp();
        if (g == 0) {
          if (tig == 0) {
            S.sm[r] = m[0];
            S.sl[r] = l[0];
          }
#pragma unroll
          for (int nd = 0; nd < 16; ++nd) {
            S.so[r][nd * 8 + 2 * tig] = o[nd][0];
            S.so[r][nd * 8 + 2 * tig + 1] = o[nd][1];
          }
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  // split partials
  for (int e = threadIdx.x; e < nreal * kAttnHeadDim; e += blockDim.x) {
    const int r = e / kAttnHeadDim, d = e % kAttnHeadDim;
    const size_t idx = ((size_t)(base + r) * a.H + h) * a.max_splits + split;
    a.po[idx * kAttnHeadDim + d] = S.so[r][d];
    if (d == 0) {
      a.pm[idx] = S.sm[r];
      a.pl[idx] = S.sl[r];
    }
  }
}

__global__ void attn_combine_kernel(AttnArgs a, int n, int splits) {
  const int i = blockIdx.x, h = blockIdx.y, d = threadIdx.x;
  const size_t base = ((size_t)i * a.H + h) * a.max_splits;
  float M = -INFINITY;
  for (int s = 0; s < splits; ++s) M = fmaxf(M, a.pm[base + s]);
  float L = 0.f, O = 0.f;
  for (int s = 0; s < splits; ++s) {
    const float w = a.pm[base + s] == -INFINITY ? 0.f : expf(a.pm[base + s] - M);
    L += a.pl[base + s] * w;
    O += a.po[(base + s) * kAttnHeadDim + d] * w;
  }
  a.out[(size_t)i * a.out_stride + h * kAttnHeadDim + d] = __float2bfloat16_rn(O / L);
}

int attn_tree(const AttnArgs& a, const LevelDev& lv, int splits, cudaStream_t st) {
  TP_CHECK(splits >= 1 && splits <= a.max_splits, TP_ESHAPE, "attention splits exceed scratch");
  const size_t smem = sizeof(AttnSmem);
  static size_t smem_set = 0;
  if (smem > smem_set) {
    TP_CUDA(cudaFuncSetAttribute(attn_tree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    smem_set = smem;
  }
  dim3 grid(a.H, splits, (lv.n + kCtaNodes - 1) / kCtaNodes);
  ::tp::count_launch(), attn_tree_kernel<<<grid, kWarps * 32, smem, st>>>(a, lv);
  TP_CUDA(cudaGetLastError());
  ::tp::count_launch(), attn_combine_kernel<<<dim3(lv.n, a.H), kAttnHeadDim, 0, st>>>(a, lv.n, splits);
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

}  // namespace tp
