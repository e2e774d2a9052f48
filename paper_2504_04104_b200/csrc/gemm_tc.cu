// K2: weight-streaming GEMM on 5th-gen tensor cores (tcgen05 + TMEM + TMA), swap-AB,
// with the split-K reduction and the layer's elementwise epilogue fused in.
//
//   y[node, j] = sum_k X[node, k] * W[j, k]       (W: [N_out, K] bf16, K-major)
//
// A tree level has at most a few dozen nodes, so the *weights* are the MMA's
// M operand (128-row tiles) and the nodes its N operand (n_pad = 16..256
// columns): D^T[128 x n_pad] += W_tile[128 x 64] . X_tile[n_pad x 64]^T, the
// accumulator in TMEM.  The kernel is HBM-bound (arithmetic intensity ~n_pad
// FLOP/B); the design goal is keeping every SM's TMA queue full:
//   * stream-K: the m-tile x k-block space is cut into one contiguous range
//     per CTA (grid = #SMs), so every SM streams the same weight bytes;
//   * warp-specialised: warp 0 = TMA producer (weights evict-first, node rows
//     evict-last), warp 1 = single-thread MMA issuer, warps 2-5 = TMEM drain
//     (up to 4 TMEM accumulator buffers: the next segments' MMAs overlap the
//     previous segment's drain), warps 6-13 = stream-K reducers fed by a
//     shared-memory queue, so a fix-up waiting on other CTAs never stalls the
//     drain (measured: the o-projection lost 16 us of 55 to fix-ups on the
//     drain warps);
//   * programmatic dependent launch: barrier init, TMEM allocation and the
//     first ring-full of *weight* tiles are issued before griddepcontrol.wait,
//     i.e. while the previous kernel is still finishing;
//   * fused fix-up: an m-tile with several contributing CTAs has each write
//     its fp32 partial; the contributors whose ranges *end* inside the tile
//     (they finish together at the end of the kernel) wait for the tile's
//     arrival counter, then each reduces a slice of the nodes in contributor
//     order and applies the epilogue op (RoPE + KV-row scatter, residual add,
//     SwiGLU, or a plain store).  A sole contributor applies it straight from
//     TMEM.  The epilogue runs one warp per node row (lane = 4 features, the
//     RoPE / SwiGLU partner feature is lane^16), two rows in flight per warp.
//   * folded RMSNorm: residual epilogues also write bf16(x) and per-(node,
//     m-tile) sums of squares; the consuming GEMM scales each node's fp32
//     accumulator by r before its op (see GemmEpi in gemm_tc.h);
//   * members of a grouped launch carry their own stream-K plans, so a launch
//     may mix shapes (a draft model's layer next to a target stage's).
// Determinism / batch invariance: segment boundaries depend only on
// (N_out, K, #SMs) of each member; partials are summed in contributor order
// whichever CTA reduces them; each output column's accumulation chain is the
// same for any n.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "gemm_tc.h"
#include "kvpage.cuh"
#include "sm100.cuh"

namespace tp {

using namespace sm100;

constexpr int kBM = 128, kBK = 64;
constexpr int kMaxStages = 16;
constexpr int kMaxTmemBufs = 4;  // accumulator buffers: the MMA may run this many segments ahead
constexpr int kDrainWarps = 4;  // one per TMEM lane quarter: drain accumulators, publish partials, sole-owner epilogue
#ifndef TP_RED_WARPS
#define TP_RED_WARPS 8
#endif
constexpr int kRedWarps = TP_RED_WARPS;  // stream-K fix-up reducers, fed through a shared-memory queue
constexpr int kThreads = 64 + 32 * (kDrainWarps + kRedWarps);
constexpr int kRedSlots = kMaxGroup + 1;  // <= one reduction per member per CTA, plus the end sentinel
constexpr int kBarBytes = 1024;           // mbarriers, TMEM holder, reduction queue
constexpr int kRsBytes = kMaxGroup * 256 * 4;  // per member and node: the folded RMSNorm scale r
struct RedItem {
  int g, mt, cnt, cfirst, clast;
};
constexpr int kABytes = kBM * kBK * 2;  // 16 KB
constexpr int kXchNodes = 32;           // epilogue exchange tile: 32 nodes x 128 features
constexpr int kXchLd = 132;
constexpr int kXchBytes = kXchNodes * kXchLd * 4;

static int g_num_sms = 0;

int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_num_sms;
}

// ---- host: tensor maps -------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

int make_tmap_kmajor(CUtensorMap* map, const void* gptr, int64_t rows, int64_t k, int box_rows) {
  static std::once_flag once;
  std::call_once(once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  TP_CHECK(g_encode, TP_ECUDA, "cuTensorMapEncodeTiled unavailable");
  TP_CHECK(k % kBK == 0, TP_ESHAPE, "GEMM K must be a multiple of 64");
  cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)k * 2};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(gptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  TP_CHECK(r == CUDA_SUCCESS, TP_ECUDA, "cuTensorMapEncodeTiled failed");
  return TP_OK;
}

// Query rows of the attention run kernel: Xq viewed as [nodes][heads][128] bf16,
// box = 64 dims x grp heads x (128 / grp) nodes, 128-byte swizzle (the smem tile
// is then the K-major SW128 A operand with row = node * grp + head).
int make_tmap_q3d(CUtensorMap* map, const void* gptr, int64_t nodes, int heads, int grp) {
  TP_CHECK(g_encode, TP_ECUDA, "cuTensorMapEncodeTiled unavailable (make_tmap_kmajor initialises it)");
  TP_CHECK(grp >= 1 && 128 % grp == 0 && heads % grp == 0, TP_ESHAPE, "query group size must divide 128");
  cuuint64_t dims[3] = {128, (cuuint64_t)heads, (cuuint64_t)nodes};
  cuuint64_t strides[2] = {256, (cuuint64_t)heads * 256};
  cuuint32_t box[3] = {64, (cuuint32_t)grp, (cuuint32_t)(128 / grp)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(gptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  TP_CHECK(r == CUDA_SUCCESS, TP_ECUDA, "cuTensorMapEncodeTiled (3d query map) failed");
  return TP_OK;
}

SkPlan sk_plan(int n_out, int k, int n) {
  SkPlan p;
  p.mtiles = n_out / kBM;
  p.KB = k / kBK;
  p.total = p.mtiles * p.KB;
  p.G = std::min(num_sms(), p.total);
  p.q = p.total / p.G;
  p.r = p.total % p.G;
  int mc = 1;
  for (int mt = 0; mt < p.mtiles; ++mt)
    mc = std::max(mc, sk_cta_of(p, (mt + 1) * p.KB - 1) - sk_cta_of(p, mt * p.KB) + 1);
  p.max_contrib = mc;
  p.n = n;
  p.n_pad = std::max(16, (n + 15) / 16 * 16);
  return p;
}

// Tuning knobs (tp_debug_gemm_knob): ring depth cap and smem budget.
static int g_knob_max_stages = getenv("TP_GEMM_MAX_STAGES") ? atoi(getenv("TP_GEMM_MAX_STAGES")) : 8;
static int g_knob_smem_kb = getenv("TP_GEMM_SMEM_KB") ? atoi(getenv("TP_GEMM_SMEM_KB")) : 200;
static int g_knob_fixup = 0;  // diagnostics only: 1 skips the reduction, 2 also the partial publish, 3 reduces without waiting for arrivals (WRONG results)

static int stages_for(int n_pad) {
  const int per = kABytes + n_pad * 128;
  return std::min(std::min(kMaxStages, g_knob_max_stages),
                  (g_knob_smem_kb * 1024 - kXchBytes - 1024 - kBarBytes - kRsBytes) / per);
}

static size_t smem_for(int n_pad) {
  return (size_t)stages_for(n_pad) * (kABytes + n_pad * 128) + kXchBytes + 1024 /*align*/ + kBarBytes + kRsBytes;
}

// ---- device --------------------------------------------------------------------
// Diagnostics (built with -DTP_GEMM_TRACE): per-CTA globaltimer stamps of the
// kernel's phases into a device buffer set by tp_debug_gemm_trace ([grid][16] u64).
// Launches are numbered in start order (every CTA of launch i starts before any of
// launch i+1: PDL releases a dependent only after all CTAs triggered), so a chain
// of launches lands in consecutive [launch][grid][16] records (kTraceLaunches max).
__device__ unsigned long long* g_gemm_trace = nullptr;
__device__ unsigned int g_gemm_trace_ctr = 0;
constexpr int kTraceLaunches = 64;
#ifdef TP_GEMM_TRACE
__device__ __forceinline__ void gemm_stamp(int slot) {
  unsigned long long* b = g_gemm_trace;
  if (!b) return;
  __shared__ unsigned int s_launch;
  if (slot == 0) s_launch = atomicAdd(&g_gemm_trace_ctr, 1u) / gridDim.x;
  const unsigned int l = s_launch;
  if (l >= kTraceLaunches) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  b[((size_t)l * gridDim.x + blockIdx.x) * 32 + slot] = t;
}
#define GSTAMP(slot) gemm_stamp(slot)
#else
#define GSTAMP(slot) ((void)0)
#endif
__device__ __forceinline__ void drain_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kDrainWarps) : "memory"); }
__device__ __forceinline__ void red_bar() { asm volatile("bar.sync 2, %0;" ::"n"(32 * kRedWarps) : "memory"); }

// ---- epilogue: one warp per node row, lane l owns features 4l..4l+3 of the m-tile.
// RoPE pairs feature r with r^64 and SwiGLU gate r with up r+64: both are lane^16.
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 ld4cg(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ float4 shfl_xor4(float4 v, int m) {
  return make_float4(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m),
                     __shfl_xor_sync(0xffffffffu, v.z, m), __shfl_xor_sync(0xffffffffu, v.w, m));
}
// Operands the op reads besides y (issued for a batch of nodes before any store).
struct EpiAux {
  float4 a, b;
  float r;  // the node's RMSNorm scale (consumers of a folded norm), else 1
};

// A node's RMSNorm scale from the producer's per-m-tile partials, in one fixed
// order (the only place r is ever formed, so this order is the definition): lane l
// sums partials l, l+32, ... in order, then a butterfly over the lanes;
// r = 1/sqrt(ss/d + eps).  Warp-uniform.  (Measured: one warp per node beats one
// thread per node with 8 loads in flight — 1845 vs 1905 us for a lone n=44 forward.)
__device__ __forceinline__ float norm_scale_from_partials(const float* ssp, int n_part, float d, float eps,
                                                          int lane) {
  float s = 0.f;
  for (int i = lane; i < n_part; i += 32) s = __fadd_rn(s, __ldcg(ssp + i));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  return 1.0f / sqrtf(s / d + eps);
}

// PRE: the node scales r were formed up front into rs (lone launches); else each
// epilogue forms r from the partials (a compile-time choice: one path per kernel).
template <bool PRE>
__device__ __forceinline__ void epi_aux(const GemmEpi& e, int mt, int f, int c, EpiAux& x, const float* rs) {
  x.r = 1.f;
  if (e.op == kOpResid) {
    x.a = ld4(e.out + (size_t)c * e.out_ld + mt * kBM + f);
  } else if (e.op == kOpQkv && mt < e.H + e.KV) {
    const float* p = e.rope + ((size_t)c * 64 + (f & 63)) * 2;  // (cos, sin) x 4 rotary pairs
    x.a = ld4(p);
    x.b = ld4(p + 4);
  }
  if (e.ssp_in) {  // once per node at the kernel's start (lone launches), else here per (node, m-tile)
    if constexpr (PRE)
      x.r = rs[c];
    else
      x.r = norm_scale_from_partials(e.ssp_in + (size_t)c * e.ssp_ld, e.ssp_n, e.norm_d, e.norm_eps, f >> 2);
  }
}

__device__ __forceinline__ float4 scale4(float4 y, float r) {
  return make_float4(__fmul_rn(y.x, r), __fmul_rn(y.y, r), __fmul_rn(y.z, r), __fmul_rn(y.w, r));
}

// Warp-uniform: every lane of the warp calls this for the same node c.
__device__ __forceinline__ void epi_finish(const GemmEpi& e, int mt, int lane, int c, float4 y, const EpiAux& x) {
  const int f = lane * 4;
  if (e.ssp_in) y = scale4(y, x.r);  // the folded RMSNorm of this GEMM's input rows
  switch (e.op) {
    case kOpStore:
      st4(e.out + (size_t)c * e.out_ld + mt * kBM + f, y);
      break;
    case kOpResid: {
      const float4 v = add4(x.a, y);
      st4(e.out + (size_t)c * e.out_ld + mt * kBM + f, v);
      if (e.xd_out) st_bf16x4(e.xd_out + (size_t)c * e.xd_ld + mt * kBM + f, v.x, v.y, v.z, v.w);
      if (e.ssp_out) {
        const float s = tile_sumsq(v);
        if (lane == 0) e.ssp_out[(size_t)c * e.ssp_ld + mt] = s;
      }
      break;
    }
    case kOpSwiglu: {
      // lanes 0-15 hold gate features 4l..4l+3, lanes 16-31 the matching up features:
      // after the exchange each half forms two of the four outputs (all 32 lanes busy)
      const float4 p = shfl_xor4(y, 16);
      const bool lo = lane < 16;
      const float g0 = lo ? y.x : p.z, g1 = lo ? y.y : p.w;
      const float u0 = lo ? p.x : y.z, u1 = lo ? p.y : y.w;
      st_bf16x2(e.xf + (size_t)c * e.f + mt * 64 + (lane & 15) * 4 + (lo ? 0 : 2), silu_mul(g0, u0), silu_mul(g1, u1));
      break;
    }
    default: {  // kOpQkv: tile mt is head mt of [q heads | k heads | v heads]
      const float4 pr = shfl_xor4(y, 16);
      float4 o = y;
      if (mt < e.H + e.KV) {
        const bool lo = lane < 16;
        o.x = rope1(y.x, pr.x, x.a.x, x.a.y, lo);
        o.y = rope1(y.y, pr.y, x.a.z, x.a.w, lo);
        o.z = rope1(y.z, pr.z, x.b.x, x.b.y, lo);
        o.w = rope1(y.w, pr.w, x.b.z, x.b.w, lo);
      }
      __nv_bfloat16* dst;
      if (mt < e.H) {
        dst = e.xq + (size_t)c * e.H * kBM + mt * kBM + f;
      } else {
        const bool is_k = mt < e.H + e.KV;
        const int kh = is_k ? mt - e.H : mt - e.H - e.KV;
        const char* const* tab = nullptr;  // paged cache row of this layer (kvpage.cuh), or a self buffer
        int row = 0;
        if (e.items) {
          const QkvItem& it = e.items[e.node_item[c]];
          if (it.append) {
            tab = it.ptab + (size_t)(e.layer - it.lo) * it.max_pages;
            row = it.row0 + (c - it.off);
          }
        } else if (e.append) {
          tab = e.ptab;
          row = e.row0 + c;
        }
        if (tab)  // lane's 8 bytes = half of the row's 16-byte chunk lane/2, swizzled
          dst = reinterpret_cast<__nv_bfloat16*>(const_cast<char*>(kv_block(tab, e.KV, is_k ? 0 : 1, kh, row)) +
                                                 page_chunk_off(row & 63, lane >> 1) + (lane & 1) * 8);
        else
          dst = (is_k ? e.kself : e.vself) + ((size_t)c * e.KV + kh) * kBM + f;
      }
      st_bf16x4(dst, o.x, o.y, o.z, o.w);
    }
  }
}

// Sum of the m-tile's cnt partials for node c, in contributor order (the order
// fixes the rounding: identical whichever CTA reduces and for any node count).
__device__ __forceinline__ float4 sum_partials(const float* base, size_t slot, int cnt, int c, int f) {
  const float* b = base + (size_t)c * kBM + f;
  float4 v[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) v[s] = s < cnt ? ld4cg(b + s * slot) : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 acc = v[0];
#pragma unroll
  for (int s = 1; s < 8; ++s)
    if (s < cnt) acc = add4(acc, v[s]);
  for (int s = 8; s < cnt; ++s) acc = add4(acc, ld4cg(b + s * slot));
  return acc;
}

// Reduce + apply nodes [lo, hi) of m-tile mt from the global partials; the NW
// reducer warps take nodes round-robin.
template <int NW, bool PRE>
__device__ __forceinline__ void reduce_apply(const GemmEpi& e, const SkPlan& p, int n, int mt, int cnt, int lo,
                                             int hi, int ew, int lane, const float* rs) {
  const float* base = e.part + (size_t)mt * p.max_contrib * n * kBM;
  const size_t slot = (size_t)n * kBM;
  const int f = lane * 4;
  // Every inlined copy of the epilogue op is instruction footprint the kernel's
  // tail pays for in instruction-cache misses (the dominant stall of the
  // epilogues, ncu source counters): two rows per batch and one row at a time
  // elsewhere (measured against four rows / two rows in flight, same box: lone
  // n=1 / n=44 forwards -1.7 % / -2.7 %, the 7-stage group -1.1 %).
  constexpr int kMaxC = 4;
  if (cnt <= kMaxC) {
    // The tail of the kernel: every load of a batch of kRows rows (their cnt
    // partials and the op's operands) is issued before any arithmetic, so the
    // reduction costs one L2 round trip per batch instead of one per row.
    constexpr int kRows = 2;
    for (int c0 = lo + ew; c0 < hi; c0 += kRows * NW) {
      float4 v[kRows][kMaxC];
      EpiAux x[kRows];
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        const int c = c0 + r * NW;
        x[r] = EpiAux{};
        if (c < hi) {
          epi_aux<PRE>(e, mt, f, c, x[r], rs);
          const float* b = base + (size_t)c * kBM + f;
#pragma unroll
          for (int s = 0; s < kMaxC; ++s) v[r][s] = s < cnt ? ld4cg(b + s * slot) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        const int c = c0 + r * NW;
        if (c < hi) {
          float4 acc = v[r][0];  // contributor order, as sum_partials
#pragma unroll
          for (int s = 1; s < kMaxC; ++s)
            if (s < cnt) acc = add4(acc, v[r][s]);
          epi_finish(e, mt, lane, c, acc, x[r]);
        }
      }
    }
    return;
  }
  for (int c = lo + ew; c < hi; c += NW) {
    EpiAux x0{};
    epi_aux<PRE>(e, mt, f, c, x0, rs);
    epi_finish(e, mt, lane, c, sum_partials(base, slot, cnt, c, f), x0);
  }
}

// Apply nodes c0 .. c0+cn-1 staged in xch[node][feature] (sole-contributor path).
template <int NW, bool PRE>
__device__ __forceinline__ void smem_apply(const GemmEpi& e, int mt, int c0, int cn, const float* xch, const float* rs,
                                           int ew,
                                           int lane) {
  const int f = lane * 4;
  for (int cc = ew; cc < cn; cc += NW) {
    const float4 y0 = *reinterpret_cast<const float4*>(xch + cc * kXchLd + f);
    EpiAux x0{};
    epi_aux<PRE>(e, mt, f, c0 + cc, x0, rs);
    epi_finish(e, mt, lane, c0 + cc, y0, x0);
  }
}

__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Work items are (member g, k-block t) for g = 0..count-1, t in [t0, t1):
// the TMA producer, the MMA issuer and the epilogue warps walk the same
// sequence, the smem ring and the TMEM double buffer continuing across members.
template <int MG>
#ifdef TP_GEMM_MAXNREG
__global__ void __maxnreg__(TP_GEMM_MAXNREG)
#else
__global__ void __launch_bounds__(kThreads, 1)
#endif
    sk_gemm_kernel(const __grid_constant__ GemmGroupT<MG> grp, int stages, int nbuf, int fixup_mode) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int c = blockIdx.x;
  // member g's k-block range of this CTA under the member's own plan (empty when
  // the member has fewer work units than the grid has CTAs)
  auto range = [&](int g, int& t0, int& t1) {
    const SkPlan& p = grp.m[g].p;
    t0 = min(p.total, sk_begin(p, c));
    t1 = min(p.total, sk_begin(p, c + 1));
  };
  const int bmax = grp.max_npad * 128;  // ring slot bytes for the node tile
  uint8_t* sA = smem;
  uint8_t* sB = smem + stages * kABytes;
  float* xch = reinterpret_cast<float*>(sB + stages * bmax);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(xch) + kXchBytes);
  uint64_t* empty = full + kMaxStages;
  uint64_t* tfull = empty + kMaxStages;
  uint64_t* tempty = tfull + kMaxTmemBufs;
  uint64_t* rfull = tempty + kMaxTmemBufs;
  uint64_t* rready = rfull + kRedSlots;  // reducer warps -> all epilogues: rsc is filled
  uint32_t* tholder = reinterpret_cast<uint32_t*>(rready + 1);
  RedItem* rq = reinterpret_cast<RedItem*>(tholder + 4);
  float* rsc = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full) + kBarBytes);  // [member][256]
  // A lone launch forms each node's folded-RMSNorm scale once, up front; a grouped
  // one forms it in the epilogues (measured faster there: 2024 vs 1983 us for the
  // 7-stage forward, while the lone n=44 forward gains 1993 -> 1842 us up front).
#ifndef TP_PRE_R
#define TP_PRE_R 1  // 0: always in the epilogues, 1: up front for lone launches, 2: always up front
#endif
  constexpr bool kPreR = TP_PRE_R == 2 || (TP_PRE_R == 1 && MG == 1);
#ifndef TP_EARLY_PROLOGUE
#define TP_EARLY_PROLOGUE 1
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) GSTAMP(0);
  uint32_t ncols = 32;
  while (ncols < (uint32_t)(nbuf * grp.max_npad)) ncols <<= 1;

  // member 0's first k-blocks: their weights do not depend on the previous kernel
  const int nbox0 = grp.m[0].n_pad / 16;
  int a0, b0;
  range(0, a0, b0);
  const int npre = min(stages, b0 - a0);
  if (warp == 0 && lane == 0) {
#if TP_EARLY_PROLOGUE
    // the tensor maps are the first thing fetched (parameter space, cold at each
    // launch), and the weight ring is filled before the CTA-wide barrier
    for (int g = 0; g < grp.count; ++g) {
      tma_prefetch(&grp.m[g].a);
      tma_prefetch(&grp.m[g].b);
    }
#endif
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < nbuf; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kDrainWarps);
    }
    for (int q = 0; q < kRedSlots; ++q) mbar_init(&rfull[q], 1);
    mbar_init(rready, kRedWarps);
    fence_barrier_init();
    GSTAMP(16);
#if TP_EARLY_PROLOGUE
    const SkPlan& p0 = grp.m[0].p;
    const uint64_t pol_w = policy_evict_first();
    for (int j = 0; j < npre; ++j) {
      const int t = a0 + j;
      mbar_expect_tx(&full[j], kABytes + nbox0 * 2048);
      tma_load_2d(sA + j * kABytes, &grp.m[0].a, (t % p0.KB) * kBK, (t / p0.KB) * kBM, &full[j], pol_w);
    }
    GSTAMP(20);
#endif
  }
  if (warp == 1) {
    tmem_alloc(tholder, ncols);
    if (lane == 0) GSTAMP(17);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = *tholder;
  if (threadIdx.x == 0) GSTAMP(18);

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first(), pol_x = policy_evict_last();
      const SkPlan& p0 = grp.m[0].p;
#if !TP_EARLY_PROLOGUE
      for (int g = 0; g < grp.count; ++g) {
        tma_prefetch(&grp.m[g].a);
        tma_prefetch(&grp.m[g].b);
      }
      GSTAMP(19);
      for (int j = 0; j < npre; ++j) {
        const int t = a0 + j;
        mbar_expect_tx(&full[j], kABytes + nbox0 * 2048);
        tma_load_2d(sA + j * kABytes, &grp.m[0].a, (t % p0.KB) * kBK, (t / p0.KB) * kBM, &full[j], pol_w);
      }
      GSTAMP(20);
#endif
      pdl_wait();  // node rows X come from the previous kernel
      GSTAMP(1);
      pdl_trigger();
      for (int j = 0; j < npre; ++j) {
        const int kb = (a0 + j) % p0.KB;
        for (int b = 0; b < nbox0; ++b)
          tma_load_2d(sB + j * bmax + b * 2048, &grp.m[0].b, kb * kBK, b * 16, &full[j], pol_x);
      }
      int stage = npre % stages;
      uint32_t phase = npre == stages ? 1 : 0;
      for (int g = 0; g < grp.count; ++g) {
        const CUtensorMap* ma = &grp.m[g].a;
        const CUtensorMap* mb = &grp.m[g].b;
        const int nbox = grp.m[g].n_pad / 16;
        const SkPlan& p = grp.m[g].p;
        int t0, t1;
        range(g, t0, t1);
        for (int t = (g == 0 ? t0 + npre : t0); t < t1; ++t) {
          const int mt = t / p.KB, kb = t % p.KB;
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], kABytes + nbox * 2048);
          tma_load_2d(sA + stage * kABytes, ma, kb * kBK, mt * kBM, &full[stage], pol_w);
          for (int b = 0; b < nbox; ++b)
            tma_load_2d(sB + stage * bmax + b * 2048, mb, kb * kBK, b * 16, &full[stage], pol_x);
          if (++stage == stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0, seg = 0;
      uint32_t phase = 0;
      for (int g = 0; g < grp.count; ++g) {
        const int npad = grp.m[g].n_pad;
        const SkPlan& p = grp.m[g].p;
        int t0, t1;
        range(g, t0, t1);
        const uint32_t idesc = idesc_bf16_f32(kBM, npad);
        int t = t0;
        while (t < t1) {
          const int mt = t / p.KB;
          const int seg_start = t, seg_end = min(t1, (mt + 1) * p.KB);
          const int buf = seg % nbuf;
          const uint32_t bphase = (seg / nbuf) & 1;
          mbar_wait(&tempty[buf], bphase ^ 1);
          tc_fence_after();
          const uint32_t d = taddr + buf * grp.max_npad;
          for (; t < seg_end; ++t) {
            mbar_wait(&full[stage], phase);
#ifdef TP_GEMM_TRACE
            if (g == 0 && t == seg_start && seg == 0) GSTAMP(2);
#endif
            tc_fence_after();
            const uint64_t ad = desc_kmajor_sw128(sA + stage * kABytes);
            const uint64_t bd = desc_kmajor_sw128(sB + stage * bmax);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              mma_bf16(d, ad + 2 * k, bd + 2 * k, idesc, (t > seg_start || k > 0) ? 1u : 0u);
            mma_commit(&empty[stage]);
            if (++stage == stages) {
              stage = 0;
              phase ^= 1;
            }
          }
          mma_commit(&tfull[buf]);
          GSTAMP(3);  // the last one written is the CTA's last accumulator
          ++seg;
        }
      }
    }
  } else if (warp < 2 + kDrainWarps) {
    // Drain warps: TMEM -> partial (or, for a sole-owner tile, straight through
    // the epilogue op), then free the accumulator buffer.  They never wait for
    // other CTAs: a tile this CTA must reduce is queued for the reducer warps,
    // so the MMA keeps streaming while the fix-up waits on its arrivals.
    const int quarter = warp & 3;  // TMEM lanes this warp may touch
    const int r = quarter * 32 + lane;
    const int ew = warp - 2;
    const int et = threadIdx.x - 64;
    int seg = 0, nq = 0;
    mbar_wait(rready, 0);  // the members' RMSNorm scales (folded norm) are in rsc
    for (int g = 0; g < grp.count; ++g) {
      const GemmEpi& e = grp.m[g].e;
      const int n = grp.m[g].n, npad = grp.m[g].n_pad;
      const SkPlan& p = grp.m[g].p;
      int t0, t1;
      range(g, t0, t1);
      int* arrive = e.counters;
      int t = t0;
      while (t < t1) {
        const int mt = t / p.KB;
        const int seg_end = min(t1, (mt + 1) * p.KB);
        const int buf = seg % nbuf;
        const uint32_t bphase = (seg / nbuf) & 1;
        const int cfirst = sk_cta_of(p, mt * p.KB);
        const int clast = sk_cta_of(p, (mt + 1) * p.KB - 1);
        const int cnt = clast - cfirst + 1;
        mbar_wait(&tfull[buf], bphase);
        tc_fence_after();
        const uint32_t tbase = taddr + ((uint32_t)(quarter * 32) << 16) + buf * grp.max_npad;
        if (et == 0) GSTAMP(cnt == 1 ? 9 : 11);  // the accumulator is ready (sole-owner / partial segment)
        if (cnt == 1) {
          for (int c0 = 0; c0 < n; c0 += kXchNodes) {
            const int cn = min(kXchNodes, n - c0);
            for (int col0 = c0; col0 < min(c0 + kXchNodes, npad); col0 += 16) {
              float v[16];
              tmem_ld_x16(tbase + col0, v);
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (col0 + i < n) xch[(col0 - c0 + i) * kXchLd + r] = v[i];
            }
            drain_bar();
            if (et == 0 && c0 == 0) GSTAMP(14);
            smem_apply<kDrainWarps, kPreR>(e, mt, c0, cn, xch, rsc + g * 256, ew, lane);
            drain_bar();
            if (et == 0 && c0 == 0) GSTAMP(15);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[buf]);
          if (et == 0) GSTAMP(10);
        } else {
          // stream-K fix-up: publish this CTA's fp32 partial of the m-tile
          float* dst = e.part + ((size_t)(mt * p.max_contrib + (c - cfirst)) * n) * kBM + r;
          for (int col0 = 0; col0 < (fixup_mode == 2 ? 0 : npad); col0 += 16) {
            float v[16];
            tmem_ld_x16(tbase + col0, v);
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (col0 + i < n) __stcg(dst + (size_t)(col0 + i) * kBM, v[i]);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[buf]);  // TMEM free: the MMA may go on
          drain_bar();
          if (et == 0) {  // barrier + one gpu-scope fence publishes every drain thread's stores
            GSTAMP(12);
            red_release_add(&arrive[mt], 1);  // release: every drain thread's partial stores (ordered by the barrier)
            // the contributors whose ranges end inside the tile reduce it, each a
            // slice of the nodes (they finish together; one CTA reducing a whole
            // tile was measured 2x slower on the o / down projections)
            if ((fixup_mode == 0 || fixup_mode == 3) && t1 <= (mt + 1) * p.KB) {
              rq[nq] = RedItem{g, mt, cnt, cfirst, clast};
              mbar_arrive(&rfull[nq]);
              ++nq;
            }
          }
        }
        t = seg_end;
        ++seg;
      }
    }
    if (et == 0) {
      GSTAMP(4);
      rq[nq].g = -1;
      mbar_arrive(&rfull[nq]);
    }
  } else {
    // Reducer warps: for each queued tile, wait for all of its partials, then
    // sum this CTA's node slice in contributor order and apply the epilogue op.
    // A wait only ever points at partials that drain warps publish without
    // waiting on anything but their own MMA: no cycle.
    const int rw = warp - 2 - kDrainWarps;
    const int rt = threadIdx.x - 64 - 32 * kDrainWarps;
    // first: every member's per-node RMSNorm scale r (a folded norm's consumer), once
    // per kernel instead of once per (node, m-tile) in the epilogues
    bool any = false;
    for (int g = 0; g < grp.count; ++g) any |= grp.m[g].e.ssp_in != nullptr;
    if (kPreR && any) {
      pdl_wait();  // the partials come from the previous kernel
      for (int g = 0; g < grp.count; ++g) {  // one node per reducer warp
        const GemmEpi& e = grp.m[g].e;
        if (!e.ssp_in) continue;
        for (int c = rw; c < grp.m[g].n; c += kRedWarps) {
          const float rr = norm_scale_from_partials(e.ssp_in + (size_t)c * e.ssp_ld, e.ssp_n, e.norm_d, e.norm_eps,
                                                    lane);
          if (lane == 0) rsc[g * 256 + c] = rr;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(rready);
    mbar_wait(rready, 0);
    if (rt == 0) GSTAMP(13);
    for (int q = 0;; ++q) {
      mbar_wait(&rfull[q], 0);
      const RedItem it = rq[q];
      if (it.g < 0) break;
      const GemmEpi& e = grp.m[it.g].e;
      const int n = grp.m[it.g].n;
      const SkPlan& p = grp.m[it.g].p;
      const int cend = sk_begin(p, it.clast + 1) <= (it.mt + 1) * p.KB ? it.clast : it.clast - 1;
      const int E = cend - it.cfirst + 1, rank = c - it.cfirst;
      if (rt == 0 && fixup_mode != 3) {  // counters only grow: this launch's arrivals are complete at (epoch+1)*cnt
        const int target = (e.epoch + 1) * it.cnt;
        GSTAMP(5);
        while (ld_acquire(&e.counters[it.mt]) < target) {
        }
        GSTAMP(6);
      }
      red_bar();
      reduce_apply<kRedWarps, kPreR>(e, p, n, it.mt, it.cnt, n * rank / E, n * (rank + 1) / E, rw, lane,
                              kPreR ? rsc + it.g * 256 : nullptr);
      if (rt == 0) GSTAMP(7);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) GSTAMP(8);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(taddr, ncols);
  }
}

// Optional per-launch timing of the GEMM (bench roofline): CUDA events on the
// launching stream around each launch, with the launch's algorithmic bytes
// (weights once + node rows once).
struct ProfRec {
  cudaEvent_t a, b;
  double bytes;
  int members;
};
static std::vector<ProfRec> g_prof;
static bool g_prof_on = false;
static std::mutex g_prof_mu;

// Launch epochs of every arrival-counter array (keyed by its device address):
// counters are never reset, a launch waits for (epoch+1)*cnt arrivals per tile.
static std::mutex g_epoch_mu;
static std::unordered_map<const int*, int> g_epochs;

void sk_counters_forget(const void* base, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_epoch_mu);
  const char* lo = static_cast<const char*>(base);
  for (auto it = g_epochs.begin(); it != g_epochs.end();) {
    const char* k = reinterpret_cast<const char*>(it->first);
    if (k >= lo && k < lo + bytes)
      it = g_epochs.erase(it);
    else
      ++it;
  }
}

std::vector<int> sk_epochs_get(const std::vector<int*>& ctr) {
  std::lock_guard<std::mutex> lk(g_epoch_mu);
  std::vector<int> v;
  for (int* c : ctr) {
    auto it = g_epochs.find(c);
    v.push_back(it == g_epochs.end() ? -1 : it->second);
  }
  return v;
}

void sk_epochs_set(const std::vector<int*>& ctr, const std::vector<int>& v) {
  std::lock_guard<std::mutex> lk(g_epoch_mu);
  for (size_t i = 0; i < ctr.size(); ++i) {
    if (v[i] < 0)
      g_epochs.erase(ctr[i]);
    else
      g_epochs[ctr[i]] = v[i];
  }
}

bool gemm_profile_on() { return g_prof_on; }

int sk_gemm_group(const GemmGroup& grp_in, const SkPlan& p, cudaStream_t st) {
  GemmGroup grp = grp_in;
  for (int g = 0; g < grp.count; ++g) grp.m[g].p = p;  // one plan for every member (same shape)
  return sk_gemm_group(grp, st);
}

// Members carry their own plans (shapes may differ: e.g. a draft model's layer
// grouped with a target stage's); CTA c streams its range of each member in turn.
int sk_gemm_group(const GemmGroup& grp_in, cudaStream_t st) {
  GemmGroup grp = grp_in;
  int grid = 1;
  for (int g = 0; g < grp.count; ++g) grid = std::max(grid, grp.m[g].p.G);
  {
    std::lock_guard<std::mutex> lk(g_epoch_mu);
    for (int g = 0; g < grp.count; ++g) {
      int& ep = g_epochs[grp.m[g].e.counters];
      const SkPlan& pg = grp.m[g].p;
      if ((int64_t)(ep + 2) * pg.max_contrib >= (1 << 30)) {  // ~7M launches: restart the count
        TP_CUDA(cudaMemsetAsync(grp.m[g].e.counters, 0, (size_t)pg.mtiles * sizeof(int), st));
        ep = 0;
      }
      grp.m[g].e.epoch = ep++;
    }
  }
  TP_CHECK(grp.count >= 1 && grp.count <= kMaxGroup, TP_ECONFIG, "GEMM group size outside [1, 8]");
  int mx = 16;
  for (int g = 0; g < grp.count; ++g) {
    const GemmMember& m = grp.m[g];
    TP_CHECK(m.n >= 1 && m.n_pad <= 256 && m.n_pad % 16 == 0 && m.n_pad >= m.n, TP_ESHAPE,
             "GEMM node count outside [1, 256]");
    TP_CHECK(m.e.counters && m.e.part, TP_ECONFIG, "GEMM epilogue needs partial + counter scratch");
    mx = std::max(mx, m.n_pad);
  }
  TP_CHECK(grp.max_npad == mx, TP_ECONFIG, "GemmGroup.max_npad must be the members' largest n_pad");
  const int stages = stages_for(mx);
  const size_t smem = smem_for(mx);
  const int nbuf = std::min(kMaxTmemBufs, 512 / mx);
  int dev = 0;
  TP_CUDA(cudaGetDevice(&dev));
  const int one = grp.count == 1 ? 1 : 0;
  {  // opt-in smem ceiling, set once per (instantiation, device): a per-launch value
     // would race between host threads launching different node counts
    static std::mutex mu;
    static bool done[2][64] = {{false}};
    std::lock_guard<std::mutex> lk(mu);
    if (!done[one][dev & 63]) {
      const int need = (int)std::max(smem_for(256), smem_for(16));
      int optin = 0;
      TP_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
      cudaFuncAttributes fa{};  // static shared memory (trace builds) comes off the opt-in ceiling
      if (one)
        TP_CUDA(cudaFuncGetAttributes(&fa, sk_gemm_kernel<1>));
      else
        TP_CUDA(cudaFuncGetAttributes(&fa, sk_gemm_kernel<kMaxGroup>));
      const int lim = std::max(need, std::min(optin - (int)fa.sharedSizeBytes, 232448));
      if (one)
        TP_CUDA(cudaFuncSetAttribute(sk_gemm_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim));
      else
        TP_CUDA(cudaFuncSetAttribute(sk_gemm_kernel<kMaxGroup>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim));
      done[one][dev & 63] = true;
    }
  }
  TP_CHECK((int)smem <= 232448, TP_ECONFIG, "GEMM shared memory above the opt-in limit");
  ProfRec rec{};
  if (g_prof_on) {
    TP_CUDA(cudaEventCreate(&rec.a));
    TP_CUDA(cudaEventCreate(&rec.b));
    TP_CUDA(cudaEventRecord(rec.a, st));
    rec.bytes = 0.0;
    rec.members = grp.count;
    for (int g = 0; g < grp.count; ++g)
      rec.bytes += (double)grp.m[g].p.mtiles * kBM * grp.m[g].p.KB * kBK * 2.0 +
                   (double)grp.m[g].n * grp.m[g].p.KB * kBK * 2.0;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_prof_on ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ::tp::count_launch();
  if (one) {
    GemmGroupT<1> g1;
    g1.m[0] = grp.m[0];
    g1.count = 1;
    g1.max_npad = grp.max_npad;
    TP_CUDA(cudaLaunchKernelEx(&cfg, sk_gemm_kernel<1>, g1, stages, nbuf, g_knob_fixup));
  } else {
    TP_CUDA(cudaLaunchKernelEx(&cfg, sk_gemm_kernel<kMaxGroup>, grp, stages, nbuf, g_knob_fixup));
  }
  if (g_prof_on) {
    TP_CUDA(cudaEventRecord(rec.b, st));
    std::lock_guard<std::mutex> g(g_prof_mu);
    g_prof.push_back(rec);
  }
  return TP_OK;
}

int sk_gemm(const CUtensorMap* tmA, const CUtensorMap* tmB, const SkPlan& p, const GemmEpi& epi, cudaStream_t st) {
  GemmGroup grp;
  grp.count = 1;
  grp.m[0].a = *tmA;
  grp.m[0].b = *tmB;
  grp.m[0].e = epi;
  grp.m[0].n = p.n;
  grp.m[0].n_pad = p.n_pad;
  grp.m[0].p = p;
  grp.max_npad = p.n_pad;
  return sk_gemm_group(grp, st);
}

}  // namespace tp

extern "C" int tp_profile_enable(int32_t on) {
  tp::g_prof_on = on != 0;
  return TP_OK;
}

extern "C" int tp_profile_read(double* gemm_ms, double* gemm_bytes, int64_t* launches) {
  std::lock_guard<std::mutex> g(tp::g_prof_mu);
  double ms = 0.0, bytes = 0.0;
  for (auto& r : tp::g_prof) {
    float t = 0.f;
    TP_CUDA(cudaEventSynchronize(r.b));
    TP_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    ms += t;
    bytes += r.bytes;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  *gemm_ms = ms;
  *gemm_bytes = bytes;
  *launches = (int64_t)tp::g_prof.size();
  tp::g_prof.clear();
  return TP_OK;
}

// The same records split by the launches' member count (index count - 1).
extern "C" int tp_profile_read_members(double* gemm_ms, double* gemm_bytes, int64_t* launches) {
  std::lock_guard<std::mutex> g(tp::g_prof_mu);
  for (int i = 0; i < tp::kMaxGroup; ++i) {
    gemm_ms[i] = gemm_bytes[i] = 0.0;
    launches[i] = 0;
  }
  for (auto& r : tp::g_prof) {
    float t = 0.f;
    TP_CUDA(cudaEventSynchronize(r.b));
    TP_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    const int k = std::min(std::max(r.members, 1), tp::kMaxGroup) - 1;
    gemm_ms[k] += t;
    gemm_bytes[k] += r.bytes;
    launches[k] += 1;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  tp::g_prof.clear();
  return TP_OK;
}

extern "C" int tp_debug_gemm_knob(int32_t knob, int32_t value) {
  if (knob == 0) tp::g_knob_max_stages = value;
  else if (knob == 1) tp::g_knob_smem_kb = value;
  else if (knob == 2) tp::g_knob_fixup = value;
  else return TP_ECONFIG;
  return TP_OK;
}

// Grouped GEMM timing (count members: distinct weights / node rows / outputs).
extern "C" int tp_debug_gemm_group_timed(int32_t device, int32_t count, const void* const* w_dev,
                                         const void* const* x_dev, const int32_t* n, int32_t n_out, int32_t k,
                                         void* const* out_dev, int32_t iters, float* ms_per_launch, void* stream) {
  using namespace tp;
  TP_CUDA(cudaSetDevice(device));
  TP_CHECK(count >= 1 && count <= kMaxGroup && n_out % 128 == 0 && k % 64 == 0 && iters >= 1, TP_ESHAPE,
           "debug GEMM shape");
  cudaStream_t st = (cudaStream_t)stream;
  SkPlan p = sk_plan(n_out, k, 1);
  GemmGroup grp;
  grp.count = count;
  grp.max_npad = 16;
  std::vector<void*> bufs;
  for (int g = 0; g < count; ++g) {
    TP_CHECK(n[g] >= 1 && n[g] <= 256, TP_ESHAPE, "debug GEMM node count");
    GemmMember& m = grp.m[g];
    TP_TRY(make_tmap_kmajor(&m.a, w_dev[g], n_out, k, 128));
    TP_TRY(make_tmap_kmajor(&m.b, x_dev[g], n[g], k, 16));
    m.n = n[g];
    m.n_pad = std::max(16, (n[g] + 15) / 16 * 16);
    grp.max_npad = std::max(grp.max_npad, m.n_pad);
    m.e = GemmEpi();
    m.e.op = kOpStore;
    m.e.out = (float*)out_dev[g];
    m.e.out_ld = n_out;
    SkPlan pg = p;
    pg.n = n[g];
    TP_CUDA(cudaMalloc((void**)&m.e.part, sk_part_floats(pg) * 4));
    TP_CUDA(cudaMalloc((void**)&m.e.counters, 2 * p.mtiles * 4));
    sk_counters_forget(m.e.counters, 2 * p.mtiles * 4);
    TP_CUDA(cudaMemsetAsync(m.e.counters, 0, 2 * p.mtiles * 4, st));
    bufs.push_back(m.e.part);
    bufs.push_back(m.e.counters);
  }
  TP_TRY(sk_gemm_group(grp, p, st));  // warm-up
  cudaEvent_t a, b;
  TP_CUDA(cudaEventCreate(&a));
  TP_CUDA(cudaEventCreate(&b));
  TP_CUDA(cudaEventRecord(a, st));
  for (int i = 0; i < iters; ++i) TP_TRY(sk_gemm_group(grp, p, st));
  TP_CUDA(cudaEventRecord(b, st));
  TP_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  TP_CUDA(cudaEventElapsedTime(&ms, a, b));
  *ms_per_launch = ms / iters;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  for (void* q : bufs) cudaFree(q);
  return TP_OK;
}

extern "C" int tp_debug_gemm(int32_t device, const void* w_dev, const void* x_dev, int32_t n, int32_t n_out,
                             int32_t k, void* out_dev, void* stream) {
  using namespace tp;
  TP_CUDA(cudaSetDevice(device));
  TP_CHECK(n >= 1 && n <= 256 && n_out % 128 == 0 && k % 64 == 0, TP_ESHAPE, "debug GEMM shape");
  cudaStream_t st = (cudaStream_t)stream;
  CUtensorMap ma, mb;
  TP_TRY(make_tmap_kmajor(&ma, w_dev, n_out, k, 128));
  TP_TRY(make_tmap_kmajor(&mb, x_dev, n, k, 16));
  SkPlan p = sk_plan(n_out, k, n);
  GemmEpi e;
  e.op = kOpStore;
  e.out = (float*)out_dev;
  e.out_ld = n_out;
  TP_CUDA(cudaMallocAsync((void**)&e.part, sk_part_floats(p) * 4, st));
  TP_CUDA(cudaMallocAsync((void**)&e.counters, 2 * p.mtiles * 4, st));
  sk_counters_forget(e.counters, 2 * p.mtiles * 4);
  TP_CUDA(cudaMemsetAsync(e.counters, 0, 2 * p.mtiles * 4, st));
  TP_TRY(sk_gemm(&ma, &mb, p, e, st));
  TP_CUDA(cudaFreeAsync(e.part, st));
  TP_CUDA(cudaFreeAsync(e.counters, st));
  TP_CUDA(cudaStreamSynchronize(st));
  return TP_OK;
}

extern "C" int tp_debug_gemm_timed(int32_t device, const void* w_dev, const void* x_dev, int32_t n, int32_t n_out,
                                   int32_t k, void* out_dev, int32_t iters, float* ms_per_launch, void* stream) {
  using namespace tp;
  TP_CUDA(cudaSetDevice(device));
  TP_CHECK(n >= 1 && n <= 256 && n_out % 128 == 0 && k % 64 == 0 && iters >= 1, TP_ESHAPE, "debug GEMM shape");
  cudaStream_t st = (cudaStream_t)stream;
  CUtensorMap ma, mb;
  TP_TRY(make_tmap_kmajor(&ma, w_dev, n_out, k, 128));
  TP_TRY(make_tmap_kmajor(&mb, x_dev, n, k, 16));
  SkPlan p = sk_plan(n_out, k, n);
  GemmEpi e;
  e.op = kOpStore;
  e.out = (float*)out_dev;
  e.out_ld = n_out;
  TP_CUDA(cudaMalloc((void**)&e.part, sk_part_floats(p) * 4));
  TP_CUDA(cudaMalloc((void**)&e.counters, 2 * p.mtiles * 4));
  sk_counters_forget(e.counters, 2 * p.mtiles * 4);
  TP_CUDA(cudaMemsetAsync(e.counters, 0, 2 * p.mtiles * 4, st));
  TP_TRY(sk_gemm(&ma, &mb, p, e, st));  // warm-up
  cudaEvent_t a, b;
  TP_CUDA(cudaEventCreate(&a));
  TP_CUDA(cudaEventCreate(&b));
  TP_CUDA(cudaEventRecord(a, st));
  for (int i = 0; i < iters; ++i) TP_TRY(sk_gemm(&ma, &mb, p, e, st));
  TP_CUDA(cudaEventRecord(b, st));
  TP_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  TP_CUDA(cudaEventElapsedTime(&ms, a, b));
  *ms_per_launch = ms / iters;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  TP_CUDA(cudaFree(e.part));
  TP_CUDA(cudaFree(e.counters));
  return TP_OK;
}

// Diagnostics / tests: ONE heterogeneous grouped launch — member g has its own
// weights [n_out[g], k[g]], node rows [n[g], k[g]] and plan (kOpStore into out[g]).
extern "C" int tp_debug_gemm_hetero(int32_t device, int32_t count, const void* const* w_dev, const void* const* x_dev,
                                    const int32_t* n, const int32_t* n_out, const int32_t* k, void* const* out_dev,
                                    void* stream) {
  using namespace tp;
  TP_CUDA(cudaSetDevice(device));
  TP_CHECK(count >= 1 && count <= kMaxGroup, TP_ESHAPE, "debug GEMM group size");
  cudaStream_t st = (cudaStream_t)stream;
  GemmGroup grp;
  grp.count = count;
  grp.max_npad = 16;
  std::vector<void*> bufs;
  for (int g = 0; g < count; ++g) {
    TP_CHECK(n[g] >= 1 && n[g] <= 256 && n_out[g] % 128 == 0 && k[g] % 64 == 0, TP_ESHAPE, "debug GEMM shape");
    GemmMember& m = grp.m[g];
    TP_TRY(make_tmap_kmajor(&m.a, w_dev[g], n_out[g], k[g], 128));
    TP_TRY(make_tmap_kmajor(&m.b, x_dev[g], n[g], k[g], 16));
    m.n = n[g];
    m.n_pad = std::max(16, (n[g] + 15) / 16 * 16);
    m.p = sk_plan(n_out[g], k[g], n[g]);
    grp.max_npad = std::max(grp.max_npad, m.n_pad);
    m.e = GemmEpi();
    m.e.op = kOpStore;
    m.e.out = (float*)out_dev[g];
    m.e.out_ld = n_out[g];
    TP_CUDA(cudaMalloc((void**)&m.e.part, sk_part_floats(m.p) * 4));
    TP_CUDA(cudaMalloc((void**)&m.e.counters, 2 * m.p.mtiles * 4));
    sk_counters_forget(m.e.counters, 2 * m.p.mtiles * 4);
    TP_CUDA(cudaMemsetAsync(m.e.counters, 0, 2 * m.p.mtiles * 4, st));
    bufs.push_back(m.e.part);
    bufs.push_back(m.e.counters);
  }
  TP_TRY(sk_gemm_group(grp, st));
  TP_CUDA(cudaStreamSynchronize(st));
  for (void* q : bufs) cudaFree(q);
  return TP_OK;
}

extern "C" int tp_debug_gemm_trace(int32_t device, void* dev_buf) {
  TP_CUDA(cudaSetDevice(device));
  unsigned long long* p = static_cast<unsigned long long*>(dev_buf);
  TP_CUDA(cudaMemcpyToSymbol(tp::g_gemm_trace, &p, sizeof(p)));
  const unsigned int zero = 0;
  TP_CUDA(cudaMemcpyToSymbol(tp::g_gemm_trace_ctr, &zero, sizeof(zero)));
  return TP_OK;
}
