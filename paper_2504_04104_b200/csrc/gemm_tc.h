// Stream-K tcgen05 GEMM plan, fused epilogues, launcher (see gemm_tc.cu).
#pragma once

#include <cuda.h>

#include <vector>

#include "common.cuh"

namespace tp {

struct SkPlan {
  int mtiles;       // N_out / 128
  int KB;           // K / 64
  int total;        // mtiles * KB k-blocks, linearised m-major
  int G, q, r;      // CTAs; CTA c owns q (+1 if c < r) consecutive k-blocks
  int max_contrib;  // max CTAs contributing to one m-tile
  int n, n_pad;     // valid node columns / MMA N (single-member launches)
};

__host__ __device__ inline int sk_begin(const SkPlan& p, int c) { return c * p.q + (c < p.r ? c : p.r); }
__host__ __device__ inline int sk_cta_of(const SkPlan& p, int t) {
  const int big = p.r * (p.q + 1);
  return t < big ? t / (p.q + 1) : p.r + (t - big) / p.q;
}

// Epilogue applied (inside the GEMM) to the fully reduced 128-feature m-tile.
enum GemmOp : int {
  kOpStore = 0,   // out[node * out_ld + j] = y
  kOpQkv = 1,     // RoPE(q, k) + scatter: q -> xq, k/v -> KV cache rows (or self buffers)
  kOpResid = 2,   // out[node * out_ld + j] += y   (fp32 residual stream)
  kOpSwiglu = 3,  // tile = 64 gate rows | 64 up rows: xf[node][mt*64 + i] = bf16(silu(g) * u)
};

// Per-request KV destination of a ragged (multi-request) QKV member: node c of
// item it = items[node_item[c]] writes its K/V rows to that request's cache.
struct QkvItem {
  char* const* ptab;  // the request-stage's paged KV table [layers][max_pages] (device, kvpage.cuh)
  int max_pages;
  int lo;                 // first layer hosted by that stage
  int row0, append, off;  // first appended row, append flag, first node of the item
};

struct GemmEpi {
  int op = kOpStore;
  float* out = nullptr;
  int out_ld = 0;
  // kOpQkv
  int H = 0, KV = 0, row0 = 0, append = 0;
  const float* rope = nullptr;  // [n][64][2] (cos, sin) per node position
  char* const* ptab = nullptr;  // single request: this layer's page table row (kvpage.cuh)
  __nv_bfloat16 *xq = nullptr, *kself = nullptr, *vself = nullptr;
  const QkvItem* items = nullptr;      // ragged member (nullptr: single request, fields above)
  const int32_t* node_item = nullptr;  // [n]
  int layer = 0;
  // kOpSwiglu
  __nv_bfloat16* xf = nullptr;
  int f = 0;
  // RMSNorm folded into the GEMMs (no norm kernel): the residual producer (kOpResid)
  // also writes xd_out = bf16(x) and, per (node, m-tile), the sum of squares of the
  // tile's 128 new residual values; the consumer (kOpQkv / kOpSwiglu, whose B
  // operand is that bf16(x)) scales each node's accumulator by
  // r = 1/sqrt(sum(ssp)/d + eps) before its op (norm weights are 1).
  __nv_bfloat16* xd_out = nullptr;  // producer: [n][xd_ld]
  int xd_ld = 0;
  float* ssp_out = nullptr;  // producer: [n][ssp_ld]
  const float* ssp_in = nullptr;  // consumer: [n][ssp_ld], ssp_n partials per node
  int ssp_ld = 0, ssp_n = 0;
  float norm_d = 1.f, norm_eps = 0.f;
  // stream-K fix-up state
  float* part = nullptr;  // [mtiles][max_contrib][n][128]
  int* counters = nullptr;  // [mtiles] arrival counters, monotonic across launches (see epoch)
  int epoch = 0;            // launches that used `counters` before this one (set by sk_gemm_group)
};

// A grouped launch: up to kMaxGroup GEMMs of the SAME (N_out, K) shape — e.g. the
// same layer slot of several pipeline stages hosted on one GPU — each with its
// own weights, node rows, node count and epilogue.  CTA c streams its stream-K
// range of member 0, then the same range of member 1, ...: every member sees
// exactly the segment boundaries of its ungrouped launch, so grouped results are
// bit-identical to ungrouped ones (batch invariance across stages).
constexpr int kMaxGroup = 8;

struct GemmMember {
  CUtensorMap a;  // weights [N_out, K]
  CUtensorMap b;  // node rows [n_pad, K]
  GemmEpi e;
  int n, n_pad;
  SkPlan p;  // this member's stream-K plan (its own (N_out, K))
};

template <int MG>
struct GemmGroupT {
  GemmMember m[MG];
  int count;
  int max_npad;
};
// Host-side group; a launch copies it into a GemmGroupT<1> when it has one member
// (kernel parameters are copied per launch: ~0.5 KB instead of ~3.6 KB).
using GemmGroup = GemmGroupT<kMaxGroup>;

__device__ __forceinline__ void st_bf16x4(__nv_bfloat16* p, float a, float b, float c, float d) {
  uint2 u;
  u.x = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(a)) |
        ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(b)) << 16);
  u.y = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(c)) |
        ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(d)) << 16);
  *reinterpret_cast<uint2*>(p) = u;
}

__device__ __forceinline__ void st_bf16x2(__nv_bfloat16* p, float a, float b) {
  *reinterpret_cast<uint32_t*>(p) = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(a)) |
                                    ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(b)) << 16);
}

// Sum of squares of a warp's 128 values (lane = 4 consecutive), in the one order
// every producer of RMSNorm partials uses (the residual epilogue, the prep launch).
__device__ __forceinline__ float tile_sumsq(float4 v) {
  float s = __fmul_rn(v.x, v.x);
  s = __fmaf_rn(v.y, v.y, s);
  s = __fmaf_rn(v.z, v.z, s);
  s = __fmaf_rn(v.w, v.w, s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  return s;
}

__device__ __forceinline__ float rope1(float y, float pr, float cs, float sn, bool lo) {
  return lo ? __fsub_rn(__fmul_rn(y, cs), __fmul_rn(pr, sn)) : __fadd_rn(__fmul_rn(y, cs), __fmul_rn(pr, sn));
}
// silu(g) * u with the approximate exp / divide (ex2.approx, rcp.approx: a few ulp,
// far below the bf16 rounding of the result).  The IEEE expf + __fdiv_rn chain
// cost ~2 us of a gate/up launch's tail at n=45 (its epilogue is latency-bound on
// 4 or 8 warps; scripts/gemm_chain_trace.py).
__device__ __forceinline__ float silu_mul(float g, float u) {
  return __fmul_rn(__fdividef(g, __fadd_rn(1.0f, __expf(-g))), u);
}

int num_sms();
int make_tmap_kmajor(CUtensorMap* map, const void* gptr, int64_t rows, int64_t k, int box_rows);
int make_tmap_q3d(CUtensorMap* map, const void* gptr, int64_t nodes, int heads, int grp);
SkPlan sk_plan(int n_out, int k, int n);
inline size_t sk_part_floats(const SkPlan& p) { return (size_t)p.mtiles * p.max_contrib * p.n * 128; }
// Launched with programmatic dependent launch: the weight prologue overlaps the
// previous kernel; activations are read only after griddepcontrol.wait.
int sk_gemm(const CUtensorMap* tmA, const CUtensorMap* tmB, const SkPlan& p, const GemmEpi& epi, cudaStream_t st);
// Grouped launch (members share p's shape; p.n / p.n_pad are ignored).
int sk_gemm_group(const GemmGroup& grp, const SkPlan& p, cudaStream_t st);
// Grouped launch of members with their own plans (m[g].p; shapes may differ).
int sk_gemm_group(const GemmGroup& grp, cudaStream_t st);
// Forget the launch epochs of counter arrays in [base, base+bytes) (call whenever
// such memory is (re)allocated and zeroed).
void sk_counters_forget(const void* base, size_t bytes);
// The launch epochs of counter arrays (-1: none yet), and setting them back (a
// captured sequence that is discarded before running).
std::vector<int> sk_epochs_get(const std::vector<int*>& ctr);
void sk_epochs_set(const std::vector<int*>& ctr, const std::vector<int>& v);


}  // namespace tp
