// K1: tree-masked attention of a level's nodes against one stage's paged KV
// cache (Llama path; replaces the gather + softmax + PV of the reference
// layer_step, `/root/reference/pkg/src/treepipe/model.py:157-167,265-276`).
//
// Node i attends its *logical* key sequence of T_i = P_i + A_i + 1 slots: cache
// rows [0, P_i) (verified prefix), its A_i speculative ancestors in row order
// (the set bits of its packed ancestor row), then itself (self last).  The
// sequence is split at a fixed distance from its end:
//
//   * chunked part, slots [0, C_i), C_i = max(0, T_i - W) (W = kAttnSuffix = 16):
//     with A_i < W these are prefix rows only — cache row = slot — so every
//     node of a tree level shares them.  Canonical 64-slot chunks (chunk c =
//     slots [64c, 64c + 64) = KV page c) are grouped into canonical runs of R
//     chunks.  A run's state is the online softmax over its chunks on the 5th-
//     generation tensor cores:
//       attn_run_kernel  one CTA per (member, KV head, run, block of 128
//                        (node, query head) rows).  A producer thread stages
//                        each chunk's K and V page blocks with ONE 16 KB bulk
//                        copy each (the pages are stored in the SW128 operand
//                        layout, kvpage.cuh; two stages, mbarrier completion);
//                        an MMA thread issues S = Q K^T (M=128, N=64, K=128)
//                        into TMEM and O += P V (M=128, N=128, K=64; V is the
//                        MN-major operand) accumulating in TMEM; four softmax
//                        warps own one row each per thread: they read the
//                        row's 64 scores from TMEM, apply the row's chunk
//                        limit, take the max, rescale the row's O in TMEM only
//                        when the max grew, write bf16 P to shared memory in
//                        the SW128 layout and keep the row sum.  S of chunk
//                        c+1 is computed while the softmax of chunk c runs.
//   * suffix, the last W slots (prefix tail, ancestors, self): node-specific.
//       attn_tail_kernel one CTA per (member, node, 8 query heads): warp 0
//                        decodes the node's suffix rows (the ancestor bit-row
//                        walked in registers: word popcounts, then the
//                        rank-th set bit) into shared memory; warp w computes
//                        head w's suffix partial on the FMA pipes in a fixed
//                        order (lane l owns dims 4l..4l+3, dot products by a
//                        butterfly sum) before griddepcontrol.wait — while
//                        the run kernel still runs — then merges the run
//                        states in order and the suffix last, and writes the
//                        bf16 output row.
//
// Batch invariance: every boundary above depends only on T_i, which is the
// node's position + 1 whether it sits in a tree level or is decoded alone.  A
// row's run state depends only on its own query and the chunk rows: tensor-
// core rows are independent, the same MMA shapes run for any number of valid
// rows, the rescale decision and factor are the row's own, masked slots
// contribute exact zeros, and merges use explicitly rounded ops.  A node
// computed inside a 64-node tree level is therefore bit-identical to the same
// position decoded alone (GPU pipeline == GPU greedy decode), whatever its
// launch-mates.
#include <cstdlib>

#include <mutex>

#include "attn.h"
#include "gemm_tc.h"
#include "sm100.cuh"

namespace tp {

using namespace sm100;

constexpr int kRowsPerCta = 128;  // tcgen05 M: (node, query head) rows of a run task
constexpr int kRunThreads = 320;  // warps 0-7 softmax (column half = warp / 4), 8 K/V producer, 9 MMA issuer + Q loader
constexpr int kKvStages = 2;
constexpr int kQBytes = kRowsPerCta * kAttnHeadDim * 2;  // 32 KB: 2 dim-blocks of [128 rows][128 B]
constexpr int kChunkBytes = 2 * kPageBlockBytes;           // K + V blocks of one chunk
constexpr int kRunSmem = kQBytes + kKvStages * kChunkBytes;  // 96 KB: two CTAs per SM
constexpr int kTmemCols = 256;  // S[b] (64 fp32 columns; P[b] packed bf16 pairs over its first 32) | O (128)
constexpr int kTmemO = 128;
constexpr int kTailWarps = 8;

__device__ __forceinline__ uint32_t pack_bf16(__nv_bfloat16 lo, __nv_bfloat16 hi) {
  return (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
}
__device__ __forceinline__ uint32_t pack_f32(float lo, float hi) {
  return pack_bf16(__float2bfloat16_rn(lo), __float2bfloat16_rn(hi));
}
// 2^x as one MUFU op (ex2.approx, flush-to-zero).  K1 keeps scores, maxima
// and run states in the base-2 domain (scores pre-multiplied by
// scale * log2 e); every path uses this same function, so batch invariance is
// unaffected.
__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float score_scale(float scale) { return __fmul_rn(scale, 1.4426950408889634f); }

// Online merge of a partial (mc, lc, oc) into the running (M, L, O).
__device__ __forceinline__ void merge_scale(float& M, float& L, float mc, float lc, float& sa, float& sb) {
  const float mn = fmaxf(M, mc);
  sa = M == -INFINITY ? 0.f : ex2f(__fsub_rn(M, mn));
  sb = ex2f(__fsub_rn(mc, mn));
  L = __fmaf_rn(L, sa, __fmul_rn(lc, sb));
  M = mn;
}
__device__ __forceinline__ float merge_val(float O, float oc, float sa, float sb) {
  return __fmaf_rn(O, sa, __fmul_rn(oc, sb));
}
__device__ __forceinline__ void merge_lane(float& M, float& L, float4& O, float mc, float lc, float4 oc) {
  float sa, sb;
  merge_scale(M, L, mc, lc, sa, sb);
  O.x = merge_val(O.x, oc.x, sa, sb);
  O.y = merge_val(O.y, oc.y, sa, sb);
  O.z = merge_val(O.z, oc.z, sa, sb);
  O.w = merge_val(O.w, oc.w, sa, sb);
}

__device__ __forceinline__ size_t part_idx(const AttnArgs& a, int node, int h, int r) {
  return ((size_t)node * a.H + h) * a.max_chunks + r;
}

// kind 0: run launch, 1: tail launch
template <class Grp>
__device__ __forceinline__ int member_of(const Grp& G, int b, int kind) {
  int gi = 0;
  while (gi + 1 < G.count && b >= (kind == 0 ? G.m[gi + 1].cta_run : G.m[gi + 1].cta_tail)) ++gi;
  return gi;
}

// Slots of node i's chunked part (T_i - W, >= 0).
__device__ __forceinline__ int chunked_slots(const LevelDev& lv, int i) {
  return max(0, __ldg(lv.prefix_rows + i) + __ldg(lv.anc_cnt + i) + 1 - kAttnSuffix);
}

// ---- tcgen05 helpers local to K1 ----------------------------------------------
// 32 lanes x 32 columns of 32-bit (no wait: pair with tmem_wait_ld).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
      "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
      "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// MN-major operand in the 128-byte-swizzled layout: 64-element (128 B) rows
// along MN, one row per K index; 8-row atoms of 1024 B along K (SBO), the next
// 64 MN elements LBO bytes further.
__device__ __forceinline__ uint64_t desc_mnmajor_sw128(const void* smem_tile, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(smem_tile) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;  // LBO: next 64 MN elements
  d |= (uint64_t)(1024 >> 4) << 32;                  // SBO: next 8 K rows
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem_dst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// D (TMEM) += A (TMEM, M rows on lanes, K packed 2 x bf16 per column) x B (shared).
__device__ __forceinline__ void mma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Canonical chunks per run: a fixed property of the numerics (every launch of a
// process must use the same value for batch invariance); knob 1 for tuning.
static int g_attn_run = 4;

// A run task: (member, KV head, run, block of 128 (node, query head) rows).
struct RunTask {
  int gi, kh, r, base, rows, c0, nch;
};
template <class Grp>
__device__ __forceinline__ RunTask run_task(const Grp& G, int t) {
  RunTask k;
  k.gi = member_of(G, t, 0);
  const AttnMember& M = G.m[k.gi];
  const AttnArgs& a = M.a;
  int local = t - M.cta_run;
  k.kh = local % a.KV;
  local /= a.KV;
  const int runs = (M.c_hi + G.run - 1) / G.run;
  k.r = local % runs;
  const int blk = local / runs;
  const int grp = a.H / a.KV, npc = kRowsPerCta / grp;
  k.base = blk * npc;
  k.rows = min(npc, M.lv.n - k.base) * grp;
  k.c0 = k.r * G.run;
  k.nch = min(M.c_hi, k.c0 + G.run) - k.c0;
  return k;
}

// Diagnostics (built with -DTP_ATTN_TRACE): per-CTA, per-role globaltimer
// events of the run kernel into a device buffer set by tp_debug_attn_trace.
__device__ unsigned long long* g_attn_trace = nullptr;
#ifdef TP_ATTN_TRACE
__device__ __forceinline__ void trace_ev(int role, int& idx, int tag, int arg) {
  unsigned long long* b = g_attn_trace;
  if (!b || idx >= 1024) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  b[((size_t)blockIdx.x * 8 + role) * 1024 + idx++] = ((unsigned long long)tag << 56) |
                                                       ((unsigned long long)(arg & 0xffff) << 40) |
                                                       (t & 0xffffffffffull);
}
#define TRACE(role, idx, tag, arg) trace_ev(role, idx, tag, arg)
#else
#define TRACE(role, idx, tag, arg) ((void)0)
#endif

// Persistent, two CTAs per SM: CTA b takes tasks b, b + grid, ...  Every role
// walks the same chunk sequence (global chunk counter g), so K/V staging runs
// ahead across task boundaries:
//   warp 8      K/V producer: one 16 KB bulk copy per K / V page block, 2 stages
//   warp 8      also stages each task's Q tile with a 3D TMA box (node x head x dim)
//   warp 9      MMA issuer (lane 0):
//               S[g&1] = Q K^T (SS), then O += P[g&1] V (TS: P from TMEM over
//               the S buffer it came from, V the MN-major shared operand); S of
//               chunk g+1 is issued before waiting for P of chunk g
//   warps 0-7   softmax; warp w owns TMEM lanes 32 (w % 4) .. +31 (rows) and
//               column half w / 4: S half-row from TMEM, the row max shared with
//               the partner warp through shared memory, lazy rescale of O in
//               TMEM, bf16 P back to TMEM, half-row sum; at a task's end the O
//               row (its 64 columns) and the state are stored.
template <int MG>
__global__ void __launch_bounds__(kRunThreads, 2) attn_run_kernel(const __grid_constant__ AttnGroupT<MG> G,
                                                                  int ntasks) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  __shared__ uint64_t bars[2 * kKvStages + 8];  // (q_full: producer TMA, expect-tx)
  __shared__ uint32_t tmem_holder;
  __shared__ float xchg[2][2][kRowsPerCta];  // [chunk parity][column half] partial row maxima
  __shared__ float xl[2][kRowsPerCta];       // [column half] a task's final row sums
  uint64_t* kv_full = bars;                 // [2] producer -> MMA
  uint64_t* kv_empty = bars + kKvStages;    // [2] MMA (PV done) -> producer
  uint64_t* s_full = bars + 2 * kKvStages;  // [2] MMA -> softmax
  uint64_t* p_full = s_full + 2;            // [2] softmax (8 warps) -> MMA
  uint64_t* pv_done = s_full + 4;           // [2] MMA -> softmax, MMA (S/P buffer reuse)
  uint64_t* q_free = s_full + 6;            // MMA: the task's last S is complete (Q tile reusable)
  uint64_t* q_full = s_full + 7;            // producer (TMA) -> MMA: the task's Q tile is staged
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* sQ = dsm;
  uint8_t* sKV = dsm + kQBytes;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(kv_full + b, 1);
      mbar_init(kv_empty + b, 1);
      mbar_init(s_full + b, 1);
      mbar_init(p_full + b, 8);
      mbar_init(pv_done + b, 1);
    }
    mbar_init(q_free, 1);
    mbar_init(q_full, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc(&tmem_holder, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  pdl_wait();  // Q and the new K/V rows come from the QKV GEMM
  pdl_trigger();
  int tix = 0;
  (void)tix;
  if (threadIdx.x == 0) TRACE(0, tix, 0, 0);
  if (warp < 8) {
    // ---- softmax warps ----
    const int t = threadIdx.x & 127, half = warp >> 2;
    const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    int g = 0;
    for (int task = blockIdx.x; task < ntasks; task += gridDim.x) {
      const RunTask k = run_task(G, task);
      const AttnArgs& a = G.m[k.gi].a;
      const LevelDev& lv = G.m[k.gi].lv;
      const float c2 = score_scale(a.scale);
      const int grp = a.H / a.KV;
      const bool valid = t < k.rows;
      const bool warp_live = (t & ~31) < k.rows;  // any valid row in this warp
      const int node = k.base + (valid ? t / grp : 0), h = k.kh * grp + (valid ? t % grp : 0);
      const int Crow = valid ? chunked_slots(lv, node) : 0;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < k.nch; ++j, ++g) {
        const int b = g & 1;
        mbar_wait(s_full + b, (g >> 1) & 1);
        if (threadIdx.x == 0) TRACE(0, tix, 1, g);
        tc_fence_after();
        uint32_t sv[32];
        if (warp_live) {
          tmem_ld32(tl + b * 64 + half * 32, sv);
          tmem_wait_ld();
        }
        if (threadIdx.x == 0) TRACE(0, tix, 8, g);
        const int lim = min(32, max(0, Crow - (k.c0 + j) * kAttnChunk - half * 32));
        const bool full = __all_sync(0xffffffffu, lim == 32);  // warp-uniform unmasked fast path
        // partial row max over this half (4 independent chains, combined in a fixed order)
        float c4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        if (warp_live) {
          if (full) {
#pragma unroll
            for (int q = 0; q < 32; ++q) c4[q & 3] = fmaxf(c4[q & 3], __uint_as_float(sv[q]));
          } else {
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (q < lim) c4[q & 3] = fmaxf(c4[q & 3], __uint_as_float(sv[q]));
          }
        }
        xchg[b][half][t] = fmaxf(fmaxf(c4[0], c4[1]), fmaxf(c4[2], c4[3]));
        // the pair of warps sharing these rows: both have read S[b] past this point,
        // so P may overwrite it
        asm volatile("bar.sync %0, 64;" ::"r"(1 + (warp & 3)) : "memory");
        const float cmax = fmaxf(xchg[b][0][t], xchg[b][1][t]);
        if (threadIdx.x == 0) TRACE(0, tix, 9, g);
        // Lazy rescale: the row keeps its reference max m until a chunk's max
        // exceeds it by more than 8 (p <= 2^8 meanwhile), so O is rescaled —
        // and the previous PV waited for — only on such jumps.  The decision
        // depends on the row's own scores only.
        const float cand = cmax == -INFINITY ? -INFINITY : __fmul_rn(cmax, c2);
        const bool grow = m != -INFINITY && cand > __fadd_rn(m, 8.f);
        const float mn = (m == -INFINITY || grow) ? cand : m;
        const float alpha = grow ? ex2f(__fsub_rn(m, mn)) : 1.f;
        uint32_t pk[16];
        float s4[4] = {0.f, 0.f, 0.f, 0.f};  // fp32 sum of the unrounded p (4 chains, fixed combine order)
        if (warp_live) {
          if (full) {
#pragma unroll
            for (int q = 0; q < 32; q += 2) {
              const float p0 = ex2f(__fmaf_rn(__uint_as_float(sv[q]), c2, -mn));
              const float p1 = ex2f(__fmaf_rn(__uint_as_float(sv[q + 1]), c2, -mn));
              const __nv_bfloat162 pp = __floats2bfloat162_rn(p0, p1);
              pk[q >> 1] = *reinterpret_cast<const uint32_t*>(&pp);
              s4[q & 3] = __fadd_rn(s4[q & 3], p0);
              s4[(q + 1) & 3] = __fadd_rn(s4[(q + 1) & 3], p1);
            }
          } else {
#pragma unroll
            for (int q = 0; q < 32; q += 2) {
              const float p0 = q < lim ? ex2f(__fmaf_rn(__uint_as_float(sv[q]), c2, -mn)) : 0.f;
              const float p1 = q + 1 < lim ? ex2f(__fmaf_rn(__uint_as_float(sv[q + 1]), c2, -mn)) : 0.f;
              const __nv_bfloat162 pp = __floats2bfloat162_rn(p0, p1);
              pk[q >> 1] = *reinterpret_cast<const uint32_t*>(&pp);
              s4[q & 3] = __fadd_rn(s4[q & 3], p0);
              s4[(q + 1) & 3] = __fadd_rn(s4[(q + 1) & 3], p1);
            }
          }
        }
        const float ls = __fadd_rn(__fadd_rn(s4[0], s4[1]), __fadd_rn(s4[2], s4[3]));
        if (threadIdx.x == 0) TRACE(0, tix, 10, g);
        if (j > 0 && warp_live && __any_sync(0xffffffffu, grow)) {  // O must be stable: the previous PV is complete
          mbar_wait(pv_done + ((g - 1) & 1), ((g - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int q2 = 0; q2 < 2; ++q2) {
            uint32_t o[32];
            const uint32_t col = tl + kTmemO + half * 64 + q2 * 32;
            tmem_ld32(col, o);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__fmul_rn(__uint_as_float(o[e]), alpha));
            tmem_st32(col, o);
          }
        }
        if (threadIdx.x == 0) TRACE(0, tix, 11, g);
        if (warp_live) tmem_st16(tl + b * 64 + half * 16, pk);  // P[b] over the S[b] columns both halves read
        tmem_wait_st();
        l = __fmaf_rn(l, alpha, ls);  // this half's running sum (the halves are added at the end)
        m = mn;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full + b);
        if (threadIdx.x == 0) TRACE(0, tix, 2, g);
      }
      mbar_wait(pv_done + ((g - 1) & 1), ((g - 1) >> 1) & 1);  // the task's last PV
      if (threadIdx.x == 0) TRACE(0, tix, 3, g);
      tc_fence_after();
      float* po = valid ? a.po + part_idx(a, node, h, k.r) * kAttnHeadDim + half * 64 : nullptr;
      if (warp_live) {
#pragma unroll 1
        for (int q2 = 0; q2 < 2; ++q2) {
          uint32_t o[32];
          tmem_ld32(tl + kTmemO + half * 64 + q2 * 32, o);
          tmem_wait_ld();
          if (valid)
#pragma unroll
            for (int e = 0; e < 32; e += 4)
              *reinterpret_cast<float4*>(po + q2 * 32 + e) =
                  make_float4(__uint_as_float(o[e]), __uint_as_float(o[e + 1]), __uint_as_float(o[e + 2]),
                              __uint_as_float(o[e + 3]));
        }
      }
      if (threadIdx.x == 0) TRACE(0, tix, 12, g);
      tc_fence_before();  // the next task's first PV (accumulate = 0) overwrites O after our p_full arrival
      xl[half][t] = l;
      asm volatile("bar.sync %0, 64;" ::"r"(1 + (warp & 3)) : "memory");
      if (valid && half == 0) {
        a.pm[part_idx(a, node, h, k.r)] = m;
        a.pl[part_idx(a, node, h, k.r)] = __fadd_rn(xl[0][t], xl[1][t]);
      }
      if (threadIdx.x == 0) TRACE(0, tix, 13, g);
    }
  } else if (warp == 8) {
    // ---- K/V producer ----
    if (lane == 0) {
      int g = 0, it = 0;
      for (int task = blockIdx.x; task < ntasks; task += gridDim.x, ++it) {
        const RunTask k = run_task(G, task);
        const AttnArgs& a = G.m[k.gi].a;
        // the task's query rows: two TMA boxes (dims 0-63, 64-127) of 128 (node, head) rows
        if (it > 0) mbar_wait(q_free, (it - 1) & 1);  // every S of the previous task has read the tile
        mbar_expect_tx(q_full, kQBytes);
        const int grp = a.H / a.KV;
#pragma unroll
        for (int kb = 0; kb < 2; ++kb)
          tma_load_3d(sQ + kb * (kQBytes / 2), &a.qmap, kb * 64, k.kh * grp, a.q_row0 + k.base, q_full);
        TRACE(2, tix, 7, it);
        for (int j = 0; j < k.nch; ++j, ++g) {
          const int s = g & 1;
          if (g >= kKvStages) mbar_wait(kv_empty + s, ((g >> 1) - 1) & 1);
          TRACE(1, tix, 4, g);
          const int row = (k.c0 + j) * kAttnChunk;
          uint8_t* dst = sKV + s * kChunkBytes;
          mbar_expect_tx(kv_full + s, kChunkBytes);
          bulk_g2s(dst, kv_block(a.ptab, a.KV, 0, k.kh, row), kPageBlockBytes, kv_full + s);
          bulk_g2s(dst + kPageBlockBytes, kv_block(a.ptab, a.KV, 1, k.kh, row), kPageBlockBytes, kv_full + s);
        }
      }
    }
    __syncwarp();
  } else {
    // ---- MMA issuer (lane 0) ----
    if (lane == 0) {
      constexpr uint32_t idS = idesc_bf16_f32(kRowsPerCta, kAttnChunk);
      constexpr uint32_t idPV = idesc_bf16_f32(kRowsPerCta, kAttnHeadDim) | (1u << 16);  // B (V) MN-major
      int gs = 0, it = 0;  // S issued (global chunk index), task iteration
      auto issue_s = [&](bool last) {
        const int b = gs & 1;
        mbar_wait(kv_full + b, (gs >> 1) & 1);
        if (gs >= 2) mbar_wait(pv_done + b, ((gs >> 1) - 1) & 1);  // P of chunk gs - 2 consumed: S[b] free
        TRACE(3, tix, 5, gs);
        tc_fence_after();
        const uint8_t* sK = sKV + b * kChunkBytes;
#pragma unroll
        for (int kb = 0; kb < 2; ++kb) {
          const uint64_t ad = desc_kmajor_sw128(sQ + kb * (kQBytes / 2));
          const uint64_t bd = desc_kmajor_sw128(sK + kb * (kPageBlockBytes / 2));
#pragma unroll
          for (int q = 0; q < 4; ++q) mma_bf16(tmem + b * 64, ad + 2 * q, bd + 2 * q, idS, (kb | q) ? 1u : 0u);
        }
        mma_commit(s_full + b);
        if (last) mma_commit(q_free);  // the Q loader may refill the tile once these MMAs complete
        ++gs;
      };
      for (int task = blockIdx.x; task < ntasks; task += gridDim.x, ++it) {
        const RunTask k = run_task(G, task);
        mbar_wait(q_full, it & 1);
        issue_s(k.nch == 1);
        for (int j = 0; j < k.nch; ++j) {
          if (j + 1 < k.nch) issue_s(j + 2 == k.nch);
          const int gc = gs - (j + 1 < k.nch ? 2 : 1);  // chunk whose PV is next
          const int b = gc & 1;
          mbar_wait(p_full + b, (gc >> 1) & 1);
          TRACE(3, tix, 6, gc);
          tc_fence_after();
          const uint8_t* sV = sKV + b * kChunkBytes + kPageBlockBytes;
#pragma unroll
          for (int q = 0; q < 4; ++q)  // 16 slots per MMA: 8 packed P columns, 2 8-row atoms of V
            mma_bf16_ts(tmem + kTmemO, tmem + b * 64 + 8 * q, desc_mnmajor_sw128(sV + q * 2048, kPageBlockBytes / 2),
                        idPV, (j > 0 || q > 0) ? 1u : 0u);
          mma_commit(pv_done + b);
          mma_commit(kv_empty + b);
        }
      }
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

// ---- per-node suffix + ordered merge --------------------------------------------

// One CTA per (member, node, 8 query heads).  Warp 0 resolves the node's suffix
// slots (prefix tail rows, ancestors decoded from the packed bit-row, self) to
// (page, row-in-page) pairs in shared memory.  Warp w then takes query head
// 8*hb + w: lanes j and j + 16 compute slot j's score over dims [0, 64) and
// [64, 128) (sequential FMAs, halves added), the softmax runs over the 16 slot
// lanes, and P.V runs with lane l owning dims 4l..4l+3 (slots in order) — all
// before griddepcontrol.wait when `early`; then the run states are merged in
// order, the suffix last, and the bf16 output row is written.
template <int MG>
#ifndef TP_TAIL_MINB
#define TP_TAIL_MINB 3  // 80 registers, 3 CTAs per SM (measured: 1.3 % faster lone n=44 forward than 104 regs / 2 CTAs; 4 CTAs spill)
#endif
__global__ void __launch_bounds__(kTailWarps * 32, TP_TAIL_MINB) attn_tail_kernel(const __grid_constant__ AttnGroupT<MG> G,
                                                                    int early) {
  if (!early) pdl_wait();
  pdl_trigger();  // the O-projection GEMM may start streaming its weights
  __shared__ const char* spg[kAttnSuffix];  // page base of the slot's row (nullptr: a self buffer row)
  __shared__ int sr[kAttnSuffix];           // row within the page
  __shared__ __align__(16) float sq[kTailWarps][kAttnHeadDim];
  const int gi = member_of(G, blockIdx.x, 1);
  const AttnArgs& a = G.m[gi].a;
  const LevelDev& lv = G.m[gi].lv;
  const int hbs = (a.H + kTailWarps - 1) / kTailWarps;
  const int local = blockIdx.x - G.m[gi].cta_tail;
  const int i = local / hbs, hb = local % hbs;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = __ldg(lv.prefix_rows + i);
  const int A = __ldg(lv.anc_cnt + i);
  const int T = P + A + 1;
  const int s0 = max(0, T - kAttnSuffix), ns = T - s0;
  if (warp == 0) {
    const int slot = s0 + lane;
    int rank = slot - P;  // >= 0: an ancestor slot (< A) or self (== A)
    int row = lane < ns && slot < P ? slot : -1;
    const uint64_t* bits = lv.anc + (size_t)i * lv.words;
    bool found = !(lane < ns && rank >= 0 && rank < A);
    for (int w0 = 0; w0 < lv.words; w0 += 32) {
      const uint64_t mine = w0 + lane < lv.words ? __ldg(bits + w0 + lane) : 0ull;
      const int nw = min(32, lv.words - w0);
      for (int w = 0; w < nw; ++w) {
        const uint64_t x = __shfl_sync(0xffffffffu, mine, w);
        const int pc = __popcll(x);
        if (!found) {
          if (rank < pc) {
            const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
            const int plo = __popc(lo);
            const int bit = rank < plo ? (int)__fns(lo, 0, rank + 1) : 32 + (int)__fns(hi, 0, rank - plo + 1);
            row = lv.bits_base + 64 * (w0 + w) + bit;
            found = true;
          } else {
            rank -= pc;
          }
        }
      }
    }
    if (lane < kAttnSuffix) {
      const bool self_buf = lane == ns - 1 && a.kself;  // recompute mode: self K/V in side buffers
      if (row < 0) row = lv.row0 + i;                   // self in the cache (append mode)
      spg[lane] = self_buf || lane >= ns ? nullptr : a.ptab[row >> 6];
      sr[lane] = row & 63;
    }
  }
  __syncthreads();
  const int h = hb * kTailWarps + warp;
  if (h >= a.H) {
    if (early) pdl_wait();
    return;
  }
  const int kh = h / (a.H / a.KV);
  const int64_t koff = (int64_t)kh * kPageBlockBytes, voff = (int64_t)(a.KV + kh) * kPageBlockBytes;
  {  // this head's query as floats (broadcast reads below)
    const uint2 qv = *reinterpret_cast<const uint2*>(a.q + (size_t)i * a.q_stride + h * kAttnHeadDim + 4 * lane);
    *reinterpret_cast<float4*>(&sq[warp][4 * lane]) =
        make_float4(__uint_as_float(qv.x << 16), __uint_as_float(qv.x & 0xffff0000u), __uint_as_float(qv.y << 16),
                    __uint_as_float(qv.y & 0xffff0000u));
  }
  __syncwarp();
  // ---- all K and V loads first (one memory round trip): lanes j (< 16) and
  // j + 16 take slot j's K over dims [0, 64) / [64, 128); for P.V lane l owns
  // dims 4l .. 4l+3 of every slot's V row (its half of 16-byte chunk l / 2)
  const int js = lane & 15, hh = lane >> 4;
  const int e16 = lane >> 1;
  const int lane_off = ((e16 >> 3) << 13) + (lane & 1) * 8;
  uint4 kc[8];
  {
    const char* pg = spg[js];
    const int r = sr[js];
    const bool live = js < ns;
    const char* blk = pg ? pg + koff + (hh << 13) + (r << 7) : nullptr;
    const uint4* kp = reinterpret_cast<const uint4*>(a.kself + ((size_t)i * a.KV + kh) * kAttnHeadDim + hh * 64);
#pragma unroll
    for (int c = 0; c < 8; ++c)
      kc[c] = !live ? make_uint4(0u, 0u, 0u, 0u)
                    : pg ? __ldcg(reinterpret_cast<const uint4*>(blk + ((c ^ (r & 7)) << 4))) : __ldcg(kp + c);
  }
  uint2 vr[kAttnSuffix];
#pragma unroll
  for (int j = 0; j < kAttnSuffix; ++j) {
    const char* pg = spg[j];
    const int r = sr[j];
    vr[j] = j >= ns ? make_uint2(0u, 0u)
            : pg   ? __ldcg(reinterpret_cast<const uint2*>(pg + voff + lane_off + (r << 7) + (((e16 & 7) ^ (r & 7)) << 4)))
                   : __ldcg(reinterpret_cast<const uint2*>(a.vself + ((size_t)i * a.KV + kh) * kAttnHeadDim + 4 * lane));
  }
  float sc;
  {
    float d = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float4 qa = *reinterpret_cast<const float4*>(&sq[warp][hh * 64 + 8 * c]);
      const float4 qb = *reinterpret_cast<const float4*>(&sq[warp][hh * 64 + 8 * c + 4]);
      d = __fmaf_rn(qa.x, __uint_as_float(kc[c].x << 16), d);
      d = __fmaf_rn(qa.y, __uint_as_float(kc[c].x & 0xffff0000u), d);
      d = __fmaf_rn(qa.z, __uint_as_float(kc[c].y << 16), d);
      d = __fmaf_rn(qa.w, __uint_as_float(kc[c].y & 0xffff0000u), d);
      d = __fmaf_rn(qb.x, __uint_as_float(kc[c].z << 16), d);
      d = __fmaf_rn(qb.y, __uint_as_float(kc[c].z & 0xffff0000u), d);
      d = __fmaf_rn(qb.z, __uint_as_float(kc[c].w << 16), d);
      d = __fmaf_rn(qb.w, __uint_as_float(kc[c].w & 0xffff0000u), d);
    }
    const float other = __shfl_xor_sync(0xffffffffu, d, 16);
    sc = js < ns ? __fmul_rn(hh ? __fadd_rn(other, d) : __fadd_rn(d, other), score_scale(a.scale)) : -INFINITY;
  }
  float mx = sc;
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const float p = js < ns ? ex2f(__fsub_rn(sc, mx)) : 0.f;
  float ls = p;
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) ls = __fadd_rn(ls, __shfl_xor_sync(0xffffffffu, ls, o));
  const float pb = __bfloat162float(__float2bfloat16_rn(p));  // P rounded to bf16, as the run path
  float4 os = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int j = 0; j < kAttnSuffix; ++j) {  // slots in order (p = 0 past ns)
    const float pj = __shfl_sync(0xffffffffu, pb, j);
    os.x = __fmaf_rn(pj, __uint_as_float(vr[j].x << 16), os.x);
    os.y = __fmaf_rn(pj, __uint_as_float(vr[j].x & 0xffff0000u), os.y);
    os.z = __fmaf_rn(pj, __uint_as_float(vr[j].y << 16), os.z);
    os.w = __fmaf_rn(pj, __uint_as_float(vr[j].y & 0xffff0000u), os.w);
  }
  if (early) pdl_wait();  // the run kernel's states are complete from here on
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

template <int MG>
static int attn_group_launch(const AttnArgs* a, const LevelDev* lv, int count, cudaStream_t st) {
  AttnGroupT<MG> G;
  G.count = count;
  G.run = g_attn_run;
  int cr = 0, ct = 0;
  for (int g = 0; g < count; ++g) {
    AttnMember& m = G.m[g];
    m.a = a[g];
    m.lv = lv[g];
    const int grp = a[g].H / a[g].KV;
    TP_CHECK(grp >= 1 && kRowsPerCta % grp == 0, TP_ESHAPE, "query group size must divide 128");
    const int max_c = std::max(0, lv[g].max_t - kAttnSuffix);  // longest chunked part of the member
    m.c_hi = (max_c + kAttnChunk - 1) / kAttnChunk;
    m.blocks = (lv[g].n * grp + kRowsPerCta - 1) / kRowsPerCta;
    TP_CHECK((m.c_hi + G.run - 1) / G.run <= a[g].max_chunks, TP_ESHAPE, "attention runs exceed scratch");
    m.cta_run = cr;
    m.cta_tail = ct;
    cr += a[g].KV * ((m.c_hi + G.run - 1) / G.run) * m.blocks;
    ct += lv[g].n * ((a[g].H + kTailWarps - 1) / kTailWarps);
  }
  static std::mutex mu;  // per instantiation; host threads of several shards launch concurrently
  static bool attr_set[64] = {false};  // per device
  int dev = 0;
  TP_CUDA(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!attr_set[dev & 63]) {
      TP_CUDA(cudaFuncSetAttribute(attn_run_kernel<MG>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRunSmem));
      attr_set[dev & 63] = true;
    }
  }
  static const int dbg = getenv("TP_ATTN_DEBUG") ? atoi(getenv("TP_ATTN_DEBUG")) : 0;  // diagnostics: 1 skip tail, 2 skip runs
  if (dbg & 2) cr = 0;
  if (dbg & 1) ct = 0;
  if (cr > 0) {
    ::tp::count_launch();
    const int grid = std::min(cr, 2 * num_sms());  // persistent: two CTAs per SM walk the tasks
    TP_CUDA(launch_pdl(attn_run_kernel<MG>, dim3(grid), dim3(kRunThreads), (size_t)kRunSmem, st, G, cr));
    TP_CUDA(cudaGetLastError());
    timeline_mark("attn_shared", st);
  }
  if (ct > 0) {
    ::tp::count_launch();
    TP_CUDA(launch_pdl(attn_tail_kernel<MG>, dim3(ct), dim3(kTailWarps * 32), 0, st, G, cr > 0 ? 1 : 0));
    TP_CUDA(cudaGetLastError());
    timeline_mark("attn_tail", st);
  }
  return TP_OK;
}

int attn_tree_group(const AttnArgs* a, const LevelDev* lv, int count, cudaStream_t st) {
  TP_CHECK(count >= 1 && count <= kAttnMaxGroup, TP_ECONFIG, "attention group size outside [1, 64]");
  if (count == 1) return attn_group_launch<1>(a, lv, count, st);
  if (count <= 8) return attn_group_launch<8>(a, lv, count, st);
  return attn_group_launch<kAttnMaxGroup>(a, lv, count, st);
}

int attn_tree(const AttnArgs& a, const LevelDev& lv, cudaStream_t st) { return attn_tree_group(&a, &lv, 1, st); }

int attn_set_trace(void* dev_buf) {
  unsigned long long* p = static_cast<unsigned long long*>(dev_buf);
  TP_CUDA(cudaMemcpyToSymbol(g_attn_trace, &p, sizeof(p)));
  return TP_OK;
}

int attn_set_run(int run) {
  TP_CHECK(run >= 1 && run <= 64, TP_ECONFIG, "attention run length outside [1, 64]");
  g_attn_run = run;
  return TP_OK;
}

}  // namespace tp
