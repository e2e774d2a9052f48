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
//     evict-last), warp 1 = single-thread MMA issuer, warps 2-5 = epilogue
//     (double-buffered TMEM accumulators: the next segment's MMAs overlap the
//     previous segment's epilogue);
//   * programmatic dependent launch: barrier init, TMEM allocation and the
//     first ring-full of *weight* tiles are issued before griddepcontrol.wait,
//     i.e. while the previous kernel is still finishing;
//   * fused fix-up: an m-tile with several contributing CTAs has each write
//     its fp32 partial; the last to arrive (atomic counter) sums all partials
//     in contributor order and applies the epilogue op (RoPE + KV-row scatter,
//     residual add, SwiGLU, or a plain store).  A sole contributor applies it
//     straight from TMEM.
// Determinism / batch invariance: segment boundaries depend only on
// (N_out, K, #SMs); partials are summed in contributor order whichever CTA
// arrives last; each output column's accumulation chain is the same for any n.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "gemm_tc.h"
#include "sm100.cuh"

namespace tp {

using namespace sm100;

constexpr int kBM = 128, kBK = 64;
constexpr int kMaxStages = 8;
constexpr int kThreads = 192;
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

static int stages_for(int n_pad) {
  const int per = kABytes + n_pad * 128;
  return std::min(kMaxStages, (200 * 1024 - kXchBytes) / per);
}

static size_t smem_for(int n_pad) {
  return (size_t)stages_for(n_pad) * (kABytes + n_pad * 128) + kXchBytes + 1024 /*align*/ + 256 /*barriers*/;
}

// ---- device --------------------------------------------------------------------
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Apply the epilogue op to reduced values xch[cc][r] for nodes c0 .. c0+cn-1.
__device__ __forceinline__ void apply_op(const GemmEpi& e, int mt, int r, int c0, int cn, const float* xch) {
  for (int cc = 0; cc < cn; ++cc) {
    const int c = c0 + cc;
    const float y = xch[cc * kXchLd + r];
    switch (e.op) {
      case kOpStore:
        e.out[(size_t)c * e.out_ld + mt * kBM + r] = y;
        break;
      case kOpResid:
        e.out[(size_t)c * e.out_ld + mt * kBM + r] += y;
        break;
      case kOpSwiglu:
        if (r < 64) {
          const float g = y, u = xch[cc * kXchLd + r + 64];
          const float a = __fmul_rn(__fdiv_rn(g, __fadd_rn(1.0f, expf(-g))), u);
          e.xf[(size_t)c * e.f + mt * 64 + r] = __float2bfloat16_rn(a);
        }
        break;
      default: {  // kOpQkv: tile mt is head mt of [q heads | k heads | v heads]
        float o = y;
        if (mt < e.H + e.KV) {
          const int i = r & 63;
          const float cs = e.rope[((size_t)c * 64 + i) * 2], sn = e.rope[((size_t)c * 64 + i) * 2 + 1];
          const float pr = xch[cc * kXchLd + (r ^ 64)];
          o = r < 64 ? __fsub_rn(__fmul_rn(y, cs), __fmul_rn(pr, sn)) : __fadd_rn(__fmul_rn(y, cs), __fmul_rn(pr, sn));
        }
        __nv_bfloat16* dst;
        if (mt < e.H) {
          dst = e.xq + (size_t)c * e.H * kBM + mt * kBM;
        } else {
          const bool is_k = mt < e.H + e.KV;
          const int kh = is_k ? mt - e.H : mt - e.H - e.KV;
          if (e.append)
            dst = (is_k ? e.kc : e.vc) + ((size_t)kh * e.cap + e.row0 + c) * kBM;
          else
            dst = (is_k ? e.kself : e.vself) + ((size_t)c * e.KV + kh) * kBM;
        }
        dst[r] = __float2bfloat16_rn(o);
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    sk_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, SkPlan p,
                   int stages, GemmEpi e) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ int s_last;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int c = blockIdx.x;
  const int t0 = sk_begin(p, c), t1 = sk_begin(p, c + 1);
  const int bbytes = p.n_pad * 128;
  uint8_t* sA = smem;
  uint8_t* sB = smem + stages * kABytes;
  float* xch = reinterpret_cast<float*>(sB + stages * bbytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(xch) + kXchBytes);
  uint64_t* empty = full + kMaxStages;
  uint64_t* tfull = empty + kMaxStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tholder = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t ncols = 32;
  while (ncols < (uint32_t)(2 * p.n_pad)) ncols <<= 1;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tholder, ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = *tholder;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch(&tmA);
      tma_prefetch(&tmB);
      const uint64_t pol_w = policy_evict_first(), pol_x = policy_evict_last();
      const int nbox = p.n_pad / 16;
      // weights do not depend on the previous kernel: fill the ring now
      const int npre = min(stages, t1 - t0);
      for (int j = 0; j < npre; ++j) {
        const int t = t0 + j;
        mbar_expect_tx(&full[j], kABytes + bbytes);
        tma_load_2d(sA + j * kABytes, &tmA, (t % p.KB) * kBK, (t / p.KB) * kBM, &full[j], pol_w);
      }
      pdl_wait();  // node rows X come from the previous kernel
      pdl_trigger();
      for (int j = 0; j < npre; ++j) {
        const int kb = (t0 + j) % p.KB;
        for (int b = 0; b < nbox; ++b)
          tma_load_2d(sB + j * bbytes + b * 2048, &tmB, kb * kBK, b * 16, &full[j], pol_x);
      }
      int stage = npre % stages;
      uint32_t phase = npre == stages ? 1 : 0;
      for (int t = t0 + npre; t < t1; ++t) {
        const int mt = t / p.KB, kb = t % p.KB;
        mbar_wait(&empty[stage], phase ^ 1);
        mbar_expect_tx(&full[stage], kABytes + bbytes);
        tma_load_2d(sA + stage * kABytes, &tmA, kb * kBK, mt * kBM, &full[stage], pol_w);
        for (int b = 0; b < nbox; ++b)
          tma_load_2d(sB + stage * bbytes + b * 2048, &tmB, kb * kBK, b * 16, &full[stage], pol_x);
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16_f32(kBM, p.n_pad);
      int stage = 0, seg = 0;
      uint32_t phase = 0;
      int t = t0;
      while (t < t1) {
        const int mt = t / p.KB;
        const int seg_start = t, seg_end = min(t1, (mt + 1) * p.KB);
        const int buf = seg & 1;
        const uint32_t bphase = (seg >> 1) & 1;
        mbar_wait(&tempty[buf], bphase ^ 1);
        tc_fence_after();
        const uint32_t d = taddr + buf * p.n_pad;
        for (; t < seg_end; ++t) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = desc_kmajor_sw128(sA + stage * kABytes);
          const uint64_t bd = desc_kmajor_sw128(sB + stage * bbytes);
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
        ++seg;
      }
    }
  } else {
    const int quarter = warp & 3;  // TMEM lanes this warp may touch
    const int r = quarter * 32 + lane;
    const int et = threadIdx.x - 64;
    int seg = 0, t = t0;
    while (t < t1) {
      const int mt = t / p.KB;
      const int seg_end = min(t1, (mt + 1) * p.KB);
      const int buf = seg & 1;
      const uint32_t bphase = (seg >> 1) & 1;
      const int cfirst = sk_cta_of(p, mt * p.KB);
      const int cnt = sk_cta_of(p, (mt + 1) * p.KB - 1) - cfirst + 1;
      mbar_wait(&tfull[buf], bphase);
      tc_fence_after();
      const uint32_t tbase = taddr + ((uint32_t)(quarter * 32) << 16) + buf * p.n_pad;
      bool last = true;
      if (cnt > 1) {
        float* dst = e.part + ((size_t)(mt * p.max_contrib + (c - cfirst)) * p.n) * kBM + r;
        for (int col0 = 0; col0 < p.n_pad; col0 += 16) {
          float v[16];
          tmem_ld_x16(tbase + col0, v);
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (col0 + i < p.n) __stcg(dst + (size_t)(col0 + i) * kBM, v[i]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);  // TMEM free: the MMA may go on
        __threadfence();
        epi_bar();
        if (et == 0) s_last = atomicAdd(&e.counters[mt], 1) == cnt - 1;
        epi_bar();
        last = s_last;
        if (last) __threadfence();
      }
      if (last) {
        const float* src = e.part + ((size_t)mt * p.max_contrib * p.n) * kBM + r;
        const size_t slot = (size_t)p.n * kBM;
        for (int c0 = 0; c0 < p.n; c0 += kXchNodes) {
          const int cn = min(kXchNodes, p.n - c0);
          if (cnt == 1) {
            for (int col0 = c0; col0 < min(c0 + kXchNodes, p.n_pad); col0 += 16) {
              float v[16];
              tmem_ld_x16(tbase + col0, v);
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (col0 + i < p.n) xch[(col0 - c0 + i) * kXchLd + r] = v[i];
            }
          } else {
            for (int cc = 0; cc < cn; ++cc) {
              const float* b = src + (size_t)(c0 + cc) * kBM;
              float v[8];
#pragma unroll
              for (int s = 0; s < 8; ++s) v[s] = s < cnt ? __ldcg(b + s * slot) : 0.f;
              float acc = v[0];
#pragma unroll
              for (int s = 1; s < 8; ++s)
                if (s < cnt) acc += v[s];
              for (int s = 8; s < cnt; ++s) acc += __ldcg(b + s * slot);
              xch[cc * kXchLd + r] = acc;
            }
          }
          epi_bar();
          apply_op(e, mt, r, c0, cn, xch);
          epi_bar();
        }
        if (cnt > 1 && et == 0) e.counters[mt] = 0;
      }
      if (cnt == 1) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
      }
      t = seg_end;
      ++seg;
    }
  }
  __syncthreads();
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
};
static std::vector<ProfRec> g_prof;
static bool g_prof_on = false;
static std::mutex g_prof_mu;

int sk_gemm(const CUtensorMap* tmA, const CUtensorMap* tmB, const SkPlan& p, const GemmEpi& epi, cudaStream_t st) {
  TP_CHECK(p.n >= 1 && p.n_pad <= 256, TP_ESHAPE, "GEMM node count outside [1, 256]");
  TP_CHECK(epi.counters && epi.part, TP_ECONFIG, "GEMM epilogue needs partial + counter scratch");
  const int stages = stages_for(p.n_pad);
  const size_t smem = smem_for(p.n_pad);
  static size_t smem_set = 0;
  if (smem > smem_set) {
    TP_CUDA(cudaFuncSetAttribute(sk_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    smem_set = smem;
  }
  ProfRec rec{};
  if (g_prof_on) {
    TP_CUDA(cudaEventCreate(&rec.a));
    TP_CUDA(cudaEventCreate(&rec.b));
    TP_CUDA(cudaEventRecord(rec.a, st));
    rec.bytes = (double)p.mtiles * kBM * p.KB * kBK * 2.0 + (double)p.n * p.KB * kBK * 2.0;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.G);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_prof_on ? 0 : 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ::tp::count_launch();
  TP_CUDA(cudaLaunchKernelEx(&cfg, sk_gemm_kernel, *tmA, *tmB, p, stages, epi));
  if (g_prof_on) {
    TP_CUDA(cudaEventRecord(rec.b, st));
    std::lock_guard<std::mutex> g(g_prof_mu);
    g_prof.push_back(rec);
  }
  return TP_OK;
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
  TP_CUDA(cudaMallocAsync((void**)&e.counters, p.mtiles * 4, st));
  TP_CUDA(cudaMemsetAsync(e.counters, 0, p.mtiles * 4, st));
  TP_TRY(sk_gemm(&ma, &mb, p, e, st));
  TP_CUDA(cudaFreeAsync(e.part, st));
  TP_CUDA(cudaFreeAsync(e.counters, st));
  TP_CUDA(cudaStreamSynchronize(st));
  return TP_OK;
}
