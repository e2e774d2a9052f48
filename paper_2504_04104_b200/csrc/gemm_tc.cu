// K2: weight-streaming GEMM on 5th-gen tensor cores (tcgen05 + TMEM + TMA), swap-AB.
//
//   out[node, j] = sum_k X[node, k] * W[j, k]       (W: [N_out, K] bf16, K-major)
//
// A tree level has at most a few dozen nodes, so the *weights* are the MMA's
// M operand (128-row tiles) and the nodes its N operand (n_pad = 16..256
// columns): D^T[128 x n_pad] += W_tile[128 x 64] . X_tile[n_pad x 64]^T with the
// accumulator in TMEM.  The kernel is HBM-bound (arithmetic intensity ~n_pad
// FLOP/B), so the design goal is keeping every SM's TMA queue full:
//   * stream-K decomposition: the m-tile x k-block space is cut into one
//     contiguous range per CTA (grid = #SMs), so every SM streams the same
//     number of weight bytes regardless of N_out / K;
//   * warp-specialised: warp 0 = TMA producer (6-stage smem ring, weights
//     evict-first, node rows evict-last), warp 1 = single-thread MMA issuer,
//     warps 2-5 = epilogue draining TMEM (double-buffered accumulators so the
//     MMA of the next m-tile segment overlaps the drain of the previous one);
//   * partial tiles go to a [m_tile][contributor][node][128] fp32 buffer and
//     the fused epilogue kernels (llama.cu) sum contributors in fixed order.
// Determinism / batch invariance: segment boundaries depend only on
// (N_out, K, #SMs), never on the node count, and each output column's
// accumulation chain is the same for any n.
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
  int per = kABytes + n_pad * 128;
  return std::min(kMaxStages, (200 * 1024) / per);
}

static size_t smem_for(int n_pad) {
  return (size_t)stages_for(n_pad) * (kABytes + n_pad * 128) + 1024 /*align*/ + 256 /*barriers*/;
}

// ---- device --------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 1)
    sk_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, SkPlan p,
                   int stages, float* __restrict__ part) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int c = blockIdx.x;
  const int t0 = sk_begin(p, c), t1 = sk_begin(p, c + 1);
  const int bbytes = p.n_pad * 128;
  uint8_t* sA = smem;
  uint8_t* sB = smem + stages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + stages * bbytes);
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
      int stage = 0;
      uint32_t phase = 0;
      const int nbox = p.n_pad / 16;
      for (int t = t0; t < t1; ++t) {
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
    const int row = quarter * 32 + lane;
    int seg = 0, t = t0;
    while (t < t1) {
      const int mt = t / p.KB;
      const int seg_end = min(t1, (mt + 1) * p.KB);
      const int buf = seg & 1;
      const uint32_t bphase = (seg >> 1) & 1;
      mbar_wait(&tfull[buf], bphase);
      tc_fence_after();
      const int slot = c - sk_cta_of(p, mt * p.KB);
      float* dst = part + ((size_t)(mt * p.max_contrib + slot) * p.n) * kBM + row;
      const uint32_t tbase = taddr + ((uint32_t)(quarter * 32) << 16) + buf * p.n_pad;
      for (int col0 = 0; col0 < p.n; col0 += 16) {
        float v[16];
        tmem_ld_x16(tbase + col0, v);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (col0 + i < p.n) dst[(size_t)(col0 + i) * kBM] = v[i];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
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

int sk_gemm(const CUtensorMap* tmA, const CUtensorMap* tmB, const SkPlan& p, float* part, cudaStream_t st) {
  TP_CHECK(p.n >= 1 && p.n_pad <= 256, TP_ESHAPE, "GEMM node count outside [1, 256]");
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
  ::tp::count_launch(), sk_gemm_kernel<<<p.G, kThreads, smem, st>>>(*tmA, *tmB, p, stages, part);
  TP_CUDA(cudaGetLastError());
  if (g_prof_on) {
    TP_CUDA(cudaEventRecord(rec.b, st));
    std::lock_guard<std::mutex> g(g_prof_mu);
    g_prof.push_back(rec);
  }
  return TP_OK;
}

__global__ void sk_reduce_kernel(const float* __restrict__ part, SkPlan p, int n_out, float* __restrict__ out) {
  const int c = blockIdx.x, j = blockIdx.y * blockDim.x + threadIdx.x;
  if (j < n_out) out[(size_t)c * n_out + j] = sk_sum(part, p, c, j);
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
  float* part = nullptr;
  TP_CUDA(cudaMallocAsync((void**)&part, sk_part_floats(p) * 4, st));
  TP_TRY(sk_gemm(&ma, &mb, p, part, st));
  ::tp::count_launch(), sk_reduce_kernel<<<dim3(n, (n_out + 255) / 256), 256, 0, st>>>(part, p, n_out, (float*)out_dev);
  TP_CUDA(cudaGetLastError());
  TP_CUDA(cudaFreeAsync(part, st));
  TP_CUDA(cudaStreamSynchronize(st));
  return TP_OK;
}
