// Stream-K tcgen05 GEMM plan + launcher (see gemm_tc.cu).
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace tp {

struct SkPlan {
  int mtiles;       // N_out / 128
  int KB;           // K / 64
  int total;        // mtiles * KB k-blocks, linearised m-major
  int G, q, r;      // CTAs; CTA c owns q (+1 if c < r) consecutive k-blocks
  int max_contrib;  // max CTAs contributing to one m-tile
  int n, n_pad;     // valid node columns / MMA N
};

__host__ __device__ inline int sk_begin(const SkPlan& p, int c) { return c * p.q + (c < p.r ? c : p.r); }
__host__ __device__ inline int sk_cta_of(const SkPlan& p, int t) {
  const int big = p.r * (p.q + 1);
  return t < big ? t / (p.q + 1) : p.r + (t - big) / p.q;
}

// Sum of one output element over its contributors, in fixed order.  All
// contributor loads are issued before the (ordered) adds so the reduction is
// one L2 round trip, not max_contrib dependent ones.
__device__ __forceinline__ float sk_sum(const float* __restrict__ part, const SkPlan& p, int node, int j) {
  const int mt = j >> 7, r = j & 127;
  const int cnt = sk_cta_of(p, (mt + 1) * p.KB - 1) - sk_cta_of(p, mt * p.KB) + 1;
  const float* b = part + ((size_t)mt * p.max_contrib * p.n + node) * 128 + r;
  const size_t stride = (size_t)p.n * 128;
  float v[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) v[s] = s < cnt ? __ldcg(b + s * stride) : 0.f;
  float acc = v[0];
#pragma unroll
  for (int s = 1; s < 8; ++s)
    if (s < cnt) acc += v[s];
  for (int s = 8; s < cnt; ++s) acc += __ldcg(b + s * stride);
  return acc;
}

int num_sms();
int make_tmap_kmajor(CUtensorMap* map, const void* gptr, int64_t rows, int64_t k, int box_rows);
SkPlan sk_plan(int n_out, int k, int n);
inline size_t sk_part_floats(const SkPlan& p) { return (size_t)p.mtiles * p.max_contrib * p.n * 128; }
int sk_gemm(const CUtensorMap* tmA, const CUtensorMap* tmB, const SkPlan& p, float* part, cudaStream_t st);

}  // namespace tp
