// K5: on-device LCG weight stream, bit-exact with the reference generator
// (`/root/reference/pkg/src/treepipe/model.py:33-44`).
//
// state_{i+1} = state_i * 6364136223846793005 + 1442695040888963407 (mod 2^64)
// sample_i    = ((state_i >> 11) * 2^-53) * 0.2 - 0.1, each op rounded
// separately (no FMA contraction: __dmul_rn / __dsub_rn).
// Every thread jumps straight to its first element with the 2^k composed
// maps held in constant memory, then steps sequentially through a run.
#include "internal.h"

namespace tp {

__constant__ LcgJump c_jump;

int fill_lcg_jump_table() {
  static bool done = false;
  if (done) return TP_OK;
  LcgJump j;
  uint64_t a = kLcgMul, c = kLcgInc;
  for (int i = 0; i < 64; ++i) {
    j.a[i] = a;
    j.c[i] = c;
    c = a * c + c;  // (a,c) o (a,c)
    a = a * a;
  }
  TP_CUDA(cudaMemcpyToSymbol(c_jump, &j, sizeof(j)));
  done = true;
  return TP_OK;
}

__device__ __forceinline__ uint64_t lcg_state(uint64_t seed, uint64_t idx) {
  // state after idx steps from seed
  uint64_t a = 1, c = 0;
  for (int i = 0; idx; ++i, idx >>= 1) {
    if (idx & 1) {
      c = c_jump.a[i] * c + c_jump.c[i];
      a = c_jump.a[i] * a;
    }
  }
  return a * seed + c;
}

__device__ __forceinline__ double lcg_sample(uint64_t s) {
  double u = (double)(s >> 11) * 0x1p-53;
  return __dsub_rn(__dmul_rn(u, 0.2), 0.1);
}

constexpr int kRun = 64;

__global__ void lcg_f64_kernel(double* __restrict__ out, int64_t count, uint64_t seed, int64_t start) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t e0 = t * kRun;
  if (e0 >= count) return;
  int64_t e1 = min(count, e0 + kRun);
  uint64_t s = lcg_state(seed, (uint64_t)(start + e0 + 1));
  for (int64_t e = e0; e < e1; ++e) {
    out[e] = lcg_sample(s);
    s = s * kLcgMul + kLcgInc;
  }
}

__device__ __forceinline__ __nv_bfloat16 to_bf16(uint64_t s, double scale) {
  return __float2bfloat16_rn(__double2float_rn(__dmul_rn(lcg_sample(s), scale)));
}

// [rows_in, cols_out] in stream order, stored transposed: column j -> dst row
// map(j) (= j + row_offset, or the 64-row gate/up interleave), element i.
__global__ void lcg_bf16_t_kernel(__nv_bfloat16* __restrict__ out, int64_t rows_in, int64_t cols_out,
                                  uint64_t seed, int64_t start, double scale, int64_t row_offset,
                                  int interleave64) {
  int64_t count = rows_in * cols_out;
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t e0 = t * kRun;
  if (e0 >= count) return;
  int64_t e1 = min(count, e0 + kRun);
  uint64_t s = lcg_state(seed, (uint64_t)(start + e0 + 1));
  int64_t i = e0 / cols_out, j = e0 % cols_out;
  for (int64_t e = e0; e < e1; ++e) {
    int64_t row = interleave64 ? (j / 64) * 128 + (j % 64) + row_offset : j + row_offset;
    out[row * rows_in + i] = to_bf16(s, scale);
    s = s * kLcgMul + kLcgInc;
    if (++j == cols_out) {
      j = 0;
      ++i;
    }
  }
}

__global__ void lcg_bf16_kernel(__nv_bfloat16* __restrict__ out, int64_t count, uint64_t seed, int64_t start,
                                double scale) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t e0 = t * kRun;
  if (e0 >= count) return;
  int64_t e1 = min(count, e0 + kRun);
  uint64_t s = lcg_state(seed, (uint64_t)(start + e0 + 1));
  for (int64_t e = e0; e < e1; ++e) {
    out[e] = to_bf16(s, scale);
    s = s * kLcgMul + kLcgInc;
  }
}

int lcg_fill_f64(double* out, int64_t count, uint64_t seed, int64_t start, cudaStream_t st) {
  TP_TRY(fill_lcg_jump_table());
  int64_t threads = ceil_div64(count, kRun);
  int block = 256;
  ::tp::count_launch(), lcg_f64_kernel<<<(unsigned)ceil_div64(threads, block), block, 0, st>>>(out, count, seed, start);
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

int lcg_fill_bf16_rows(__nv_bfloat16* out, int64_t rows_in, int64_t cols_out, uint64_t seed, int64_t start,
                       double scale, int64_t row_offset, int interleave64, cudaStream_t st) {
  TP_TRY(fill_lcg_jump_table());
  int64_t threads = ceil_div64(rows_in * cols_out, kRun);
  int block = 256;
  ::tp::count_launch(), lcg_bf16_t_kernel<<<(unsigned)ceil_div64(threads, block), block, 0, st>>>(out, rows_in, cols_out, seed,
                                                                           start, scale, row_offset,
                                                                           interleave64);
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

int lcg_fill_bf16(__nv_bfloat16* out, int64_t count, uint64_t seed, int64_t start, double scale,
                  cudaStream_t st) {
  TP_TRY(fill_lcg_jump_table());
  int64_t threads = ceil_div64(count, kRun);
  ::tp::count_launch(), lcg_bf16_kernel<<<(unsigned)ceil_div64(threads, 256), 256, 0, st>>>(out, count, seed, start, scale);
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

}  // namespace tp
