// Shared helpers for the treepipe_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <string>
#include <utility>

#include "../../include/treepipe_b200.h"

namespace tp {

void set_error(const std::string& msg);

struct Status {
  int code;
  std::string msg;
};

#define TP_CUDA(expr)                                                                        \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess) {                                                                 \
      ::tp::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));                   \
      return TP_ECUDA;                                                                       \
    }                                                                                        \
  } while (0)

#define TP_CHECK(cond, code, msg)                                                            \
  do {                                                                                       \
    if (!(cond)) {                                                                           \
      ::tp::set_error(msg);                                                                  \
      return (code);                                                                         \
    }                                                                                        \
  } while (0)

#define TP_TRY(expr)                                                                         \
  do {                                                                                       \
    int _s = (expr);                                                                         \
    if (_s != TP_OK) return _s;                                                              \
  } while (0)

// ---- LCG weight stream (reference model.py:28-44) -------------------------
constexpr uint64_t kLcgMul = 6364136223846793005ull;
constexpr uint64_t kLcgInc = 1442695040888963407ull;

// s -> a*s + c composed 2^i times, i = 0..63 (filled once per process)
struct LcgJump {
  uint64_t a[64];
  uint64_t c[64];
};

// Launch helpers -------------------------------------------------------------
inline int ceil_div(int a, int b) { return (a + b - 1) / b; }
inline int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_sum_f32(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max_f32(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace tp

namespace tp {
// Programmatic dependent launch (PDL): kernels launched with launch_pdl start as
// soon as every CTA of the previous kernel has started (or triggered); they call
// pdl_wait() before touching anything an earlier kernel produced and
// pdl_trigger() so the next kernel can do the same.  No-ops without PDL.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
}  // namespace tp

namespace tp {
// Every kernel launch site calls this (`count_launch(), k<<<...>>>(...)`), so the
// bench can report how many of our kernels ran inside its timed region.
void count_launch();
}  // namespace tp
