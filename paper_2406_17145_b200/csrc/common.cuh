// Shared helpers for the sm_100a stage-executor kernels (libgpp_b200.so).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>

#include "../../include/gpp_b200.h"

namespace gpp {

// Thread-local last-error string behind gpp_last_error() (SURVEY.md §8(b) "Errors").
void set_error(const std::string& msg);
void count_launch();

#define GPP_ARG_CHECK(cond, msg)              \
  do {                                        \
    if (!(cond)) {                            \
      ::gpp::set_error(std::string(__func__) + ": " + (msg)); \
      return GPP_ERR_ARG;                     \
    }                                         \
  } while (0)

#define GPP_LAUNCH_CHECK()                                                           \
  do {                                                                               \
    cudaError_t e__ = cudaGetLastError();                                            \
    if (e__ != cudaSuccess) {                                                        \
      ::gpp::set_error(std::string(__func__) + ": " + cudaGetErrorString(e__));      \
      return GPP_ERR_CUDA;                                                           \
    }                                                                                \
    ::gpp::count_launch();                                                           \
  } while (0)

using bf16 = __nv_bfloat16;

template <typename T> __device__ __forceinline__ float to_f(T v);
template <> __device__ __forceinline__ float to_f<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f<bf16>(bf16 v) { return __bfloat162float(v); }

template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }

// Activations.  GELU is the tanh form (torch gelu(approximate="tanh")):
//   gelu(x) = x/2 (1 + tanh u),  u = sqrt(2/pi) (x + 0.044715 x^3),
// evaluated with the SFU's tanh.approx.f32 (|error| < 2^-10.9): ONE MUFU op and five FMA-pipe
// ops per element.  The GEMM epilogues apply it to 8192 x 4096 tiles; the earlier
// x * sigmoid(2u) form took two MUFU ops (ex2 + rcp) and four more instructions, and the
// FFN1 forward epilogue (bias + GELU + pre-activation store) ran 18 us behind the plain one.
// The absolute error (< 2.5e-4 |x| on the output) is below bf16 resolution of the results.
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float act_fwd(float x, int act) {
  if (act == GPP_ACT_RELU) return x > 0.f ? x : 0.f;
  if (act == GPP_ACT_GELU) {
    const float u = x * fmaf(0.0356774081f * x, x, 0.7978845608f);
    const float hx = 0.5f * x;
    return fmaf(hx, tanh_approx(u), hx);
  }
  return x;
}
// Derivative given the saved tensor: RELU saved = activation OUTPUT, GELU saved = pre-activation.
//   gelu'(x) = (1 + t) / 2 + x/2 (1 - t^2) u',  t = tanh u,  u' = sqrt(2/pi) (1 + 3 * 0.044715 x^2)
__device__ __forceinline__ float act_bwd(float saved, int act) {
  if (act == GPP_ACT_RELU) return saved > 0.f ? 1.f : 0.f;
  if (act == GPP_ACT_GELU) {
    const float x2 = saved * saved;
    const float t = tanh_approx(saved * fmaf(0.0356774081f, x2, 0.7978845608f));
    const float du = fmaf(0.1070322243f, x2, 0.7978845608f);
    const float a = 0.5f * saved * fmaf(-t, t, 1.f);
    return fmaf(0.5f, t, fmaf(a, du, 0.5f));
  }
  return 1.f;
}

inline int dtype_bytes(int dtype) { return dtype == GPP_BF16 ? 2 : 4; }

// Programmatic dependent launch.  Kernels started by launch_pdl may begin while the
// previous kernel of the stream drains (its CTAs have all issued pdl_trigger); they run
// their prologue (barrier init, TMEM alloc, tensormap prefetch) and then block in
// pdl_wait() until that kernel has completed and its writes are visible.  Every kernel
// launched this way calls pdl_wait() before its first global access (and before any
// early return), so completion stays transitive along the stream.  For a kernel launched
// without the attribute both instructions are no-ops.  GPP_PDL (a bit mask over the kernel
// families, GPP_PDL_CLASS of each translation unit; default all but 16) selects where it is used.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled(int family);
#ifndef GPP_PDL_CLASS
#define GPP_PDL_CLASS 0
#endif

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_impl(int family, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                   cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled(family) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
#define launch_pdl(...) launch_pdl_impl(GPP_PDL_CLASS, __VA_ARGS__)

}  // namespace gpp
