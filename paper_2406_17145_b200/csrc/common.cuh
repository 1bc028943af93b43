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

// Activations. GELU is the exact erf form (torch.nn.functional.gelu default).
__device__ __forceinline__ float act_fwd(float x, int act) {
  if (act == GPP_ACT_RELU) return x > 0.f ? x : 0.f;
  if (act == GPP_ACT_GELU) return 0.5f * x * (1.f + erff(x * 0.70710678118654752f));
  return x;
}
// Derivative given the saved tensor: RELU saved = activation OUTPUT, GELU saved = pre-activation.
__device__ __forceinline__ float act_bwd(float saved, int act) {
  if (act == GPP_ACT_RELU) return saved > 0.f ? 1.f : 0.f;
  if (act == GPP_ACT_GELU) {
    const float cdf = 0.5f * (1.f + erff(saved * 0.70710678118654752f));
    const float pdf = 0.39894228040143268f * __expf(-0.5f * saved * saved);
    return cdf + saved * pdf;
  }
  return 1.f;
}

inline int dtype_bytes(int dtype) { return dtype == GPP_BF16 ? 2 : 4; }

}  // namespace gpp
