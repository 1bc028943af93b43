#include <algorithm>
// C-ABI entry points (include/gpp_b200.h) and the SIMT kernels around the GEMMs:
// N=1 heads, fused losses, bias-grad column sums, the fused SGD step, casts and
// strided row copies.  All memory-bound; vectorised where alignment allows.
#include <atomic>
#include <cstdlib>
#include <string>

#define GPP_PDL_CLASS 8  // programmatic-dependent-launch family: heads, column sums, SGD, copies
#include "gemm.cuh"

namespace gpp {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }

static thread_local const void* g_pf_ptr = nullptr;
static thread_local int64_t g_pf_bytes = 0;
void take_prefetch_hint(EpiParams& ep) {
  ep.pf_ptr = g_pf_ptr;
  ep.pf_bytes = g_pf_bytes;
  g_pf_ptr = nullptr;
  g_pf_bytes = 0;
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
// Default: every family except the embedding bags (16), measured 0.45 ms per DLRM step
// slower with PDL (profiles/pdl_r2.json); GEMM / attention / LN / head kernels gain 1-4%.
bool pdl_enabled(int family) {
  static const long mask = [] { const char* e = std::getenv("GPP_PDL"); return e ? std::strtol(e, nullptr, 0) : ~16L; }();
  return (mask & family) != 0;
}

namespace {

template <typename T>
__device__ __forceinline__ T ld(const void* p, int64_t i) {
  return static_cast<const T*>(p)[i];
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum; every thread receives the result.  blockDim.x multiple of 32, <= 1024.
__device__ float block_sum(float v) {
  __shared__ float red[32];
  __shared__ float total;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    float s = lane < (blockDim.x >> 5) ? red[lane] : 0.f;
    s = warp_sum(s);
    if (lane == 0) total = s;
  }
  __syncthreads();
  return total;
}

__device__ float block_max(float v) {
  __shared__ float red[32];
  __shared__ float total;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    float s = lane < (blockDim.x >> 5) ? red[lane] : -INFINITY;
    s = warp_max(s);
    if (lane == 0) total = s;
  }
  __syncthreads();
  return total;
}

// ---------------- heads ----------------
template <typename T>
__global__ void rowdot_fwd_kernel(float* out, const T* x, int64_t ldx, const float* w,
                                  const float* bias, int64_t M, int64_t K) {
  pdl_wait();
  pdl_trigger();
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const T* xr = x + row * ldx;
  float s = 0.f;
  for (int64_t k = lane; k < K; k += 32) s = fmaf(to_f<T>(xr[k]), w[k], s);
  s = warp_sum(s);
  if (lane == 0) out[row] = s + (bias ? bias[0] : 0.f);
}

// Fused N=1 head + loss: z[m] = dot(x[m,:K], w) + b, then MSE (kind 0: l = (z-y)^2,
// dz = 2 scale (z-y)) or BCE-with-logits (kind 1: dz = scale (sigmoid(z) - y)); one warp per
// row (16-byte bf16 loads when K % 256 == 0), per-block loss partials reduced in block
// order by the last block to arrive (deterministic; the counter re-arms for graph replay).
template <typename T>
__global__ void __launch_bounds__(256) rowdot_loss_kernel(float* __restrict__ z, float* __restrict__ dz,
                                                          float* __restrict__ loss_acc, float* __restrict__ part,
                                                          unsigned* __restrict__ counter, const T* __restrict__ x,
                                                          int64_t ldx, const float* __restrict__ w,
                                                          const float* __restrict__ bias,
                                                          const float* __restrict__ y, int64_t M, int64_t K,
                                                          int kind, float scale) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[8];
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + warp;
  float l = 0.f;
  if (row < M) {
    const T* xr = x + row * ldx;
    float s = 0.f;
    if constexpr (sizeof(T) == 2) {
      if (K % 256 == 0 && ldx % 8 == 0) {
        for (int64_t k = lane * 8; k < K; k += 256) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(xr + k));
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float2 f = __bfloat1622float2(h[t]);
            s = fmaf(f.x, __ldg(w + k + 2 * t), fmaf(f.y, __ldg(w + k + 2 * t + 1), s));
          }
        }
      } else {
        for (int64_t k = lane; k < K; k += 32) s = fmaf(to_f<T>(xr[k]), w[k], s);
      }
    } else {
      for (int64_t k = lane; k < K; k += 32) s = fmaf(to_f<T>(xr[k]), w[k], s);
    }
    s = warp_sum(s);
    if (lane == 0) {
      const float zi = s + (bias ? bias[0] : 0.f), yi = y[row];
      z[row] = zi;
      if (kind == 0) {
        const float d = zi - yi;
        l = d * d;
        dz[row] = 2.f * scale * d;
      } else {
        l = fmaxf(zi, 0.f) - zi * yi + log1pf(__expf(-fabsf(zi)));
        dz[row] = scale * (1.f / (1.f + __expf(-zi)) - yi);
      }
    }
  }
  if (lane == 0) red[warp] = l;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += red[i];
    part[blockIdx.x] = t;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  float t = 0.f;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) t += __ldcg(part + i);
  t = block_sum(t);
  if (threadIdx.x == 0) {
    loss_acc[0] += scale * t;
    *counter = 0;
  }
}

template <typename T>
__global__ void rowdot_dx_kernel(T* dx, int64_t lddx, const float* dout, const float* w,
                                 const T* saved, int64_t ldsaved, int act, int64_t M, int64_t K) {
  pdl_wait();
  pdl_trigger();
  const int64_t n = M * K;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t m = i / K, k = i % K;
    float v = dout[m] * w[k];
    if (act != GPP_ACT_NONE) v *= act_bwd(to_f<T>(saved[m * ldsaved + k]), act);
    dx[m * lddx + k] = from_f<T>(v);
  }
}

// bf16 rows of K % 8 == 0: 8 columns (one 16 B vector of dx / saved) per thread, 32-bit
// indices.  The scalar kernel above ran the DLRM head (8192 x 4096) at ~1.5 TB/s.
__global__ void __launch_bounds__(256) rowdot_dx_vec_kernel(bf16* dx, int64_t lddx, const float* dout,
                                                            const float* w, const bf16* saved,
                                                            int64_t ldsaved, int act, uint32_t M,
                                                            uint32_t K8) {
  pdl_wait();
  pdl_trigger();
  const uint32_t n = M * K8;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t m = i / K8, k = (i % K8) * 8;
    const float d = dout[m];
    float v[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) v[t] = d * __ldg(w + k + t);  // w: K floats, L1-resident
    if (act != GPP_ACT_NONE) {
      const uint4 sv = __ldcs(reinterpret_cast<const uint4*>(saved + static_cast<int64_t>(m) * ldsaved + k));
      const bf16* sp = reinterpret_cast<const bf16*>(&sv);
#pragma unroll
      for (int t = 0; t < 8; ++t) v[t] *= act_bwd(__bfloat162float(sp[t]), act);
    }
    uint4 o;
    bf16* op = reinterpret_cast<bf16*>(&o);
#pragma unroll
    for (int t = 0; t < 8; ++t) op[t] = __float2bfloat16(v[t]);
    *reinterpret_cast<uint4*>(dx + static_cast<int64_t>(m) * lddx + k) = o;
  }
}

// out[0] (+)= sum_m v[m]: one block, fixed-order (per-thread strided sums, then block_sum).
__global__ void __launch_bounds__(1024) sum_kernel(float* out, const float* v, int64_t M, int accumulate) {
  pdl_wait();
  pdl_trigger();
  float s = 0.f;
  for (int64_t m = threadIdx.x; m < M; m += blockDim.x) s += v[m];
  s = block_sum(s);
  if (threadIdx.x == 0) out[0] = (accumulate ? out[0] : 0.f) + s;
}

// out[n] (+)= sum_m wts[m] * x[m, n]   (wts == nullptr -> 1).  Deterministic:
// block = 8 row-groups x 32 columns, fixed-order smem reduction.
template <typename T>
__global__ void colsum_kernel(float* out, const T* x, int64_t ldx, const float* wts, int64_t M,
                              int64_t N, int accumulate) {
  __shared__ float part[8][33];
  const int c = threadIdx.x & 31, r = threadIdx.x >> 5;
  const int64_t col = static_cast<int64_t>(blockIdx.x) * 32 + c;
  float s = 0.f;
  if (col < N) {
    for (int64_t m = r; m < M; m += 8) {
      const float v = to_f<T>(x[m * ldx + col]);
      s = wts ? fmaf(wts[m], v, s) : s + v;
    }
  }
  part[r][c] = s;
  __syncthreads();
  if (r == 0 && col < N) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += part[i][c];
    out[col] = accumulate ? out[col] + t : t;
  }
}


// Bias-gradient column sums, deterministic two-pass.  Pass 1: block (64 columns x
// 8 warps) over a row split, lanes read 2 adjacent columns (one 4-byte bf16x2 /
// 8-byte float2 load -> 128/256 B per warp-row); fixed-order smem reduction into
// partial[split][col].  Pass 2 sums the partials in split order.
template <typename T>
__global__ void __launch_bounds__(256) colsum_part_kernel(float* part, const T* x, int64_t ldx,
                                                          const float* wts, int64_t M, int64_t N,
                                                          int64_t rows_per_split) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[8][65];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t col = static_cast<int64_t>(blockIdx.x) * 64 + lane * 2;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per_split;
  const int64_t r1 = min(M, r0 + rows_per_split);
  float s0 = 0.f, s1 = 0.f;
  if (col + 1 < N && ((ldx & 1) == 0)) {
    for (int64_t m = r0 + w; m < r1; m += 8) {
      const T* p = x + m * ldx + col;
      float a, b;
      if constexpr (sizeof(T) == 2) {
        const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(p);
        a = __low2float(v); b = __high2float(v);
      } else {
        const float2 v = *reinterpret_cast<const float2*>(p);
        a = v.x; b = v.y;
      }
      const float wt = wts ? wts[m] : 1.f;
      s0 = fmaf(wt, a, s0);
      s1 = fmaf(wt, b, s1);
    }
  } else {
    for (int64_t m = r0 + w; m < r1; m += 8) {
      const float wt = wts ? wts[m] : 1.f;
      if (col < N) s0 = fmaf(wt, to_f<T>(x[m * ldx + col]), s0);
      if (col + 1 < N) s1 = fmaf(wt, to_f<T>(x[m * ldx + col + 1]), s1);
    }
  }
  red[w][lane * 2] = s0;
  red[w][lane * 2 + 1] = s1;
  __syncthreads();
  if (threadIdx.x < 64) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += red[i][threadIdx.x];
    const int64_t c = static_cast<int64_t>(blockIdx.x) * 64 + threadIdx.x;
    if (c < N) part[static_cast<int64_t>(blockIdx.y) * N + c] = t;
  }
}

__global__ void colsum_final_kernel(float* out, const float* part, int splits, int64_t N,
                                    int accumulate) {
  pdl_wait();
  pdl_trigger();
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= N) return;
  float t = 0.f;
  for (int s = 0; s < splits; ++s) t += part[static_cast<int64_t>(s) * N + c];
  out[c] = accumulate ? out[c] + t : t;
}

// Single-launch column sums for aligned, unweighted inputs.  Block = 8 warps x 32 lanes,
// each lane owning VEC adjacent columns (one 16-byte load per row), so a block covers
// 32*VEC columns over one row split with 8 rows in flight per thread.  The block's
// fixed-order partial goes to part[split][col]; the last block of a column range to
// arrive (per-range arrival counter) sums the partials in split order and writes out,
// then re-arms its counter -- deterministic, and graph-replay safe.
template <typename T>
__device__ __forceinline__ void colsum_vec_body(float* out, float* part, unsigned* counters, const T* x,
                                                int64_t ldx, int64_t M, int64_t N, int64_t rows_per_split,
                                                int accumulate, unsigned bx, unsigned by, unsigned nsplit) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int CPB = 32 * VEC;
  constexpr int UNROLL = 8;
  __shared__ float red[8][CPB + 1];
  __shared__ bool is_last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t col = static_cast<int64_t>(bx) * CPB + lane * VEC;
  const int64_t r0 = static_cast<int64_t>(by) * rows_per_split;
  const int64_t r1 = min(M, r0 + rows_per_split);
  float acc[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) acc[j] = 0.f;
  auto add = [&](const uint4& v) {
    if constexpr (sizeof(T) == 2) {
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[2 * j] += __low2float(h[j]);
        acc[2 * j + 1] += __high2float(h[j]);
      }
    } else {
      const float* f = reinterpret_cast<const float*>(&v);
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] += f[j];
    }
  };
  if (col < N) {
    int64_t m = r0 + w;
    for (; m + 8 * (UNROLL - 1) < r1; m += 8 * UNROLL) {
      uint4 v[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) v[u] = __ldg(reinterpret_cast<const uint4*>(x + (m + 8 * u) * ldx + col));
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) add(v[u]);
    }
    for (; m < r1; m += 8) add(__ldg(reinterpret_cast<const uint4*>(x + m * ldx + col)));
  }
#pragma unroll
  for (int j = 0; j < VEC; ++j) red[w][lane * VEC + j] = acc[j];
  __syncthreads();
  const int64_t c = static_cast<int64_t>(bx) * CPB + threadIdx.x;
  if (threadIdx.x < CPB && c < N) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += red[i][threadIdx.x];
    part[static_cast<int64_t>(by) * N + c] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(&counters[bx], 1u) == nsplit - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  if (threadIdx.x < CPB && c < N) {
    float t = 0.f;
    for (unsigned sp = 0; sp < nsplit; ++sp) t += __ldcg(part + static_cast<int64_t>(sp) * N + c);
    out[c] = accumulate ? out[c] + t : t;
  }
  if (threadIdx.x == 0) counters[bx] = 0;
}

template <typename T>
__global__ void __launch_bounds__(256) colsum_vec_kernel(float* out, float* part, unsigned* counters,
                                                         const T* x, int64_t ldx, int64_t M,
                                                         int64_t N, int64_t rows_per_split,
                                                         int accumulate) {
  pdl_wait();
  pdl_trigger();
  colsum_vec_body<T>(out, part, counters, x, ldx, M, N, rows_per_split, accumulate, blockIdx.x, blockIdx.y,
                     gridDim.y);
}

// Several column sums in ONE launch (the bias gradients of a whole backward task): job i
// owns blocks [blk0, blk0 + vb * splits) of the 1-D grid, its own partial / counter ranges.
constexpr int kColsumJobs = 24;
struct ColsumJob {
  const void* x;
  float* out;
  int64_t ldx, M, N, rps;
  int part_off, cnt_off, vb, splits, blk0, pad;
};
struct ColsumJobs {
  ColsumJob j[kColsumJobs];
  int n, accumulate;
};

template <typename T>
__global__ void __launch_bounds__(256) colsum_multi_kernel(float* part, unsigned* counters,
                                                           const __grid_constant__ ColsumJobs jobs) {
  pdl_wait();
  pdl_trigger();
  const int b = static_cast<int>(blockIdx.x);
  int i = 0;
  while (i + 1 < jobs.n && b >= jobs.j[i + 1].blk0) ++i;
  const ColsumJob& jb = jobs.j[i];
  const int local = b - jb.blk0;
  colsum_vec_body<T>(jb.out, part + jb.part_off, counters + jb.cnt_off, static_cast<const T*>(jb.x), jb.ldx, jb.M,
                     jb.N, jb.rps, jobs.accumulate, static_cast<unsigned>(local % jb.vb),
                     static_cast<unsigned>(local / jb.vb), static_cast<unsigned>(jb.splits));
}

// Persistent per-device scratch for the partial sums and the arrival counters
// (allocated on first use, outside any graph capture: the first call happens in warm-up).
constexpr int64_t kScratchFloats = 4 << 20;
constexpr int64_t kCounters = 1 << 16;
float* colsum_scratch() {
  static float* bufs[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!bufs[dev]) {
    if (cudaMalloc(&bufs[dev], kScratchFloats * sizeof(float) + kCounters * sizeof(unsigned)) != cudaSuccess) {
      bufs[dev] = nullptr;
      return nullptr;
    }
    cudaMemset(bufs[dev] + kScratchFloats, 0, kCounters * sizeof(unsigned));
  }
  return bufs[dev];
}

template <typename T>
int colsum_launch(float* out, const T* x, int64_t ldx, const float* wts, int64_t M, int64_t N,
                  int accumulate, cudaStream_t s) {
  constexpr int VEC = 16 / sizeof(T);
  const int64_t vec_blocks = (N + 32 * VEC - 1) / (32 * VEC);
  if (!wts && N % VEC == 0 && ldx % VEC == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
      vec_blocks <= kCounters) {
    // ~4 blocks per SM, >= 64 rows (8 per warp) per split
    int64_t splits = (148 * 4 + vec_blocks - 1) / vec_blocks;
    if (splits > (M + 63) / 64) splits = (M + 63) / 64;
    if (splits < 1) splits = 1;
    while (splits > 1 && splits * N > kScratchFloats) --splits;
    float* part = colsum_scratch();
    if (!part) { set_error("colsum scratch allocation failed"); return GPP_ERR_CUDA; }
    const int64_t rps = (M + splits - 1) / splits;
    launch_pdl(colsum_vec_kernel<T>, dim3(dim3(static_cast<unsigned>(vec_blocks), static_cast<unsigned>(splits))), dim3(256), 0, s, out, part, reinterpret_cast<unsigned*>(part + kScratchFloats), x, ldx, M, N, rps, accumulate);
    GPP_LAUNCH_CHECK();
    return GPP_OK;
  }
  const int64_t col_blocks = (N + 63) / 64;
  int splits = static_cast<int>((148 * 4 + col_blocks - 1) / col_blocks);
  splits = splits < 1 ? 1 : (splits > 64 ? 64 : splits);
  if (splits > (M + 63) / 64) splits = static_cast<int>((M + 63) / 64);
  if (splits < 1) splits = 1;
  while (splits > 1 && static_cast<int64_t>(splits) * N > kScratchFloats) --splits;
  float* part = colsum_scratch();
  if (!part) { set_error("colsum scratch allocation failed"); return GPP_ERR_CUDA; }
  const int64_t rps = (M + splits - 1) / splits;
  launch_pdl(colsum_part_kernel<T>, dim3(dim3(static_cast<unsigned>(col_blocks), splits)), dim3(256), 0, s, part, x, ldx, wts, M, N, rps);
  GPP_LAUNCH_CHECK();
  launch_pdl(colsum_final_kernel, dim3(static_cast<unsigned>((N + 255) / 256)), dim3(256), 0, s, out, part, splits, N, accumulate);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

// colsum of several [M_i, N_i] tensors: vectorisable jobs share launches of <= kColsumJobs
// (partial and counter ranges laid out per job); the rest go through colsum_launch.
template <typename T>
int colsum_multi_launch(int n, const void* const* xs, const int64_t* lds, const int64_t* Ms, const int64_t* Ns,
                        float* const* outs, int accumulate, cudaStream_t s) {
  constexpr int VEC = 16 / sizeof(T);
  float* part = colsum_scratch();
  if (!part) { set_error("colsum scratch allocation failed"); return GPP_ERR_CUDA; }
  unsigned* counters = reinterpret_cast<unsigned*>(part + kScratchFloats);
  ColsumJobs jobs{};
  int64_t part_used = 0, cnt_used = 0, blocks = 0;
  auto flush = [&]() -> int {
    if (jobs.n == 0) return GPP_OK;
    jobs.accumulate = accumulate;
    launch_pdl(colsum_multi_kernel<T>, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, s, part, counters, jobs);
    GPP_LAUNCH_CHECK();
    jobs.n = 0;
    part_used = cnt_used = blocks = 0;
    return GPP_OK;
  };
  for (int i = 0; i < n; ++i) {
    const T* x = static_cast<const T*>(xs[i]);
    const int64_t M = Ms[i], N = Ns[i], ld = lds[i];
    GPP_ARG_CHECK(x && outs[i] && M > 0 && N > 0, "bad colsum job");
    const int64_t vb = (N + 32 * VEC - 1) / (32 * VEC);
    if (N % VEC != 0 || ld % VEC != 0 || (reinterpret_cast<uintptr_t>(x) & 15) != 0 || vb > kCounters) {
      const int rc = colsum_launch<T>(outs[i], x, ld, nullptr, M, N, accumulate, s);
      if (rc) return rc;
      continue;
    }
    int64_t splits = (148 * 4 + vb - 1) / vb;
    if (splits > (M + 63) / 64) splits = (M + 63) / 64;
    if (splits < 1) splits = 1;
    while (splits > 1 && splits * N > kScratchFloats) --splits;
    if (jobs.n == kColsumJobs || part_used + splits * N > kScratchFloats || cnt_used + vb > kCounters) {
      const int rc = flush();
      if (rc) return rc;
    }
    ColsumJob& jb = jobs.j[jobs.n++];
    jb.x = x;
    jb.out = outs[i];
    jb.ldx = ld;
    jb.M = M;
    jb.N = N;
    jb.rps = (M + splits - 1) / splits;
    jb.part_off = static_cast<int>(part_used);
    jb.cnt_off = static_cast<int>(cnt_used);
    jb.vb = static_cast<int>(vb);
    jb.splits = static_cast<int>(splits);
    jb.blk0 = static_cast<int>(blocks);
    part_used += splits * N;
    cnt_used += vb;
    blocks += vb * splits;
  }
  return flush();
}

// ---------------- losses (single block, deterministic reductions) ----------------
__global__ void mse_kernel(float* loss_acc, float* dpred, const float* pred, const float* y,
                           int64_t M, float scale) {
  pdl_wait();
  pdl_trigger();
  float s = 0.f;
  for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
    const float d = pred[i] - y[i];
    s = fmaf(d, d, s);
    dpred[i] = 2.f * scale * d;
  }
  s = block_sum(s);
  if (threadIdx.x == 0) loss_acc[0] += scale * s;
}

__global__ void bce_kernel(float* loss_acc, float* dz, const float* z, const float* y, int64_t M,
                           float scale) {
  pdl_wait();
  pdl_trigger();
  float s = 0.f;
  for (int64_t i = threadIdx.x; i < M; i += blockDim.x) {
    const float zi = z[i], yi = y[i];
    s += fmaxf(zi, 0.f) - zi * yi + log1pf(__expf(-fabsf(zi)));
    dz[i] = scale * (1.f / (1.f + __expf(-zi)) - yi);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) loss_acc[0] += scale * s;
}

// One block per row: softmax cross-entropy; writes dlogits, adds the row loss.
template <typename T>
__global__ void ce_kernel(float* loss_acc, T* dl, int64_t lddl, const T* logits, int64_t ldl,
                          const int64_t* labels, int64_t C, float scale) {
  pdl_wait();
  pdl_trigger();
  const int64_t row = blockIdx.x;
  const T* lr = logits + row * ldl;
  float mx = -INFINITY;
  for (int64_t c = threadIdx.x; c < C; c += blockDim.x) mx = fmaxf(mx, to_f<T>(lr[c]));
  mx = block_max(mx);
  float se = 0.f;
  for (int64_t c = threadIdx.x; c < C; c += blockDim.x) se += __expf(to_f<T>(lr[c]) - mx);
  se = block_sum(se);
  const float lse = mx + logf(se);
  const int64_t lab = labels[row];
  T* dr = dl + row * lddl;
  for (int64_t c = threadIdx.x; c < C; c += blockDim.x) {
    const float p = __expf(to_f<T>(lr[c]) - lse);
    dr[c] = from_f<T>(scale * (p - (c == lab ? 1.f : 0.f)));
  }
  if (threadIdx.x == 0) atomicAdd(loss_acc, scale * (lse - to_f<T>(lr[lab])));
}

// Strided row copy (concat / split of branch activations and their gradients): rows of
// `cv` vectors of type V, flattened over rows x cv, 4 independent loads in flight per thread.
// cudaMemcpy2DAsync ran these 8 MB slices at ~1 TB/s (copy-engine path); this is HBM-bound.
template <typename V, typename I>  // I: uint32_t index math when rows x cv < 2^32
__global__ void __launch_bounds__(256) copy_rows_kernel(V* __restrict__ dst, int64_t ldd,
                                                        const V* __restrict__ src, int64_t lds,
                                                        I cv, I n) {
  pdl_wait();
  pdl_trigger();
  constexpr int U = 4;
  const I stride = static_cast<I>(gridDim.x) * blockDim.x;
  for (I base = static_cast<I>(blockIdx.x) * blockDim.x + threadIdx.x; base < n; base += stride * U) {
    V v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const I i = base + u * stride;
      if (i < n) v[u] = __ldcs(src + (i / cv) * lds + (i % cv));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const I i = base + u * stride;
      if (i < n) dst[(i / cv) * ldd + (i % cv)] = v[u];
    }
  }
}

// Several slices of one concat / split in one launch: blockIdx.y = slice.  The descriptors
// travel by value in the kernel parameters, so a captured CUDA graph owns them.
constexpr int kMaxCopySlices = 32;
struct CopySlices {
  char* dst[kMaxCopySlices];
  const char* src[kMaxCopySlices];
  int64_t ldd[kMaxCopySlices], lds[kMaxCopySlices];  // in vectors
  uint32_t cv[kMaxCopySlices];                         // vectors per row
};

template <typename V>
__global__ void __launch_bounds__(256) copy_slices_kernel(const __grid_constant__ CopySlices d,
                                                          uint32_t rows) {
  pdl_wait();
  pdl_trigger();
  constexpr int U = 4;
  const int k = blockIdx.y;
  const uint32_t cv = d.cv[k], n = cv * rows;
  V* __restrict__ dst = reinterpret_cast<V*>(d.dst[k]);
  const V* __restrict__ src = reinterpret_cast<const V*>(d.src[k]);
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x + threadIdx.x; base < n; base += stride * U) {
    V v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = base + u * stride;
      if (i < n) v[u] = __ldcs(src + (i / cv) * d.lds[k] + (i % cv));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t i = base + u * stride;
      if (i < n) dst[(i / cv) * d.ldd[k] + (i % cv)] = v[u];
    }
  }
}

// ---------------- optimizer ----------------
__global__ void sgd_kernel(float* __restrict__ master, bf16* __restrict__ shadow,
                           const float* __restrict__ grad, int64_t n, float lr) {
  pdl_wait();
  pdl_trigger();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t n4 = n / 4;
  float4* m4 = reinterpret_cast<float4*>(master);
  const float4* g4 = reinterpret_cast<const float4*>(grad);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += stride) {
    float4 m = m4[i];
    const float4 g = g4[i];
    m.x -= lr * g.x; m.y -= lr * g.y; m.z -= lr * g.z; m.w -= lr * g.w;
    m4[i] = m;
    if (shadow) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(m.x, m.y);
      __nv_bfloat162 hi = __floats2bfloat162_rn(m.z, m.w);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(shadow)[i] = pk;
    }
  }
  for (int64_t i = n4 * 4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const float m = master[i] - lr * grad[i];
    master[i] = m;
    if (shadow) shadow[i] = __float2bfloat16_rn(m);
  }
}

template <typename D, typename S>
__global__ void cast_kernel(D* dst, const S* src, int64_t n) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = from_f<D>(to_f<S>(src[i]));
}

int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

}  // namespace
}  // namespace gpp

using namespace gpp;

extern "C" {

int gpp_version(void) { return 1; }

#ifndef GPP_SOURCE_DIGEST
#define GPP_SOURCE_DIGEST "unknown"
#endif
/* digest of the sources this binary was built from (checked by _build.py / lib.load) */
const char* gpp_source_digest(void) { return "gpp-digest:" GPP_SOURCE_DIGEST; }

int gpp_gemm_prefetch_hint(const void* ptr, int64_t bytes) {
  g_pf_ptr = ptr;
  g_pf_bytes = ptr ? bytes : 0;
  return GPP_OK;
}
const char* gpp_last_error(void) { return g_last_error.c_str(); }
uint64_t gpp_launch_count(void) { return g_launches.load(); }

static int gemm_any(int epi, const void* a, int64_t lda, int a_mn, const void* b, int64_t ldb,
                    int b_mn, const EpiParams& ep, int64_t M, int64_t N, int64_t K, int dtype,
                    void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == GPP_BF16) return tc_gemm(epi, a, lda, a_mn, b, ldb, b_mn, ep, M, N, K, s);
  if (dtype == GPP_F32) {
    const int rc = simt_gemm(epi, a, lda, a_mn, b, ldb, b_mn, ep, M, N, K, s);
    if (rc || !ep.colsum) return rc;
    GPP_ARG_CHECK(a_mn, "column sum needs the MN-major (wgrad) A operand");
    return colsum_launch<float>(ep.colsum, static_cast<const float*>(a), lda, nullptr, K, M, ep.colsum_acc, s);
  }
  set_error("unknown dtype");
  return GPP_ERR_ARG;
}

int gpp_linear_fwd(void* y, int64_t ldy, const void* x, int64_t ldx, const void* w, int64_t ldw,
                   const float* bias, const void* residual, int64_t ldres, void* pre_out,
                   int64_t ldpre, int64_t M, int64_t N, int64_t K, int act, int dtype,
                   void* stream) {
  GPP_ARG_CHECK(y && x && w, "null pointer");
  EpiParams ep{y, ldy, bias, residual, ldres, pre_out, ldpre, 1.f, 0.f, act, 0.f, nullptr, 0, 0, 0, nullptr, 0};
  return gemm_any(EPI_FWD, x, ldx, 0, w, ldw, 0, ep, M, N, K, dtype, stream);
}

int gpp_linear_dgrad(void* dx, int64_t lddx, const void* dy, int64_t lddy, const void* w,
                     int64_t ldw, const void* saved, int64_t ldsaved, int64_t M, int64_t N,
                     int64_t K, int act, int dtype, void* stream) {
  GPP_ARG_CHECK(dx && dy && w, "null pointer");
  GPP_ARG_CHECK(act == GPP_ACT_NONE || saved, "act' needs the saved tensor");
  EpiParams ep{dx, lddx, nullptr, saved, ldsaved, nullptr, 0, 1.f, 0.f, act, 0.f, nullptr, 0, 0, 0, nullptr, 0};
  // dx[M,K] = dy[M,N] . w[N,K]: GEMM (M, K, N); B(n=k_in, k=n_out) = w[n_out][k_in] is MN-major.
  return gemm_any(EPI_DGRAD, dy, lddy, 0, w, ldw, 1, ep, M, K, N, dtype, stream);
}

int gpp_linear_wgrad(float* dw, int64_t lddw, float* dbias, const void* dy, int64_t lddy,
                     const void* x, int64_t ldx, int64_t M, int64_t N, int64_t K,
                     int accumulate, int dtype, void* stream) {
  GPP_ARG_CHECK(dw && dy && x, "null pointer");
  EpiParams ep{dw, lddw, nullptr, nullptr, 0, nullptr, 0, 1.f, accumulate ? 1.f : 0.f, 0, 0.f, nullptr, 0, 0, 0, nullptr, 0};
  ep.colsum = dbias;  // dbias[n] = sum_m dy[m, n]: fused into the GEMM where possible
  ep.colsum_acc = accumulate;
  // dw[N,K] = sum_m dy[m,n] x[m,k]: GEMM (N, K, M) with both operands MN-major.
  return gemm_any(EPI_F32, dy, lddy, 1, x, ldx, 1, ep, N, K, M, dtype, stream);
}

int gpp_linear_wgrad_sgd(float* master, int64_t ldm, void* shadow, int64_t lds, float* grad,
                         int64_t ldg, float lr, int accumulate, int store_grad, const void* dy,
                         int64_t lddy, const void* x, int64_t ldx, int64_t M, int64_t N, int64_t K,
                         float* dbias, int dtype, void* stream) {
  GPP_ARG_CHECK(master && grad && dy && x, "null pointer");
  GPP_ARG_CHECK(dtype == GPP_F32 || shadow, "bf16 path needs the shadow weights");
  EpiParams ep{master, ldm, nullptr, nullptr, 0, shadow, lds, 1.f, accumulate ? 1.f : 0.f, 0,
               lr, grad, ldg, store_grad, 0, nullptr, 0};
  ep.colsum = dbias;  // the bias GRADIENT (applied later by the flat SGD), fused when possible
  ep.colsum_acc = accumulate;
  return gemm_any(EPI_SGD, dy, lddy, 1, x, ldx, 1, ep, N, K, M, dtype, stream);
}

int gpp_gemm(void* c, int64_t ldc, const void* a, int64_t lda, int a_mn, const void* b,
             int64_t ldb, int b_mn, int64_t M, int64_t N, int64_t K, float alpha, float beta,
             int out_f32, int dtype, void* stream) {
  GPP_ARG_CHECK(c && a && b, "null pointer");
  EpiParams ep{c, ldc, nullptr, nullptr, 0, nullptr, 0, alpha, beta, 0, 0.f, nullptr, 0, 0, 0, nullptr, 0};
  const int epi = (dtype == GPP_F32 || out_f32) ? EPI_F32 : EPI_BF16;
  return gemm_any(epi, a, lda, a_mn, b, ldb, b_mn, ep, M, N, K, dtype, stream);
}

int gpp_rowdot_fwd(float* out, const void* x, int64_t ldx, const float* w, const float* bias,
                   int64_t M, int64_t K, int dtype, void* stream) {
  GPP_ARG_CHECK(out && x && w && M > 0 && K > 0, "bad argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int blocks = static_cast<int>((M + 7) / 8);
  if (dtype == GPP_BF16)
    launch_pdl(rowdot_fwd_kernel<bf16>, dim3(blocks), dim3(256), 0, s, out, static_cast<const bf16*>(x), ldx, w, bias, M, K);
  else
    launch_pdl(rowdot_fwd_kernel<float>, dim3(blocks), dim3(256), 0, s, out, static_cast<const float*>(x), ldx, w, bias, M, K);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_rowdot_bwd(void* dx, int64_t lddx, float* dw, float* dbias, const float* dout,
                   const void* x, int64_t ldx, const float* w, const void* saved,
                   int64_t ldsaved, int act, int64_t M, int64_t K, int accumulate, int dtype,
                   void* stream) {
  GPP_ARG_CHECK(dout && x && w && M > 0 && K > 0, "bad argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dx) {
    const int g = grid_for(M * K, 256);
    const bool vec = dtype == GPP_BF16 && K % 8 == 0 && lddx % 8 == 0 && M * K < (1ll << 31) &&
                     reinterpret_cast<uintptr_t>(dx) % 16 == 0 &&
                     (act == GPP_ACT_NONE || (ldsaved % 8 == 0 && reinterpret_cast<uintptr_t>(saved) % 16 == 0));
    if (vec)
      launch_pdl(rowdot_dx_vec_kernel, dim3(grid_for(M * K / 8, 256)), dim3(256), 0, s, static_cast<bf16*>(dx), lddx, dout, w, static_cast<const bf16*>(saved), ldsaved, act,
          static_cast<uint32_t>(M), static_cast<uint32_t>(K / 8));
    else if (dtype == GPP_BF16)
      launch_pdl(rowdot_dx_kernel<bf16>, dim3(g), dim3(256), 0, s, static_cast<bf16*>(dx), lddx, dout, w,
                                               static_cast<const bf16*>(saved), ldsaved, act, M, K);
    else
      launch_pdl(rowdot_dx_kernel<float>, dim3(g), dim3(256), 0, s, static_cast<float*>(dx), lddx, dout, w,
                                                static_cast<const float*>(saved), ldsaved, act, M, K);
    GPP_LAUNCH_CHECK();
  }
  if (dw) {
    const int rc = dtype == GPP_BF16
        ? colsum_launch<bf16>(dw, static_cast<const bf16*>(x), ldx, dout, M, K, accumulate, s)
        : colsum_launch<float>(dw, static_cast<const float*>(x), ldx, dout, M, K, accumulate, s);
    if (rc) return rc;
  }
  if (dbias) {
    launch_pdl(sum_kernel, dim3(1), dim3(1024), 0, s, dbias, dout, M, accumulate);
    GPP_LAUNCH_CHECK();
  }
  return GPP_OK;
}

int gpp_rowdot_loss(float* z, float* dz, float* loss_acc, const void* x, int64_t ldx, const float* w,
                    const float* bias, const float* y, int64_t M, int64_t K, int kind, float scale, int dtype,
                    void* stream) {
  GPP_ARG_CHECK(z && dz && loss_acc && x && w && y && M > 0 && K > 0, "bad argument");
  GPP_ARG_CHECK(kind == 0 || kind == 1, "loss kind: 0 = MSE, 1 = BCE-with-logits");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t blocks = (M + 7) / 8;
  GPP_ARG_CHECK(blocks <= kScratchFloats, "too many rows");
  float* part = colsum_scratch();  // per-block partials + a re-arming arrival counter
  if (!part) { set_error("loss scratch allocation failed"); return GPP_ERR_CUDA; }
  unsigned* counter = reinterpret_cast<unsigned*>(part + kScratchFloats) + (kCounters - 1);
  if (dtype == GPP_BF16)
    launch_pdl(rowdot_loss_kernel<bf16>, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, s, z, dz, loss_acc, part, counter, static_cast<const bf16*>(x), ldx, w, bias, y, M, K, kind, scale);
  else
    launch_pdl(rowdot_loss_kernel<float>, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, s, z, dz, loss_acc, part, counter, static_cast<const float*>(x), ldx, w, bias, y, M, K, kind, scale);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_mse_loss(float* loss_acc, float* dpred, const float* pred, const float* y, int64_t M,
                 float scale, void* stream) {
  GPP_ARG_CHECK(loss_acc && dpred && pred && y && M > 0, "bad argument");
  launch_pdl(mse_kernel, dim3(1), dim3(1024), 0, static_cast<cudaStream_t>(stream), loss_acc, dpred, pred, y, M, scale);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_bce_loss(float* loss_acc, float* dlogit, const float* logit, const float* y, int64_t M,
                 float scale, void* stream) {
  GPP_ARG_CHECK(loss_acc && dlogit && logit && y && M > 0, "bad argument");
  launch_pdl(bce_kernel, dim3(1), dim3(1024), 0, static_cast<cudaStream_t>(stream), loss_acc, dlogit, logit, y, M, scale);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_ce_loss(float* loss_acc, void* dlogits, int64_t lddl, const void* logits, int64_t ldl,
                const int64_t* labels, int64_t M, int64_t C, float scale, int dtype,
                void* stream) {
  GPP_ARG_CHECK(loss_acc && dlogits && logits && labels && M > 0 && C > 0, "bad argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == GPP_BF16)
    launch_pdl(ce_kernel<bf16>, dim3(static_cast<unsigned>(M)), dim3(256), 0, s, loss_acc, static_cast<bf16*>(dlogits), lddl,
                                                             static_cast<const bf16*>(logits), ldl, labels, C, scale);
  else
    launch_pdl(ce_kernel<float>, dim3(static_cast<unsigned>(M)), dim3(256), 0, s, loss_acc, static_cast<float*>(dlogits), lddl,
                                                              static_cast<const float*>(logits), ldl, labels, C, scale);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_colsum(float* out, const void* x, int64_t ldx, int64_t M, int64_t N, int accumulate,
               int dtype, void* stream) {
  GPP_ARG_CHECK(out && x && M > 0 && N > 0, "bad argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return dtype == GPP_BF16
      ? colsum_launch<bf16>(out, static_cast<const bf16*>(x), ldx, nullptr, M, N, accumulate, s)
      : colsum_launch<float>(out, static_cast<const float*>(x), ldx, nullptr, M, N, accumulate, s);
}

int gpp_colsum_multi(int n, const void* const* x, const int64_t* ldx, const int64_t* M, const int64_t* N,
                     float* const* out, int accumulate, int dtype, void* stream) {
  GPP_ARG_CHECK(n >= 0 && (n == 0 || (x && ldx && M && N && out)), "bad argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return dtype == GPP_BF16 ? colsum_multi_launch<bf16>(n, x, ldx, M, N, out, accumulate, s)
                           : colsum_multi_launch<float>(n, x, ldx, M, N, out, accumulate, s);
}

int gpp_sgd_step(float* master, void* shadow_bf16, const float* grad, int64_t n, float lr,
                 void* stream) {
  GPP_ARG_CHECK(master && grad && n > 0, "bad argument");
  GPP_ARG_CHECK((reinterpret_cast<uintptr_t>(master) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(grad) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(shadow_bf16) & 7) == 0,
                "sgd buffers must be 16-byte aligned");
  launch_pdl(sgd_kernel, dim3(grid_for(n / 4 + 1, 256)), dim3(256), 0, static_cast<cudaStream_t>(stream), master, static_cast<bf16*>(shadow_bf16), grad, n, lr);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_copy_rows(void* dst, int64_t lddst, const void* src, int64_t ldsrc, int64_t rows,
                  int64_t cols, int elem_bytes, void* stream) {
  GPP_ARG_CHECK(rows >= 0 && cols >= 0, "bad argument");
  if (rows == 0 || cols == 0) return GPP_OK;  // empty tensors may carry null pointers
  GPP_ARG_CHECK(dst && src, "bad argument");
  GPP_ARG_CHECK(lddst >= cols && ldsrc >= cols && elem_bytes > 0, "bad leading dimension");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t rb = static_cast<uint64_t>(cols) * elem_bytes;
  const uint64_t db = static_cast<uint64_t>(lddst) * elem_bytes, sb = static_cast<uint64_t>(ldsrc) * elem_bytes;
  const uint64_t al = reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | rb | db | sb;
  // widest vector every row start, row length and pitch is aligned to
  const int vb = (al % 16 == 0) ? 16 : (al % 8 == 0) ? 8 : (al % 4 == 0) ? 4 : (al % 2 == 0) ? 2 : 1;
  const uint64_t cv = rb / vb, n = cv * static_cast<uint64_t>(rows);
  const int g = grid_for(static_cast<int64_t>((n + 3) / 4), 256);
  const bool i32 = n + 4ull * 256 * g < (1ull << 32);  // no wrap of base + u * stride either
#define GPP_COPY_ROWS(V)                                                                          \
  if (i32)                                                                                        \
    launch_pdl(copy_rows_kernel<V, uint32_t>, dim3(g), dim3(256), 0, s, static_cast<V*>(dst), db / vb,                \
        static_cast<const V*>(src), sb / vb, static_cast<uint32_t>(cv), static_cast<uint32_t>(n)); \
  else                                                                                            \
    launch_pdl(copy_rows_kernel<V, uint64_t>, dim3(g), dim3(256), 0, s, static_cast<V*>(dst), db / vb,                \
        static_cast<const V*>(src), sb / vb, cv, n)
  switch (vb) {
    case 16: GPP_COPY_ROWS(uint4); break;
    case 8: GPP_COPY_ROWS(uint2); break;
    case 4: GPP_COPY_ROWS(uint32_t); break;
    case 2: GPP_COPY_ROWS(uint16_t); break;
    default: GPP_COPY_ROWS(uint8_t); break;
  }
#undef GPP_COPY_ROWS
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_copy_rows_multi(int n, void* const* dst, const int64_t* lddst, const void* const* src,
                        const int64_t* ldsrc, int64_t rows, const int64_t* cols, int elem_bytes,
                        void* stream) {
  GPP_ARG_CHECK(n >= 0 && rows >= 0 && elem_bytes > 0 && (n == 0 || (dst && lddst && src && ldsrc && cols)),
                "bad argument");
  if (n == 0 || rows == 0) return GPP_OK;
  uint64_t al = 0, most = 0;
  for (int k = 0; k < n; ++k) {
    GPP_ARG_CHECK(cols[k] >= 0, "bad slice");
    if (cols[k] == 0) continue;
    GPP_ARG_CHECK(dst[k] && src[k] && lddst[k] >= cols[k] && ldsrc[k] >= cols[k],
                  "bad slice");
    al |= reinterpret_cast<uintptr_t>(dst[k]) | reinterpret_cast<uintptr_t>(src[k]) |
          static_cast<uint64_t>(cols[k]) * elem_bytes | static_cast<uint64_t>(lddst[k]) * elem_bytes |
          static_cast<uint64_t>(ldsrc[k]) * elem_bytes;
    most = std::max(most, static_cast<uint64_t>(cols[k]) * elem_bytes * rows);
  }
  // one vector width for all slices: 16 B for the bf16 concat / interaction slices, else
  // (or for > 4 GB slices) one strided copy per slice
  if (al % 16 != 0 || most / 16 + 4ull * 256 * 148 * 16 >= (1ull << 32)) {
    for (int k = 0; k < n; ++k) {
      const int rc = gpp_copy_rows(dst[k], lddst[k], src[k], ldsrc[k], rows, cols[k], elem_bytes, stream);
      if (rc != GPP_OK) return rc;
    }
    return GPP_OK;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int k0 = 0; k0 < n; k0 += kMaxCopySlices) {
    const int nk = std::min(kMaxCopySlices, n - k0);
    CopySlices d{};
    uint64_t big = 0;
    for (int k = 0; k < nk; ++k) {
      d.dst[k] = static_cast<char*>(dst[k0 + k]);
      d.src[k] = static_cast<const char*>(src[k0 + k]);
      d.ldd[k] = lddst[k0 + k] * elem_bytes / 16;
      d.lds[k] = ldsrc[k0 + k] * elem_bytes / 16;
      d.cv[k] = static_cast<uint32_t>(cols[k0 + k] * elem_bytes / 16);
      big = std::max(big, static_cast<uint64_t>(d.cv[k]) * rows);
    }
    // ~148*16 blocks over all slices
    int gx = grid_for(static_cast<int64_t>((big + 3) / 4), 256);
    gx = std::max(1, std::min(gx, (148 * 16 + nk - 1) / nk));
    launch_pdl(copy_slices_kernel<uint4>, dim3(dim3(gx, nk)), dim3(256), 0, s, d, static_cast<uint32_t>(rows));
    GPP_LAUNCH_CHECK();
  }
  return GPP_OK;
}

int gpp_cast(void* dst, int dst_dtype, const void* src, int src_dtype, int64_t n, void* stream) {
  GPP_ARG_CHECK(dst && src && n >= 0, "bad argument");
  if (n == 0) return GPP_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int g = grid_for(n, 256);
  if (dst_dtype == GPP_F32 && src_dtype == GPP_BF16)
    launch_pdl(cast_kernel<float, bf16>, dim3(g), dim3(256), 0, s, static_cast<float*>(dst), static_cast<const bf16*>(src), n);
  else if (dst_dtype == GPP_BF16 && src_dtype == GPP_F32)
    launch_pdl(cast_kernel<bf16, float>, dim3(g), dim3(256), 0, s, static_cast<bf16*>(dst), static_cast<const float*>(src), n);
  else {
    set_error("gpp_cast: unsupported dtype pair");
    return GPP_ERR_ARG;
  }
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

}  // extern "C"
