// Multi-Modal Transformer (MMT) layer operators around the tcgen05 GEMMs (
// SURVEY.md §2.3): pre-LN LayerNorm fwd/bwd, attention softmax fwd/bwd over fp32 scores,
// token mean-pool fwd/bwd, and the batched attention GEMM entry point.  Warp-per-row,
// registers only, fp32 statistics; deterministic column reductions via partial buffers.
#include <algorithm>

#define GPP_PDL_CLASS 4  // programmatic-dependent-launch family: LayerNorm / mean-pool
#include <cstdlib>

#include "gemm.cuh"

namespace gpp {
namespace {

__device__ __forceinline__ float wsum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float wmax(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---- LayerNorm: y = (x - mu) * rstd * g + b   (D <= 32 * 64, D % 64 == 0) --------------
template <int PER>  // elements per lane = D / 32
__global__ void __launch_bounds__(256) ln_fwd_kernel(bf16* __restrict__ y, float* __restrict__ mean,
                                                     float* __restrict__ rstd,
                                                     const bf16* __restrict__ x,
                                                     const float* __restrict__ g,
                                                     const float* __restrict__ b, int64_t T, int D,
                                                     float eps) {
  pdl_wait();
  pdl_trigger();
  const int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= T) return;
  const bf16* xr = x + r * D;
  float v[PER];
#pragma unroll
  for (int i = 0; i < PER / 2; ++i) {
    const float2 f = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(xr)[lane + 32 * i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) s += v[i];
  const float mu = wsum(s) / D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) q += (v[i] - mu) * (v[i] - mu);
  const float rs = rsqrtf(wsum(q) / D + eps);
  bf16* yr = y + r * D;
#pragma unroll
  for (int i = 0; i < PER / 2; ++i) {
    const int c = 2 * (lane + 32 * i);
    const float a0 = (v[2 * i] - mu) * rs * g[c] + b[c];
    const float a1 = (v[2 * i + 1] - mu) * rs * g[c + 1] + b[c + 1];
    reinterpret_cast<__nv_bfloat162*>(yr)[lane + 32 * i] = __floats2bfloat162_rn(a0, a1);
  }
  if (lane == 0) {
    mean[r] = mu;
    rstd[r] = rs;
  }
}

// dx = rstd * (dyg - mean(dyg) - xhat * mean(dyg * xhat)) [+ dres];  per-block partial
// sums of dgamma = sum dy*xhat and dbeta = sum dy into part[blockIdx.x][2*D].
template <int PER>
__global__ void __launch_bounds__(256) ln_bwd_kernel(bf16* __restrict__ dx, float* __restrict__ part,
                                                     const bf16* __restrict__ dy,
                                                     const bf16* __restrict__ x,
                                                     const float* __restrict__ mean,
                                                     const float* __restrict__ rstd,
                                                     const float* __restrict__ g,
                                                     const bf16* __restrict__ dres, int64_t T, int D,
                                                     int rows_per_block) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float red[];  // [8 warps][2 * D]
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float dg[PER], db[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) dg[i] = db[i] = 0.f;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * rows_per_block;
  for (int64_t r = r0 + w; r < r0 + rows_per_block && r < T; r += 8) {
    const float mu = mean[r], rs = rstd[r];
    float xh[PER], gy[PER];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < PER / 2; ++i) {
      const int c = 2 * (lane + 32 * i);
      const float2 xv = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(x + r * D)[lane + 32 * i]);
      const float2 dv = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(dy + r * D)[lane + 32 * i]);
      xh[2 * i] = (xv.x - mu) * rs;
      xh[2 * i + 1] = (xv.y - mu) * rs;
      gy[2 * i] = dv.x * g[c];
      gy[2 * i + 1] = dv.y * g[c + 1];
      dg[2 * i] += dv.x * xh[2 * i];
      dg[2 * i + 1] += dv.y * xh[2 * i + 1];
      db[2 * i] += dv.x;
      db[2 * i + 1] += dv.y;
      s1 += gy[2 * i] + gy[2 * i + 1];
      s2 += gy[2 * i] * xh[2 * i] + gy[2 * i + 1] * xh[2 * i + 1];
    }
    const float m1 = wsum(s1) / D, m2 = wsum(s2) / D;
#pragma unroll
    for (int i = 0; i < PER / 2; ++i) {
      float a0 = rs * (gy[2 * i] - m1 - xh[2 * i] * m2);
      float a1 = rs * (gy[2 * i + 1] - m1 - xh[2 * i + 1] * m2);
      if (dres) {
        const float2 rv = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(dres + r * D)[lane + 32 * i]);
        a0 += rv.x;
        a1 += rv.y;
      }
      reinterpret_cast<__nv_bfloat162*>(dx + r * D)[lane + 32 * i] = __floats2bfloat162_rn(a0, a1);
    }
  }
#pragma unroll
  for (int i = 0; i < PER / 2; ++i) {
    const int c = 2 * (lane + 32 * i);
    red[w * 2 * D + c] = dg[2 * i];
    red[w * 2 * D + c + 1] = dg[2 * i + 1];
    red[w * 2 * D + D + c] = db[2 * i];
    red[w * 2 * D + D + c + 1] = db[2 * i + 1];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 2 * D; c += blockDim.x) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k * 2 * D + c];
    part[static_cast<int64_t>(blockIdx.x) * 2 * D + c] = t;
  }
}

// 32 columns per block, the partial rows split over the 8 warps (coalesced 128 B loads,
// nblocks / 8 independent loads per thread), then a fixed-order smem reduction.
__global__ void __launch_bounds__(256) ln_bwd_final_kernel(float* __restrict__ dgamma, float* __restrict__ dbeta,
                                                           const float* __restrict__ part, int nblocks, int D,
                                                           int accumulate) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + tx;
  float t = 0.f;
  if (c < 2 * D) {
#pragma unroll 4
    for (int k = ty; k < nblocks; k += 8) t += part[static_cast<int64_t>(k) * 2 * D + c];
  }
  red[ty][tx] = t;
  __syncthreads();
  if (ty == 0 && c < 2 * D) {
#pragma unroll
    for (int i = 1; i < 8; ++i) t += red[i][tx];
    float* o = c < D ? dgamma + c : dbeta + (c - D);
    *o = accumulate ? *o + t : t;
  }
}

// ---- 16-byte vectorised LayerNorm forward (D % 256 == 0): lane owns 8-element chunks
// lane + 32 i, so every warp instruction moves 512 contiguous bytes of a row --------------
__device__ __forceinline__ void unpack8(const uint4& r, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const float2 x = __bfloat1622float2(h[t]);
    f[2 * t] = x.x;
    f[2 * t + 1] = x.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float* f) {
  uint4 r;
  uint32_t* u = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * t], f[2 * t + 1]);
    u[t] = *reinterpret_cast<const uint32_t*>(&h);
  }
  return r;
}
__device__ __forceinline__ void load8f(const float* p, float* f) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

template <int PER>
__global__ void __launch_bounds__(256) ln_fwd_vec_kernel(bf16* __restrict__ y, float* __restrict__ mean,
                                                         float* __restrict__ rstd, const bf16* __restrict__ x,
                                                         const float* __restrict__ g, const float* __restrict__ b,
                                                         int64_t T, int D, float eps) {
  pdl_wait();
  pdl_trigger();
  constexpr int NV = PER / 8;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= T) return;
  const uint4* xr = reinterpret_cast<const uint4*>(x + r * D);
  uint4 raw[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) raw[i] = __ldg(xr + lane + 32 * i);
  float v[PER];
#pragma unroll
  for (int i = 0; i < NV; ++i) unpack8(raw[i], v + 8 * i);
  float sm = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) sm += v[i];
  const float mu = wsum(sm) / D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) q += (v[i] - mu) * (v[i] - mu);
  const float rs = rsqrtf(wsum(q) / D + eps);
  uint4* yr = reinterpret_cast<uint4*>(y + r * D);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = 8 * (lane + 32 * i);
    float gg[8], bb[8], o[8];
    load8f(g + c, gg);
    load8f(b + c, bb);
#pragma unroll
    for (int t = 0; t < 8; ++t) o[t] = (v[8 * i + t] - mu) * rs * gg[t] + bb[t];
    yr[lane + 32 * i] = pack8(o);
  }
  if (lane == 0) {
    mean[r] = mu;
    rstd[r] = rs;
  }
}

// ---- LayerNorm, 16-byte vectors, R rows per warp (D % 256 == 0) ---------------------------
// All R rows' loads are issued before any reduction.  At T = 8192, D = 1024 with R = 4 the
// 256 blocks fit in one wave (two per SM) with the whole 16.8 MB input in flight; R = 2 left
// 512 blocks at 3 per SM = 1.15 waves (13 us cold, 1.3 TB/s).
template <int PER, int R>
__global__ void __launch_bounds__(256, R >= 4 ? 2 : 3) ln_fwd_vec2_kernel(bf16* __restrict__ y, float* __restrict__ mean,
                                                                       float* __restrict__ rstd,
                                                                       const bf16* __restrict__ x,
                                                                       const float* __restrict__ g,
                                                                       const float* __restrict__ b, int64_t T, int D,
                                                                       float eps) {
  pdl_wait();
  pdl_trigger();
  constexpr int NV = PER / 8;
  const int64_t r0 = (static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5)) * R;
  const int lane = threadIdx.x & 31;
  if (r0 >= T) return;
  uint4 raw[R][NV];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    if (r0 + k < T) {
#pragma unroll
      for (int i = 0; i < NV; ++i) raw[k][i] = __ldg(reinterpret_cast<const uint4*>(x + (r0 + k) * D) + lane + 32 * i);
    }
  }
#pragma unroll
  for (int k = 0; k < R; ++k) {
    if (r0 + k >= T) break;
    const int64_t r = r0 + k;
    float v[PER];
#pragma unroll
    for (int i = 0; i < NV; ++i) unpack8(raw[k][i], v + 8 * i);
    float sm = 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i) sm += v[i];
    const float mu = wsum(sm) / D;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i) q += (v[i] - mu) * (v[i] - mu);
    const float rs = rsqrtf(wsum(q) / D + eps);
    uint4* yr = reinterpret_cast<uint4*>(y + r * D);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = 8 * (lane + 32 * i);
      float gg[8], bb[8], o[8];
      load8f(g + c, gg);
      load8f(b + c, bb);
#pragma unroll
      for (int t = 0; t < 8; ++t) o[t] = (v[8 * i + t] - mu) * rs * gg[t] + bb[t];
      yr[lane + 32 * i] = pack8(o);
    }
    if (lane == 0) {
      mean[r] = mu;
      rstd[r] = rs;
    }
  }
}

// LayerNorm backward, 16-byte vectors (D % 256 == 0), register-lean so two 256-thread blocks
// share an SM: the row's x / dy stay packed (uint4) and x-hat, g*dy are recomputed in the
// second pass instead of being held as floats; gamma is staged in shared memory.
//   dx = rstd * (g dy - mean(g dy) - xhat * mean(g dy xhat)) [+ dres]
// per-block partials of dgamma = sum dy*xhat and dbeta = sum dy -> part[blockIdx.x][2*D].
template <int PER, int ROWS>
__global__ void __launch_bounds__(256, ROWS == 1 ? 2 : 1)
    ln_bwd_vec_kernel(bf16* __restrict__ dx, float* __restrict__ part, const bf16* __restrict__ dy,
                      const bf16* __restrict__ x, const float* __restrict__ mean, const float* __restrict__ rstd,
                      const float* __restrict__ g, const bf16* __restrict__ dres, int64_t T, int D,
                      int rows_per_block) {
  pdl_wait();
  pdl_trigger();
  constexpr int NV = PER / 8;
  extern __shared__ float sm[];  // gamma [D] | red [8 warps][2 * D]
  float* gs = sm;
  float* red = sm + D;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = threadIdx.x; c < D; c += 256) gs[c] = g[c];
  __syncthreads();
  float dg[PER], db[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) dg[i] = db[i] = 0.f;
  const int64_t rb = static_cast<int64_t>(blockIdx.x) * rows_per_block;
  const int64_t re = min(T, rb + rows_per_block);
  for (int64_t r0 = rb + ROWS * w; r0 < re; r0 += 8 * ROWS) {
    // ROWS rows per warp: every row's x / dy loads issued before the first is processed
    uint4 xr[ROWS][NV], dr[ROWS][NV];
#pragma unroll
    for (int k = 0; k < ROWS; ++k) {
      if (r0 + k >= re) break;
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        xr[k][i] = __ldg(reinterpret_cast<const uint4*>(x + (r0 + k) * D) + lane + 32 * i);
        dr[k][i] = __ldg(reinterpret_cast<const uint4*>(dy + (r0 + k) * D) + lane + 32 * i);
      }
    }
#pragma unroll
    for (int k = 0; k < ROWS; ++k) {
      const int64_t r = r0 + k;
      if (r >= re) break;
      const float mu = __ldg(mean + r), rs = __ldg(rstd + r);
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        float xv[8], dv[8];
        unpack8(xr[k][i], xv);
        unpack8(dr[k][i], dv);
        const int c = 8 * (lane + 32 * i);
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const float xh = (xv[t] - mu) * rs;
          const float gy = dv[t] * gs[c + t];
          dg[8 * i + t] = fmaf(dv[t], xh, dg[8 * i + t]);
          db[8 * i + t] += dv[t];
          s1 += gy;
          s2 = fmaf(gy, xh, s2);
        }
      }
      const float m1 = wsum(s1) / D, m2 = wsum(s2) / D;
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        float xv[8], dv[8], o[8];
        unpack8(xr[k][i], xv);
        unpack8(dr[k][i], dv);
        const int c = 8 * (lane + 32 * i);
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const float xh = (xv[t] - mu) * rs;
          o[t] = rs * (dv[t] * gs[c + t] - m1 - xh * m2);
        }
        if (dres) {
          float rv[8];
          unpack8(__ldg(reinterpret_cast<const uint4*>(dres + r * D) + lane + 32 * i), rv);
#pragma unroll
          for (int t = 0; t < 8; ++t) o[t] += rv[t];
        }
        reinterpret_cast<uint4*>(dx + r * D)[lane + 32 * i] = pack8(o);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = 8 * (lane + 32 * i);
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      red[w * 2 * D + c + t] = dg[8 * i + t];
      red[w * 2 * D + D + c + t] = db[8 * i + t];
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 2 * D; c += blockDim.x) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k * 2 * D + c];
    part[static_cast<int64_t>(blockIdx.x) * 2 * D + c] = t;
  }
}

// ---- LayerNorm, software-pipelined persistent form (D = 32 PER, PER in {16, 32}) ----------
// Warp w of the grid takes rows w, w + NW, w + 2 NW, ... (NW = every warp of the grid) and
// loads its NEXT row into a second register set before it processes the current one, so
// each warp keeps one row of loads in flight while it computes and stores -- reads and
// writes stream concurrently instead of in one load phase and one store phase per wave.
template <int PER>
struct LnFwdRow {
  uint4 x[PER / 8];
};

template <int PER>
__device__ __forceinline__ void ln_fwd_load(LnFwdRow<PER>& a, const bf16* __restrict__ x, int64_t r, int D, int lane) {
#pragma unroll
  for (int i = 0; i < PER / 8; ++i) a.x[i] = __ldg(reinterpret_cast<const uint4*>(x + r * D) + lane + 32 * i);
}

template <int PER>
__device__ __forceinline__ void ln_fwd_row(const LnFwdRow<PER>& a, bf16* __restrict__ y, float* __restrict__ mean,
                                           float* __restrict__ rstd, const float* __restrict__ gs,
                                           const float* __restrict__ bs, int64_t r, int D, float eps, int lane) {
  constexpr int NV = PER / 8;
  float v[PER];
#pragma unroll
  for (int i = 0; i < NV; ++i) unpack8(a.x[i], v + 8 * i);
  float sm = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) sm += v[i];
  const float mu = wsum(sm) / D;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) q += (v[i] - mu) * (v[i] - mu);
  const float rs = rsqrtf(wsum(q) / D + eps);
  uint4* yr = reinterpret_cast<uint4*>(y + r * D);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = 8 * (lane + 32 * i);
    const float4 g0 = *reinterpret_cast<const float4*>(gs + c), g1 = *reinterpret_cast<const float4*>(gs + c + 4);
    const float4 b0 = *reinterpret_cast<const float4*>(bs + c), b1 = *reinterpret_cast<const float4*>(bs + c + 4);
    const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    float o[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) o[t] = (v[8 * i + t] - mu) * rs * gg[t] + bb[t];
    yr[lane + 32 * i] = pack8(o);
  }
  if (lane == 0) {
    mean[r] = mu;
    rstd[r] = rs;
  }
}

template <int PER>
__global__ void __launch_bounds__(256, 2) ln_fwd_pipe_kernel(bf16* __restrict__ y, float* __restrict__ mean,
                                                             float* __restrict__ rstd, const bf16* __restrict__ x,
                                                             const float* __restrict__ g, const float* __restrict__ b,
                                                             int64_t T, int D, float eps) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float sm[];  // gamma [D] | beta [D]
  for (int c = threadIdx.x; c < D; c += 256) {
    sm[c] = g[c];
    sm[D + c] = b[c];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t NW = static_cast<int64_t>(gridDim.x) * 8;
  int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  LnFwdRow<PER> A, B;
  if (r < T) ln_fwd_load(A, x, r, D, lane);
  while (r < T) {
    if (r + NW < T) ln_fwd_load(B, x, r + NW, D, lane);
    ln_fwd_row(A, y, mean, rstd, sm, sm + D, r, D, eps, lane);
    r += NW;
    if (r >= T) break;
    if (r + NW < T) ln_fwd_load(A, x, r + NW, D, lane);
    ln_fwd_row(B, y, mean, rstd, sm, sm + D, r, D, eps, lane);
    r += NW;
  }
}

template <int PER>
struct LnBwdRow {
  uint4 x[PER / 8], dy[PER / 8];
  float mu, rs;
};

template <int PER>
__device__ __forceinline__ void ln_bwd_load(LnBwdRow<PER>& a, const bf16* __restrict__ dy, const bf16* __restrict__ x,
                                            const float* __restrict__ mean, const float* __restrict__ rstd,
                                            int64_t r, int D, int lane) {
#pragma unroll
  for (int i = 0; i < PER / 8; ++i) {
    a.x[i] = __ldg(reinterpret_cast<const uint4*>(x + r * D) + lane + 32 * i);
    a.dy[i] = __ldg(reinterpret_cast<const uint4*>(dy + r * D) + lane + 32 * i);
  }
  a.mu = __ldg(mean + r);
  a.rs = __ldg(rstd + r);
}

//   dx = rstd * (g dy - mean(g dy) - xhat * mean(g dy xhat)) [+ dres];  dg += dy xhat, db += dy
// (the residual gradient is loaded at the row's start -- its latency hides behind the first
// pass -- rather than prefetched a row ahead, which spilled the register-resident accumulators)
template <int PER>
__device__ __forceinline__ void ln_bwd_row(const LnBwdRow<PER>& a, bf16* __restrict__ dx, const float* __restrict__ gs,
                                           const bf16* __restrict__ dres, float (&dg)[PER], float (&db)[PER],
                                           int64_t r, int D, int lane) {
  constexpr int NV = PER / 8;
  const float mu = a.mu, rs = a.rs;
  uint4 dr[NV];
  if (dres) {
#pragma unroll
    for (int i = 0; i < NV; ++i) dr[i] = __ldg(reinterpret_cast<const uint4*>(dres + r * D) + lane + 32 * i);
  }
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float xv[8], dv[8];
    unpack8(a.x[i], xv);
    unpack8(a.dy[i], dv);
    const int c = 8 * (lane + 32 * i);
    const float4 g0 = *reinterpret_cast<const float4*>(gs + c), g1 = *reinterpret_cast<const float4*>(gs + c + 4);
    const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const float xh = (xv[t] - mu) * rs;
      const float gy = dv[t] * gg[t];
      dg[8 * i + t] = fmaf(dv[t], xh, dg[8 * i + t]);
      db[8 * i + t] += dv[t];
      s1 += gy;
      s2 = fmaf(gy, xh, s2);
    }
  }
  const float m1 = wsum(s1) / D, m2 = wsum(s2) / D;
  uint4* dxr = reinterpret_cast<uint4*>(dx + r * D);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float xv[8], dv[8], o[8];
    unpack8(a.x[i], xv);
    unpack8(a.dy[i], dv);
    const int c = 8 * (lane + 32 * i);
    const float4 g0 = *reinterpret_cast<const float4*>(gs + c), g1 = *reinterpret_cast<const float4*>(gs + c + 4);
    const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const float xh = (xv[t] - mu) * rs;
      o[t] = rs * (dv[t] * gg[t] - m1 - xh * m2);
    }
    if (dres) {
      float rv[8];
      unpack8(dr[i], rv);
#pragma unroll
      for (int t = 0; t < 8; ++t) o[t] += rv[t];
    }
    dxr[lane + 32 * i] = pack8(o);
  }
}

// per-block partials of dgamma / dbeta -> part[blockIdx.x][2 D] (ln_bwd_final16_kernel sums them)
template <int PER>
__global__ void __launch_bounds__(256, PER == 32 ? 1 : 2)
    ln_bwd_pipe_kernel(bf16* __restrict__ dx, float* __restrict__ part, const bf16* __restrict__ dy,
                       const bf16* __restrict__ x, const float* __restrict__ mean, const float* __restrict__ rstd,
                       const float* __restrict__ g, const bf16* __restrict__ dres, int64_t T, int D) {
  pdl_wait();
  pdl_trigger();
  constexpr int NV = PER / 8;
  extern __shared__ float sm[];  // gamma [D] | red [8 warps][2 * D]
  float* gs = sm;
  float* red = sm + D;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = threadIdx.x; c < D; c += 256) gs[c] = g[c];
  __syncthreads();
  float dg[PER], db[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) dg[i] = db[i] = 0.f;
  const int64_t NW = static_cast<int64_t>(gridDim.x) * 8;
  int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + w;
  LnBwdRow<PER> A, B;
  if (r < T) ln_bwd_load(A, dy, x, mean, rstd, r, D, lane);
  while (r < T) {
    if (r + NW < T) ln_bwd_load(B, dy, x, mean, rstd, r + NW, D, lane);
    ln_bwd_row(A, dx, gs, dres, dg, db, r, D, lane);
    r += NW;
    if (r >= T) break;
    if (r + NW < T) ln_bwd_load(A, dy, x, mean, rstd, r + NW, D, lane);
    ln_bwd_row(B, dx, gs, dres, dg, db, r, D, lane);
    r += NW;
  }
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = 8 * (lane + 32 * i);
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      red[w * 2 * D + c + t] = dg[8 * i + t];
      red[w * 2 * D + D + c + t] = db[8 * i + t];
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 2 * D; c += blockDim.x) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k * 2 * D + c];
    part[static_cast<int64_t>(blockIdx.x) * 2 * D + c] = t;
  }
}

// Column sums of the [nblocks, 2D] partials, 16 columns per block x 16 row groups (every
// thread's loads independent and in flight together), fixed-order smem reduction.
__global__ void __launch_bounds__(256) ln_bwd_final16_kernel(float* __restrict__ dgamma, float* __restrict__ dbeta,
                                                             const float* __restrict__ part, int nblocks, int D,
                                                             int accumulate) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[16][17];
  const int cx = threadIdx.x & 15, ry = threadIdx.x >> 4;
  const int c = blockIdx.x * 16 + cx;
  float t = 0.f;
  if (c < 2 * D) {
#pragma unroll 8
    for (int k = ry; k < nblocks; k += 16) t += __ldg(part + static_cast<int64_t>(k) * 2 * D + c);
  }
  red[ry][cx] = t;
  __syncthreads();
  if (ry == 0 && c < 2 * D) {
#pragma unroll
    for (int i = 1; i < 16; ++i) t += red[i][cx];
    float* o = c < D ? dgamma + c : dbeta + (c - D);
    *o = accumulate ? *o + t : t;
  }
}

// ---- attention softmax: P = softmax(s) row-wise (fp32 scores, already scaled) ------------
template <int PER>
__global__ void __launch_bounds__(256) softmax_fwd_kernel(bf16* __restrict__ p,
                                                          const float* __restrict__ s, int64_t R,
                                                          int L) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= R) return;
  float v[PER];
  const float4* sr = reinterpret_cast<const float4*>(s + r * L);
#pragma unroll
  for (int i = 0; i < PER / 4; ++i) {
    const float4 f = sr[lane + 32 * i];
    v[4 * i] = f.x; v[4 * i + 1] = f.y; v[4 * i + 2] = f.z; v[4 * i + 3] = f.w;
  }
  float mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < PER; ++i) mx = fmaxf(mx, v[i]);
  mx = wmax(mx);
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    v[i] = __expf(v[i] - mx);
    sum += v[i];
  }
  const float inv = 1.f / wsum(sum);
  __nv_bfloat162* pr = reinterpret_cast<__nv_bfloat162*>(p + r * L);
#pragma unroll
  for (int i = 0; i < PER / 4; ++i) {
    pr[2 * (lane + 32 * i)] = __floats2bfloat162_rn(v[4 * i] * inv, v[4 * i + 1] * inv);
    pr[2 * (lane + 32 * i) + 1] = __floats2bfloat162_rn(v[4 * i + 2] * inv, v[4 * i + 3] * inv);
  }
}

// dS = scale * P * (dP - sum(dP * P))   (bf16 out; P bf16, dP fp32)
template <int PER>
__global__ void __launch_bounds__(256) softmax_bwd_kernel(bf16* __restrict__ ds,
                                                          const bf16* __restrict__ p,
                                                          const float* __restrict__ dp, int64_t R,
                                                          int L, float scale) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= R) return;
  float pv[PER], gv[PER];
  const float4* dr = reinterpret_cast<const float4*>(dp + r * L);
  const __nv_bfloat162* prr = reinterpret_cast<const __nv_bfloat162*>(p + r * L);
  float dot = 0.f;
#pragma unroll
  for (int i = 0; i < PER / 4; ++i) {
    const float4 f = dr[lane + 32 * i];
    const float2 a = __bfloat1622float2(prr[2 * (lane + 32 * i)]);
    const float2 b = __bfloat1622float2(prr[2 * (lane + 32 * i) + 1]);
    gv[4 * i] = f.x; gv[4 * i + 1] = f.y; gv[4 * i + 2] = f.z; gv[4 * i + 3] = f.w;
    pv[4 * i] = a.x; pv[4 * i + 1] = a.y; pv[4 * i + 2] = b.x; pv[4 * i + 3] = b.y;
#pragma unroll
    for (int j = 0; j < 4; ++j) dot += gv[4 * i + j] * pv[4 * i + j];
  }
  dot = wsum(dot);
  __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(ds + r * L);
#pragma unroll
  for (int i = 0; i < PER / 4; ++i) {
    float t[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) t[j] = scale * pv[4 * i + j] * (gv[4 * i + j] - dot);
    o[2 * (lane + 32 * i)] = __floats2bfloat162_rn(t[0], t[1]);
    o[2 * (lane + 32 * i) + 1] = __floats2bfloat162_rn(t[2], t[3]);
  }
}

// ---- token mean-pool over S rows per sample (branch output of MMT) ------------------------
// out[m, c] = mean over the S rows of sample m.  Vector form (D % 64 == 0, 16-byte rows):
// one block per (sample, 64 columns); 8 threads x 8 columns cover the 64 columns, 32 row
// slices split the S rows (every thread's 16-byte loads independent), fixed-order smem
// reduction over the slices.  The scalar form (one thread per column, S dependent loads)
// kept 6% of the warps busy: 35 us for 16.8 MB.
__global__ void __launch_bounds__(256) meanpool_fwd_vec_kernel(bf16* __restrict__ out, int64_t ldo,
                                                               const bf16* __restrict__ x, int64_t M, int S, int D) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[32][65];
  const int m = blockIdx.y, cg = threadIdx.x & 7, sl = threadIdx.x >> 3;
  const int c0 = blockIdx.x * 64 + cg * 8;
  const bf16* xm = x + static_cast<int64_t>(m) * S * D + c0;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
  for (int t = sl; t < S; t += 32) {
    float v[8];
    unpack8(__ldg(reinterpret_cast<const uint4*>(xm + static_cast<int64_t>(t) * D)), v);
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] += v[i];
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) red[sl][cg * 8 + i] = acc[i];
  __syncthreads();
  if (threadIdx.x < 64) {
    float t = 0.f;
#pragma unroll 8
    for (int k = 0; k < 32; ++k) t += red[k][threadIdx.x];
    out[static_cast<int64_t>(m) * ldo + blockIdx.x * 64 + threadIdx.x] = __float2bfloat16_rn(t / S);
  }
}

__global__ void meanpool_fwd_kernel(bf16* __restrict__ out, int64_t ldo, const bf16* __restrict__ x,
                                    int64_t M, int S, int D) {
  pdl_wait();
  pdl_trigger();
  const int64_t m = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M || c >= D) return;
  const bf16* xm = x + m * S * D + c;
  float s = 0.f;
  for (int t = 0; t < S; ++t) s += __bfloat162float(xm[static_cast<int64_t>(t) * D]);
  out[m * ldo + c] = __float2bfloat16_rn(s / S);
}

// dx[m, t, :] = dout[m, :] / S; vector form: 8 columns (one 16-byte store) per thread.
__global__ void __launch_bounds__(256) meanpool_bwd_vec_kernel(bf16* __restrict__ dx, const bf16* __restrict__ dout,
                                                               int64_t lddo, int64_t M, int S, int D) {
  pdl_wait();
  pdl_trigger();
  const int64_t n8 = M * S * D / 8;
  const float inv = 1.f / S;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t e = i * 8;
    const int64_t m = e / (static_cast<int64_t>(S) * D);
    const int c = static_cast<int>(e % D);
    float v[8];
    unpack8(__ldg(reinterpret_cast<const uint4*>(dout + m * lddo + c)), v);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] *= inv;
    reinterpret_cast<uint4*>(dx)[i] = pack8(v);
  }
}

__global__ void meanpool_bwd_kernel(bf16* __restrict__ dx, const bf16* __restrict__ dout,
                                    int64_t lddo, int64_t M, int S, int D) {
  pdl_wait();
  pdl_trigger();
  const int64_t n = M * S * D;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t m = i / (static_cast<int64_t>(S) * D);
    const int c = static_cast<int>(i % D);
    dx[i] = __float2bfloat16_rn(__bfloat162float(dout[m * lddo + c]) / S);
  }
}

// Per-device scratch for the LayerNorm-backward dgamma/dbeta partials.  Grows only outside
// CUDA-graph capture and never frees: a graph captured earlier may still reference the old
// buffer, so a grown-out buffer is retired (kept allocated) instead of released.
float* ln_scratch(size_t floats, cudaStream_t stream) {
  static float* bufs[64] = {nullptr};
  static size_t caps[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (caps[dev] >= floats) return bufs[dev];
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &st);
  if (st != cudaStreamCaptureStatusNone) {
    set_error("LayerNorm scratch must be sized before CUDA-graph capture (run one eager step first)");
    return nullptr;
  }
  size_t want = floats < (size_t(4) << 20) ? (size_t(4) << 20) : floats;
  float* p = nullptr;
  if (cudaMalloc(&p, want * sizeof(float)) != cudaSuccess) {
    set_error("LayerNorm scratch allocation failed");
    return nullptr;
  }
  bufs[dev] = p;
  caps[dev] = want;
  return p;
}

}  // namespace
}  // namespace gpp

using namespace gpp;


static bool a16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

static int sm_count() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return n;
}
// GPP_LN_PIPE=0: the one-wave LayerNorm kernels (ln_fwd_vec2 / ln_bwd_vec) instead of the
// software-pipelined persistent ones, for A/B measurement
static bool ln_pipe() {
  static const bool on = [] { const char* e = std::getenv("GPP_LN_PIPE"); return !(e && e[0] == '0'); }();
  return on;
}

extern "C" {

int gpp_layernorm_fwd(void* y, float* mean, float* rstd, const void* x, const float* gamma,
                      const float* beta, int64_t T, int64_t D, float eps, void* stream) {
  GPP_ARG_CHECK(y && mean && rstd && x && gamma && beta && T > 0, "bad argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const unsigned grid = static_cast<unsigned>((T + 7) / 8);
  const int d = static_cast<int>(D);
  GPP_ARG_CHECK(D == 128 || (a16(y) && a16(x) && a16(gamma) && a16(beta)), "16-byte aligned rows / affine params");
  if ((D == 512 || D == 1024) && ln_pipe()) {
    const unsigned pg = static_cast<unsigned>(std::min<int64_t>((T + 7) / 8, 2 * sm_count()));
    const size_t smem = 2 * D * sizeof(float);
    if (D == 1024)
      launch_pdl(ln_fwd_pipe_kernel<32>, dim3(pg), dim3(256), smem, s, static_cast<bf16*>(y), mean, rstd,
                 static_cast<const bf16*>(x), gamma, beta, T, d, eps);
    else
      launch_pdl(ln_fwd_pipe_kernel<16>, dim3(pg), dim3(256), smem, s, static_cast<bf16*>(y), mean, rstd,
                 static_cast<const bf16*>(x), gamma, beta, T, d, eps);
    GPP_LAUNCH_CHECK();
    return GPP_OK;
  }
  switch (D) {
    case 128: launch_pdl(ln_fwd_kernel<4>, dim3(grid), dim3(256), 0, s, static_cast<bf16*>(y), mean, rstd, static_cast<const bf16*>(x), gamma, beta, T, d, eps); break;
    case 256: launch_pdl(ln_fwd_vec_kernel<8>, dim3(grid), dim3(256), 0, s, static_cast<bf16*>(y), mean, rstd, static_cast<const bf16*>(x), gamma, beta, T, d, eps); break;
    case 512:
      launch_pdl(ln_fwd_vec2_kernel<16, 4>, dim3(static_cast<unsigned>((T + 31) / 32)), dim3(256), 0, s, static_cast<bf16*>(y), mean, rstd,
                                                                                     static_cast<const bf16*>(x), gamma, beta, T, d, eps);
      break;
    case 1024:
      launch_pdl(ln_fwd_vec2_kernel<32, 4>, dim3(static_cast<unsigned>((T + 31) / 32)), dim3(256), 0, s, static_cast<bf16*>(y), mean, rstd,
                                                                                     static_cast<const bf16*>(x), gamma, beta, T, d, eps);
      break;
    default: set_error("layernorm: D must be 128/256/512/1024"); return GPP_ERR_UNSUPPORTED;
  }
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_layernorm_bwd(void* dx, float* dgamma, float* dbeta, const void* dy, const void* x,
                      const float* mean, const float* rstd, const float* gamma, const void* dres,
                      int64_t T, int64_t D, int accumulate, void* stream) {
  GPP_ARG_CHECK(dx && dgamma && dbeta && dy && x && mean && rstd && gamma && T > 0, "bad argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int d = static_cast<int>(D);
  auto* dxp = static_cast<bf16*>(dx);
  auto* dyp = static_cast<const bf16*>(dy);
  auto* xp = static_cast<const bf16*>(x);
  auto* drp = static_cast<const bf16*>(dres);
  if ((D == 512 || D == 1024) && a16(dx) && a16(dy) && a16(x) && (!dres || a16(dres)) && ln_pipe()) {
    // persistent, one (D = 1024) or two (D = 512) blocks per SM, rows strided over all warps
    const int nblk = static_cast<int>(std::min<int64_t>((T + 7) / 8, sm_count() * (D == 1024 ? 1 : 2)));
    float* part = ln_scratch(static_cast<size_t>(nblk) * 2 * D, s);
    if (!part) return GPP_ERR_CUDA;
    const size_t smem = (D + 8 * 2 * D) * sizeof(float);
    if (D == 1024) {
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(ln_bwd_pipe_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        attr = true;
      }
      launch_pdl(ln_bwd_pipe_kernel<32>, dim3(nblk), dim3(256), smem, s, dxp, part, dyp, xp, mean, rstd, gamma, drp, T, d);
    } else {
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(ln_bwd_pipe_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        attr = true;
      }
      launch_pdl(ln_bwd_pipe_kernel<16>, dim3(nblk), dim3(256), smem, s, dxp, part, dyp, xp, mean, rstd, gamma, drp, T, d);
    }
    GPP_LAUNCH_CHECK();
    launch_pdl(ln_bwd_final16_kernel, dim3(static_cast<unsigned>((2 * D + 15) / 16)), dim3(256), 0, s, dgamma, dbeta,
               part, nblk, d, accumulate);
    GPP_LAUNCH_CHECK();
    return GPP_OK;
  }
  if ((D == 512 || D == 1024) && a16(dx) && a16(dy) && a16(x) && (!dres || a16(dres))) {
    // D = 1024: one block per SM, two rows per warp in flight; D = 512: two blocks per SM,
    // one row per warp.  Rows per block rounded up to the rows one pass of 8 warps covers.
    const int per_sm = D == 1024 ? 1 : 2, rows = D == 1024 ? 16 : 8;
    const int64_t nb0 = 148 * per_sm;
    // rows per block: ceil(T / (blocks per SM x SMs)) rounded to the 8 warps (T = 8192: 56 rows,
    // 147 blocks; rounding to a whole 16-row pass left 20 SMs idle)
    const int rpb = static_cast<int>(std::max<int64_t>(rows, ((T + nb0 - 1) / nb0 + 7) / 8 * 8));
    const int nblk = static_cast<int>((T + rpb - 1) / rpb);
    float* part = ln_scratch(static_cast<size_t>(nblk) * 2 * D, s);
    if (!part) return GPP_ERR_CUDA;
    const size_t smem = (D + 8 * 2 * D) * sizeof(float);
    if (D == 1024) {
      cudaFuncSetAttribute(ln_bwd_vec_kernel<32, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      launch_pdl(ln_bwd_vec_kernel<32, 2>, dim3(nblk), dim3(256), smem, s, dxp, part, dyp, xp, mean, rstd, gamma, drp, T, d, rpb);
    } else {
      cudaFuncSetAttribute(ln_bwd_vec_kernel<16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      launch_pdl(ln_bwd_vec_kernel<16, 1>, dim3(nblk), dim3(256), smem, s, dxp, part, dyp, xp, mean, rstd, gamma, drp, T, d, rpb);
    }
    GPP_LAUNCH_CHECK();
    launch_pdl(ln_bwd_final16_kernel, dim3(static_cast<unsigned>((2 * D + 15) / 16)), dim3(256), 0, s, dgamma, dbeta, part, nblk, d,
                                                                                 accumulate);
    GPP_LAUNCH_CHECK();
    return GPP_OK;
  }
  // one block per SM: rows per block = ceil(T / 148) rounded up to the 8 warps (T = 8192:
  // 56 rows, 147 blocks; 64 rows left 20 SMs idle)
  const int rpb = static_cast<int>(std::max<int64_t>(8, ((T + 147) / 148 + 7) / 8 * 8));
  const int nblk = static_cast<int>((T + rpb - 1) / rpb);
  float* part = ln_scratch(static_cast<size_t>(nblk) * 2 * D, s);
  if (!part) return GPP_ERR_CUDA;
  const size_t smem = 8 * 2 * D * sizeof(float);
  switch (D) {
    case 128: launch_pdl(ln_bwd_kernel<4>, dim3(nblk), dim3(256), smem, s, dxp, part, dyp, xp, mean, rstd, gamma, drp, T, d, rpb); break;
    case 256: launch_pdl(ln_bwd_kernel<8>, dim3(nblk), dim3(256), smem, s, dxp, part, dyp, xp, mean, rstd, gamma, drp, T, d, rpb); break;
    case 512: launch_pdl(ln_bwd_kernel<16>, dim3(nblk), dim3(256), smem, s, dxp, part, dyp, xp, mean, rstd, gamma, drp, T, d, rpb); break;
    case 1024:
      cudaFuncSetAttribute(ln_bwd_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      launch_pdl(ln_bwd_kernel<32>, dim3(nblk), dim3(256), smem, s, dxp, part, dyp, xp, mean, rstd, gamma, drp, T, d, rpb); break;
    default: set_error("layernorm: D must be 128/256/512/1024"); return GPP_ERR_UNSUPPORTED;
  }
  GPP_LAUNCH_CHECK();
  launch_pdl(ln_bwd_final_kernel, dim3(static_cast<unsigned>((2 * D + 31) / 32)), dim3(256), 0, s, dgamma, dbeta, part, nblk, d, accumulate);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_softmax_fwd(void* p, const float* scores, int64_t R, int64_t L, void* stream) {
  GPP_ARG_CHECK(p && scores && R > 0, "bad argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const unsigned grid = static_cast<unsigned>((R + 7) / 8);
  switch (L) {
    case 128: softmax_fwd_kernel<4><<<grid, 256, 0, s>>>(static_cast<bf16*>(p), scores, R, 128); break;
    case 256: softmax_fwd_kernel<8><<<grid, 256, 0, s>>>(static_cast<bf16*>(p), scores, R, 256); break;
    case 512: softmax_fwd_kernel<16><<<grid, 256, 0, s>>>(static_cast<bf16*>(p), scores, R, 512); break;
    case 1024: softmax_fwd_kernel<32><<<grid, 256, 0, s>>>(static_cast<bf16*>(p), scores, R, 1024); break;
    default: set_error("softmax: L must be 128/256/512/1024"); return GPP_ERR_UNSUPPORTED;
  }
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_softmax_bwd(void* ds, const void* p, const float* dp, int64_t R, int64_t L, float scale,
                    void* stream) {
  GPP_ARG_CHECK(ds && p && dp && R > 0, "bad argument");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const unsigned grid = static_cast<unsigned>((R + 7) / 8);
  auto* o = static_cast<bf16*>(ds);
  auto* pp = static_cast<const bf16*>(p);
  switch (L) {
    case 128: softmax_bwd_kernel<4><<<grid, 256, 0, s>>>(o, pp, dp, R, 128, scale); break;
    case 256: softmax_bwd_kernel<8><<<grid, 256, 0, s>>>(o, pp, dp, R, 256, scale); break;
    case 512: softmax_bwd_kernel<16><<<grid, 256, 0, s>>>(o, pp, dp, R, 512, scale); break;
    case 1024: softmax_bwd_kernel<32><<<grid, 256, 0, s>>>(o, pp, dp, R, 1024, scale); break;
    default: set_error("softmax: L must be 128/256/512/1024"); return GPP_ERR_UNSUPPORTED;
  }
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_meanpool_fwd(void* out, int64_t ldo, const void* x, int64_t M, int64_t S, int64_t D,
                     void* stream) {
  GPP_ARG_CHECK(out && x && M > 0 && S > 0 && D > 0, "bad argument");
  if (D % 64 == 0 && a16(x)) {
    launch_pdl(meanpool_fwd_vec_kernel, dim3(static_cast<unsigned>(D / 64), static_cast<unsigned>(M)), dim3(256), 0,
               static_cast<cudaStream_t>(stream), static_cast<bf16*>(out), ldo, static_cast<const bf16*>(x), M,
               static_cast<int>(S), static_cast<int>(D));
    GPP_LAUNCH_CHECK();
    return GPP_OK;
  }
  dim3 grid(static_cast<unsigned>((D + 127) / 128), static_cast<unsigned>(M));
  launch_pdl(meanpool_fwd_kernel, dim3(grid), dim3(128), 0, static_cast<cudaStream_t>(stream), static_cast<bf16*>(out), ldo, static_cast<const bf16*>(x), M, static_cast<int>(S), static_cast<int>(D));
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_meanpool_bwd(void* dx, const void* dout, int64_t lddo, int64_t M, int64_t S, int64_t D,
                     void* stream) {
  GPP_ARG_CHECK(dx && dout && M > 0, "bad argument");
  int64_t n = M * S * D;
  if (D % 8 == 0 && lddo % 8 == 0 && a16(dx) && a16(dout)) {
    const int64_t g8 = std::min<int64_t>((n / 8 + 255) / 256, 148 * 8);
    launch_pdl(meanpool_bwd_vec_kernel, dim3(static_cast<unsigned>(g8)), dim3(256), 0, static_cast<cudaStream_t>(stream),
               static_cast<bf16*>(dx), static_cast<const bf16*>(dout), lddo, M, static_cast<int>(S), static_cast<int>(D));
    GPP_LAUNCH_CHECK();
    return GPP_OK;
  }
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  launch_pdl(meanpool_bwd_kernel, dim3(static_cast<unsigned>(g)), dim3(256), 0, static_cast<cudaStream_t>(stream), static_cast<bf16*>(dx), static_cast<const bf16*>(dout), lddo, M, static_cast<int>(S), static_cast<int>(D));
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

// Batched GEMM (attention): spec = {nbatch, nlo, a_m0, a_m_hi, a_m_lo, a_k0, a_k_hi, a_k_lo,
// b_n0, b_n_hi, b_n_lo, b_k0, b_k_hi, b_k_lo, c0, c_hi, c_lo} (17 ints); a_rows / b_rows =
// full operand row counts.
int gpp_gemm_batched(void* c, int64_t ldc, const void* a, int64_t lda, int64_t a_rows, int a_mn,
                     const void* b, int64_t ldb, int64_t b_rows, int b_mn, int64_t M, int64_t N,
                     int64_t K, float alpha, float beta, int out_f32, const int64_t* spec,
                     void* stream) {
  GPP_ARG_CHECK(c && a && b && spec, "null pointer");
  BatchSpec bs;
  bs.nbatch = static_cast<int>(spec[0]);
  bs.nlo = static_cast<int>(spec[1]);
  bs.a_m0 = static_cast<int>(spec[2]); bs.a_m_hi = static_cast<int>(spec[3]); bs.a_m_lo = static_cast<int>(spec[4]);
  bs.a_k0 = static_cast<int>(spec[5]); bs.a_k_hi = static_cast<int>(spec[6]); bs.a_k_lo = static_cast<int>(spec[7]);
  bs.b_n0 = static_cast<int>(spec[8]); bs.b_n_hi = static_cast<int>(spec[9]); bs.b_n_lo = static_cast<int>(spec[10]);
  bs.b_k0 = static_cast<int>(spec[11]); bs.b_k_hi = static_cast<int>(spec[12]); bs.b_k_lo = static_cast<int>(spec[13]);
  bs.c0 = spec[14]; bs.c_hi = spec[15]; bs.c_lo = spec[16];
  EpiParams ep{c, ldc, nullptr, nullptr, 0, nullptr, 0, alpha, beta, 0, 0.f, nullptr, 0, 0, 0, nullptr, 0};
  return tc_gemm_batched(out_f32 ? EPI_F32 : EPI_BF16, a, lda, a_rows, a_mn, b, ldb, b_rows, b_mn, ep,
                         bs, M, N, K, static_cast<cudaStream_t>(stream));
}

static BatchSpec batch_spec(const int64_t* spec) {
  BatchSpec bs;
  bs.nbatch = static_cast<int>(spec[0]);
  bs.nlo = static_cast<int>(spec[1]);
  bs.a_m0 = static_cast<int>(spec[2]); bs.a_m_hi = static_cast<int>(spec[3]); bs.a_m_lo = static_cast<int>(spec[4]);
  bs.a_k0 = static_cast<int>(spec[5]); bs.a_k_hi = static_cast<int>(spec[6]); bs.a_k_lo = static_cast<int>(spec[7]);
  bs.b_n0 = static_cast<int>(spec[8]); bs.b_n_hi = static_cast<int>(spec[9]); bs.b_n_lo = static_cast<int>(spec[10]);
  bs.b_k0 = static_cast<int>(spec[11]); bs.b_k_hi = static_cast<int>(spec[12]); bs.b_k_lo = static_cast<int>(spec[13]);
  bs.c0 = spec[14]; bs.c_hi = spec[15]; bs.c_lo = spec[16];
  return bs;
}

int gpp_attn_softmax(void* p, int64_t ldp, const void* q, int64_t ldq, int64_t q_rows, const void* k,
                     int64_t ldk, int64_t k_rows, int64_t M, int64_t N, int64_t K, float scale,
                     const int64_t* spec, void* stream) {
  GPP_ARG_CHECK(p && q && k && spec, "null pointer");
  return tc_attn_softmax(0, p, ldp, nullptr, 0, q, ldq, q_rows, k, ldk, k_rows, batch_spec(spec), M, N, K, scale,
                         static_cast<cudaStream_t>(stream));
}

int gpp_attn_softmax_bwd(void* ds, int64_t ldc, const void* p, int64_t ldp, const void* dout, int64_t ldo,
                         int64_t o_rows, const void* v, int64_t ldv, int64_t v_rows, int64_t M, int64_t N,
                         int64_t K, float scale, const int64_t* spec, void* stream) {
  GPP_ARG_CHECK(ds && p && dout && v && spec, "null pointer");
  return tc_attn_softmax(1, ds, ldc, p, ldp, dout, ldo, o_rows, v, ldv, v_rows, batch_spec(spec), M, N, K, scale,
                         static_cast<cudaStream_t>(stream));
}

}  // extern "C"
