// DLRM operators (Appendix B): embedding-bag
// gather-sum, its sparse SGD scatter, and the pairwise dot interaction.
// All HBM / latency bound: warp-per-bag with 8-byte vector row loads, ILP over the
// bag, warp-per-sample interaction staged through padded shared memory.
#include <cstdlib>

#include "common.cuh"

namespace gpp {
namespace {

// Count of out-of-range embedding indices seen by the gather / scatter kernels since the
// last gpp_embbag_bad_indices() read.  Such a bag element contributes nothing and updates
// nothing (PyTorch's embedding_bag raises on them; the host API raises on a nonzero count).
__device__ unsigned long long g_bad_indices = 0;

// pooled[m, :D] = sum_b table[idx[m, b], :D]   (fp32 table, bf16 pooled, D = 64)
__global__ void __launch_bounds__(256) embbag_fwd_kernel(bf16* __restrict__ out, int64_t ldo,
                                                         const float* __restrict__ table,
                                                         const int64_t* __restrict__ idx,
                                                         int64_t ldi, int64_t M, int bag,
                                                         int64_t rows) {
  const int64_t m = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (m >= M) return;
  const int64_t* ix = idx + m * ldi;
  float2 acc = make_float2(0.f, 0.f);
  for (int b0 = 0; b0 < bag; b0 += 32) {
    const int nb = bag - b0 < 32 ? bag - b0 : 32;
    int64_t my = lane < nb ? __ldg(ix + b0 + lane) : 0;
    const bool bad = my < 0 || my >= rows;
    if (bad) atomicAdd(&g_bad_indices, 1ull);
    my = bad ? -1 : my;  // -1: contributes zero, never read out of the table
    int b = 0;
    for (; b + 4 <= nb; b += 4) {
      const int64_t r0 = __shfl_sync(0xffffffffu, my, b);
      const int64_t r1 = __shfl_sync(0xffffffffu, my, b + 1);
      const int64_t r2 = __shfl_sync(0xffffffffu, my, b + 2);
      const int64_t r3 = __shfl_sync(0xffffffffu, my, b + 3);
      const float2 z = make_float2(0.f, 0.f);
      const float2 v0 = r0 >= 0 ? __ldg(reinterpret_cast<const float2*>(table + r0 * 64) + lane) : z;
      const float2 v1 = r1 >= 0 ? __ldg(reinterpret_cast<const float2*>(table + r1 * 64) + lane) : z;
      const float2 v2 = r2 >= 0 ? __ldg(reinterpret_cast<const float2*>(table + r2 * 64) + lane) : z;
      const float2 v3 = r3 >= 0 ? __ldg(reinterpret_cast<const float2*>(table + r3 * 64) + lane) : z;
      acc.x += (v0.x + v1.x) + (v2.x + v3.x);
      acc.y += (v0.y + v1.y) + (v2.y + v3.y);
    }
    for (; b < nb; ++b) {
      const int64_t r = __shfl_sync(0xffffffffu, my, b);
      if (r < 0) continue;
      const float2 v = __ldg(reinterpret_cast<const float2*>(table + r * 64) + lane);
      acc.x += v.x;
      acc.y += v.y;
    }
  }
  reinterpret_cast<__nv_bfloat162*>(out + m * ldo)[lane] = __floats2bfloat162_rn(acc.x, acc.y);
}

// table[idx[m, b], :] -= lr * dpooled[m, :]   for every (m, b): synchronous sparse SGD
__global__ void __launch_bounds__(256) embbag_sgd_kernel(float* __restrict__ table,
                                                         const bf16* __restrict__ dpool,
                                                         int64_t ldd, const int64_t* __restrict__ idx,
                                                         int64_t ldi, int64_t M, int bag, float lr,
                                                         int64_t rows) {
  const int64_t m = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (m >= M) return;
  const float2 g = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(dpool + m * ldd)[lane]);
  const float2 u = make_float2(-lr * g.x, -lr * g.y);
  const int64_t* ix = idx + m * ldi;
  for (int b0 = 0; b0 < bag; b0 += 32) {
    const int nb = bag - b0 < 32 ? bag - b0 : 32;
    int64_t my = lane < nb ? __ldg(ix + b0 + lane) : 0;
    if (my < 0 || my >= rows) {  // skipped (never redirected to row 0), counted for the host
      atomicAdd(&g_bad_indices, 1ull);
      my = -1;
    }
    for (int b = 0; b < nb; ++b) {
      const int64_t r = __shfl_sync(0xffffffffu, my, b);
      if (r < 0) continue;
      float* p = table + r * 64 + 2 * lane;
      atomicAdd(reinterpret_cast<float2*>(p), u);
    }
  }
}

// Interaction: z [M, F*D] (F feature vectors of D=64, feature 0 = bottom-MLP output).
// out[m, 0:D] = z[m, 0, :];  out[m, D + p(i,j)] = <z_i, z_j> for i > j (p in row-major
// lower-triangle order: (1,0),(2,0),(2,1),...);  out[m, D+P : ldo_valid] = 0 (padding).
constexpr int ZLD = 65;  // padded smem row (floats): conflict-free column reads

__global__ void __launch_bounds__(128) interaction_fwd_kernel(bf16* __restrict__ out, int64_t ldo,
                                                              int64_t out_cols,
                                                              const bf16* __restrict__ z,
                                                              int64_t ldz, int64_t M, int F) {
  extern __shared__ float zs[];  // 4 warps x F x ZLD
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m = static_cast<int64_t>(blockIdx.x) * 4 + w;
  if (m >= M) return;
  float* my = zs + w * F * ZLD;
  const bf16* zr = z + m * ldz;
  for (int i = 0; i < F; ++i) {
    const float2 v = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(zr + i * 64)[lane]);
    my[i * ZLD + 2 * lane] = v.x;
    my[i * ZLD + 2 * lane + 1] = v.y;
  }
  __syncwarp();
  bf16* o = out + m * ldo;
  o[2 * lane] = zr[2 * lane];
  o[2 * lane + 1] = zr[2 * lane + 1];
  const int P = F * (F - 1) / 2;
  for (int p = lane; p < P; p += 32) {
    // invert p -> (i, j): i = floor((1 + sqrt(1 + 8p)) / 2)
    int i = static_cast<int>((1.f + sqrtf(1.f + 8.f * p)) * 0.5f);
    while (i * (i - 1) / 2 > p) --i;
    while ((i + 1) * i / 2 <= p) ++i;
    const int j = p - i * (i - 1) / 2;
    const float* a = my + i * ZLD;
    const float* b = my + j * ZLD;
    float s = 0.f;
#pragma unroll 16
    for (int k = 0; k < 64; ++k) s = fmaf(a[k], b[k], s);
    o[64 + p] = __float2bfloat16_rn(s);
  }
  for (int64_t c = 64 + P + lane; c < out_cols; c += 32) o[c] = __float2bfloat16_rn(0.f);
}

// dz[m, i, :] = sum_{j != i} dpair(i,j) z[m, j, :]  (+ dout[m, 0:D] for i = 0),
// times relu'(z_0) on feature 0 when mask_first (the bottom MLP's ReLU output).
__global__ void __launch_bounds__(128) interaction_bwd_kernel(bf16* __restrict__ dz, int64_t lddz,
                                                              const bf16* __restrict__ dout,
                                                              int64_t lddo,
                                                              const bf16* __restrict__ z,
                                                              int64_t ldz, int64_t M, int F,
                                                              int mask_first) {
  extern __shared__ float sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m = static_cast<int64_t>(blockIdx.x) * 4 + w;
  if (m >= M) return;
  const int P = F * (F - 1) / 2;
  float* zsm = sm + w * (F * ZLD + P + 1);
  float* dp = zsm + F * ZLD;
  const bf16* zr = z + m * ldz;
  for (int i = 0; i < F; ++i) {
    const float2 v = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(zr + i * 64)[lane]);
    zsm[i * ZLD + 2 * lane] = v.x;
    zsm[i * ZLD + 2 * lane + 1] = v.y;
  }
  const bf16* dr = dout + m * lddo;
  for (int p = lane; p < P; p += 32) dp[p] = __bfloat162float(dr[64 + p]);
  __syncwarp();
  bf16* o = dz + m * lddz;
  for (int i = 0; i < F; ++i) {
    float a0 = 0.f, a1 = 0.f;
    for (int j = 0; j < F; ++j) {
      if (j == i) continue;
      const int p = i > j ? i * (i - 1) / 2 + j : j * (j - 1) / 2 + i;
      const float g = dp[p];
      a0 = fmaf(g, zsm[j * ZLD + 2 * lane], a0);
      a1 = fmaf(g, zsm[j * ZLD + 2 * lane + 1], a1);
    }
    if (i == 0) {
      a0 += __bfloat162float(dr[2 * lane]);
      a1 += __bfloat162float(dr[2 * lane + 1]);
      if (mask_first) {
        a0 = zsm[2 * lane] > 0.f ? a0 : 0.f;
        a1 = zsm[2 * lane + 1] > 0.f ? a1 : 0.f;
      }
    }
    reinterpret_cast<__nv_bfloat162*>(o + i * 64)[lane] = __floats2bfloat162_rn(a0, a1);
  }
}

// Same arithmetic (same j order, same fmaf chain -> bit-identical) with the feature count
// fixed at compile time: each lane keeps its two columns of all F features in registers,
// so the inner loop reads only the broadcast dp[p] from shared memory (the generic kernel
// above reads a z value from smem per FMA: ~150 us per DLRM step at B = 8192).
template <int F>
__global__ void __launch_bounds__(128) interaction_bwd_reg_kernel(bf16* __restrict__ dz, int64_t lddz,
                                                                  const bf16* __restrict__ dout,
                                                                  int64_t lddo,
                                                                  const bf16* __restrict__ z,
                                                                  int64_t ldz, int64_t M, int mask_first) {
  constexpr int P = F * (F - 1) / 2;
  __shared__ float dps[4][P + 1];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m = static_cast<int64_t>(blockIdx.x) * 4 + w;
  if (m >= M) return;
  float* dp = dps[w];
  const bf16* zr = z + m * ldz;
  float z0[F], z1[F];
#pragma unroll
  for (int i = 0; i < F; ++i) {
    const float2 v = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(zr + i * 64)[lane]);
    z0[i] = v.x;
    z1[i] = v.y;
  }
  const bf16* dr = dout + m * lddo;
  for (int p = lane; p < P; p += 32) dp[p] = __bfloat162float(dr[64 + p]);
  __syncwarp();
  bf16* o = dz + m * lddz;
#pragma unroll
  for (int i = 0; i < F; ++i) {
    float a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int j = 0; j < F; ++j) {
      if (j == i) continue;
      const float g = dp[i > j ? i * (i - 1) / 2 + j : j * (j - 1) / 2 + i];
      a0 = fmaf(g, z0[j], a0);
      a1 = fmaf(g, z1[j], a1);
    }
    if (i == 0) {
      a0 += __bfloat162float(dr[2 * lane]);
      a1 += __bfloat162float(dr[2 * lane + 1]);
      if (mask_first) {
        a0 = z0[0] > 0.f ? a0 : 0.f;
        a1 = z1[0] > 0.f ? a1 : 0.f;
      }
    }
    reinterpret_cast<__nv_bfloat162*>(o + i * 64)[lane] = __floats2bfloat162_rn(a0, a1);
  }
}

}  // namespace
}  // namespace gpp

using namespace gpp;

extern "C" {

int gpp_embbag_bad_indices(uint64_t* count, int reset) {
  GPP_ARG_CHECK(count, "bad argument");
  unsigned long long v = 0;
  cudaError_t e = cudaMemcpyFromSymbol(&v, g_bad_indices, sizeof(v));
  if (e == cudaSuccess && reset && v) {
    const unsigned long long zero = 0;
    e = cudaMemcpyToSymbol(g_bad_indices, &zero, sizeof(zero));
  }
  if (e != cudaSuccess) {
    set_error(std::string("gpp_embbag_bad_indices: ") + cudaGetErrorString(e));
    return GPP_ERR_CUDA;
  }
  *count = v;
  return GPP_OK;
}

int gpp_embbag_fwd(void* out, int64_t ldo, const float* table, const int64_t* idx, int64_t ldi,
                   int64_t M, int64_t bag, int64_t D, int64_t rows, void* stream) {
  GPP_ARG_CHECK(out && table && idx && M > 0 && bag > 0, "bad argument");
  GPP_ARG_CHECK(D == 64, "embedding dim must be 64 (Appendix B DLRM)");
  GPP_ARG_CHECK((reinterpret_cast<uintptr_t>(table) & 7) == 0 && ldo % 2 == 0, "alignment");
  embbag_fwd_kernel<<<static_cast<unsigned>((M + 7) / 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<bf16*>(out), ldo, table, idx, ldi, M, static_cast<int>(bag), rows);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_embbag_sgd(float* table, const void* dpooled, int64_t ldd, const int64_t* idx, int64_t ldi,
                   int64_t M, int64_t bag, int64_t D, int64_t rows, float lr, void* stream) {
  GPP_ARG_CHECK(table && dpooled && idx && M > 0 && bag > 0, "bad argument");
  GPP_ARG_CHECK(D == 64, "embedding dim must be 64");
  embbag_sgd_kernel<<<static_cast<unsigned>((M + 7) / 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      table, static_cast<const bf16*>(dpooled), ldd, idx, ldi, M, static_cast<int>(bag), lr, rows);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_interaction_fwd(void* out, int64_t ldo, int64_t out_cols, const void* z, int64_t ldz,
                        int64_t M, int64_t F, int64_t D, void* stream) {
  GPP_ARG_CHECK(out && z && M > 0 && F >= 2 && D == 64, "bad argument");
  GPP_ARG_CHECK(out_cols >= 64 + F * (F - 1) / 2 && out_cols <= ldo, "output too narrow");
  const size_t smem = 4 * F * ZLD * sizeof(float);
  interaction_fwd_kernel<<<static_cast<unsigned>((M + 3) / 4), 128, smem, static_cast<cudaStream_t>(stream)>>>(
      static_cast<bf16*>(out), ldo, out_cols, static_cast<const bf16*>(z), ldz, M, static_cast<int>(F));
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_interaction_bwd(void* dz, int64_t lddz, const void* dout, int64_t lddo, const void* z,
                        int64_t ldz, int64_t M, int64_t F, int64_t D, int mask_first, void* stream) {
  GPP_ARG_CHECK(dz && dout && z && M > 0 && F >= 2 && D == 64, "bad argument");
  // GPP_INTERACTION_GENERIC=1 forces the generic kernel (tests assert both are bit-identical)
  const char* gen = getenv("GPP_INTERACTION_GENERIC");
  if (F == 27 && !(gen && gen[0] == '1')) {  // DLRM: 26 tables + the bottom MLP
    interaction_bwd_reg_kernel<27><<<static_cast<unsigned>((M + 3) / 4), 128, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<bf16*>(dz), lddz, static_cast<const bf16*>(dout), lddo, static_cast<const bf16*>(z), ldz, M,
        mask_first);
    GPP_LAUNCH_CHECK();
    return GPP_OK;
  }
  const size_t smem = 4 * (F * ZLD + F * (F - 1) / 2 + 1) * sizeof(float);
  interaction_bwd_kernel<<<static_cast<unsigned>((M + 3) / 4), 128, smem, static_cast<cudaStream_t>(stream)>>>(
      static_cast<bf16*>(dz), lddz, static_cast<const bf16*>(dout), lddo, static_cast<const bf16*>(z), ldz, M,
      static_cast<int>(F), mask_first);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

}  // extern "C"
