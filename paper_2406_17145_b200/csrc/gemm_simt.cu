// Exact-fp32 SIMT GEMM (FFMA) with the same layout flags and fused epilogues as the
// tcgen05 path.  Used for the fp32 toy config (BASELINE.json configs[0]), whose
// rtol 1e-4 rules out TF32 tensor cores, and for tiny heads.
#include "gemm.cuh"

namespace gpp {
namespace simt {

constexpr int TM = 64, TN = 64, TK = 16;

template <int EPI>
__device__ __forceinline__ void epi_scalar(const EpiParams& ep, float acc, int row, int col) {
  float v = acc * ep.alpha;
  if constexpr (EPI == EPI_FWD) {
    if (ep.bias) v += ep.bias[col];
    if (ep.pre) static_cast<float*>(ep.pre)[static_cast<int64_t>(row) * ep.ldpre + col] = v;
    v = act_fwd(v, ep.act);
    if (ep.aux) v += static_cast<const float*>(ep.aux)[static_cast<int64_t>(row) * ep.ldaux + col];
  } else if constexpr (EPI == EPI_DGRAD) {
    if (ep.act != GPP_ACT_NONE)
      v *= act_bwd(static_cast<const float*>(ep.aux)[static_cast<int64_t>(row) * ep.ldaux + col],
                   ep.act);
  }
  if constexpr (EPI == EPI_SGD) {
    float* grad = ep.grad + static_cast<int64_t>(row) * ep.ldgrad + col;
    const float g = v + (ep.beta != 0.f ? *grad : 0.f);
    if (ep.store_grad) *grad = g;
    float* master = static_cast<float*>(ep.out) + static_cast<int64_t>(row) * ep.ldo + col;
    *master -= ep.lr * g;
    return;
  }
  float* out = static_cast<float*>(ep.out) + static_cast<int64_t>(row) * ep.ldo + col;
  if constexpr (EPI == EPI_F32 || EPI == EPI_BF16) {
    if (ep.beta != 0.f) v += ep.beta * *out;
  }
  *out = v;
}

template <bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(256)
    gemm_simt_kernel(const float* __restrict__ A, int64_t lda, const float* __restrict__ B,
                     int64_t ldb, EpiParams ep, int M, int N, int K) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int k0 = 0; k0 < K; k0 += TK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = threadIdx.x + i * 256;
      int r, kk;
      if (A_MN) { r = e % TM; kk = e / TM; } else { kk = e % TK; r = e / TK; }
      const int gr = m0 + r, gk = k0 + kk;
      float v = 0.f;
      if (gr < M && gk < K)
        v = A_MN ? A[static_cast<int64_t>(gk) * lda + gr] : A[static_cast<int64_t>(gr) * lda + gk];
      As[kk][r] = v;
      if (B_MN) { r = e % TN; kk = e / TN; } else { kk = e % TK; r = e / TK; }
      const int gn = n0 + r, gk2 = k0 + kk;
      float w = 0.f;
      if (gn < N && gk2 < K)
        w = B_MN ? B[static_cast<int64_t>(gk2) * ldb + gn] : B[static_cast<int64_t>(gn) * ldb + gk2];
      Bs[kk][r] = w;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + ty * 4 + i;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = n0 + tx * 4 + j;
      if (col < N) epi_scalar<EPI>(ep, acc[i][j], row, col);
    }
  }
}

template <int EPI>
static int launch(const void* a, int64_t lda, int a_mn, const void* b, int64_t ldb, int b_mn,
                  const EpiParams& ep, int64_t M, int64_t N, int64_t K, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((N + TN - 1) / TN), static_cast<unsigned>((M + TM - 1) / TM));
  const float* A = static_cast<const float*>(a);
  const float* B = static_cast<const float*>(b);
  const int m = static_cast<int>(M), n = static_cast<int>(N), k = static_cast<int>(K);
  if (!a_mn && !b_mn) gemm_simt_kernel<false, false, EPI><<<grid, 256, 0, s>>>(A, lda, B, ldb, ep, m, n, k);
  else if (!a_mn && b_mn) gemm_simt_kernel<false, true, EPI><<<grid, 256, 0, s>>>(A, lda, B, ldb, ep, m, n, k);
  else if (a_mn && !b_mn) gemm_simt_kernel<true, false, EPI><<<grid, 256, 0, s>>>(A, lda, B, ldb, ep, m, n, k);
  else gemm_simt_kernel<true, true, EPI><<<grid, 256, 0, s>>>(A, lda, B, ldb, ep, m, n, k);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

}  // namespace simt

int simt_gemm(int epi, const void* a, int64_t lda, int a_mn, const void* b, int64_t ldb,
              int b_mn, const EpiParams& ep, int64_t M, int64_t N, int64_t K,
              cudaStream_t stream) {
  GPP_ARG_CHECK(M > 0 && N > 0 && K > 0, "M, N, K must be positive");
  GPP_ARG_CHECK(M < (1LL << 31) && N < (1LL << 31) && K < (1LL << 31), "dimension too large");
  switch (epi) {
    case EPI_FWD: return simt::launch<EPI_FWD>(a, lda, a_mn, b, ldb, b_mn, ep, M, N, K, stream);
    case EPI_DGRAD: return simt::launch<EPI_DGRAD>(a, lda, a_mn, b, ldb, b_mn, ep, M, N, K, stream);
    case EPI_F32: return simt::launch<EPI_F32>(a, lda, a_mn, b, ldb, b_mn, ep, M, N, K, stream);
    case EPI_SGD: return simt::launch<EPI_SGD>(a, lda, a_mn, b, ldb, b_mn, ep, M, N, K, stream);
    default: return simt::launch<EPI_BF16>(a, lda, a_mn, b, ldb, b_mn, ep, M, N, K, stream);
  }
}

}  // namespace gpp
