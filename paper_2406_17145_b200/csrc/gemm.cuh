// GEMM epilogue contract shared by the tcgen05 (bf16) and SIMT (fp32) GEMMs.
#pragma once
#include "common.cuh"

namespace gpp {

enum {
  EPI_FWD = 0,    // out(dtype) = act(alpha*acc + bias) [+ residual];  optional pre-act store
  EPI_DGRAD = 1,  // out(dtype) = alpha*acc * act'(saved)
  EPI_F32 = 2,    // out(f32)   = alpha*acc + beta*out
  EPI_BF16 = 3,   // out(dtype) = alpha*acc + beta*out
  EPI_SGD = 4     // wgrad + fused SGD: g = alpha*acc (+ grad if beta); [grad = g];
                  // out(f32 master) -= lr*g; pre(bf16 shadow) = bf16(master)
};

struct EpiParams {
  void* out;
  int64_t ldo;
  const float* bias;  // EPI_FWD: [N] or null
  const void* aux;    // EPI_FWD: residual (dtype); EPI_DGRAD: act'-saved (dtype)
  int64_t ldaux;
  void* pre;          // EPI_FWD: optional pre-activation store (dtype)
  int64_t ldpre;
  float alpha;
  float beta;
  int act;
  float lr;          // EPI_SGD
  float* grad;       // EPI_SGD: fp32 gradient buffer (read if beta != 0, written if store_grad)
  int64_t ldgrad;
  int store_grad;
  int64_t split_stride;  // split-K: partial s is written at (float*)out + s * split_stride
  const void* pf_ptr;    // L2 prefetch hint: bytes another kernel will read next (or null)
  int64_t pf_bytes;
  // wgrad (A = dy^T, MN-major): also colsum[m] (+)= sum_k A[m, k] -- the bias gradient,
  // summed from the A tiles already staged in shared memory (or one column-sum kernel
  // after the GEMM where that is not possible: split-K, 1-CTA tiles, fp32)
  float* colsum;
  int colsum_acc;
};

// One-shot L2 prefetch hint consumed by the next GEMM launched on this host thread.
void take_prefetch_hint(EpiParams& ep);

// Batched GEMM (attention): batch z = hi * nlo + lo.  Each batch multiplies logical
// sub-matrices of the SAME 2-D operands, offset in (m, k) / (n, k) coordinates, and
// writes C (and aux / pre) at element offset z_hi * c_hi + z_lo * c_lo.  Requires the
// per-batch K to be a multiple of 64 (a K-tile never straddles two batches).
struct BatchSpec {
  int nbatch = 1, nlo = 1;
  int a_m0 = 0, a_m_hi = 0, a_m_lo = 0, a_k0 = 0, a_k_hi = 0, a_k_lo = 0;
  int b_n0 = 0, b_n_hi = 0, b_n_lo = 0, b_k0 = 0, b_k_hi = 0, b_k_lo = 0;
  int64_t c0 = 0, c_hi = 0, c_lo = 0;
};

// Batched bf16 GEMM (1-CTA tcgen05 kernel over batch x tiles).
// Attention scores + fused softmax (bwd = 0: P = softmax(alpha Q K^T)) or fused softmax
// backward (bwd = 1: dS = alpha P o (dO V^T - rowsum(P o dO V^T))); both operands K-major,
// keys N <= 512.  P / out share the BatchSpec C offsets.
int tc_attn_softmax(int bwd, void* out, int64_t ldc, const void* P, int64_t ldp, const void* a, int64_t lda,
                    int64_t a_rows, const void* b, int64_t ldb, int64_t b_rows, const BatchSpec& bs, int64_t M,
                    int64_t N, int64_t K, float alpha, cudaStream_t stream);

int tc_gemm_batched(int epi, const void* a, int64_t lda, int64_t a_rows, int a_mn, const void* b,
                    int64_t ldb, int64_t b_rows, int b_mn, const EpiParams& ep, const BatchSpec& bs,
                    int64_t M, int64_t N, int64_t K, cudaStream_t stream);
// MMT attention, one CTA per (sample x head, 128 query rows), S % 128 == 0, S <= 512,
// head dim 64, packed QKV [T, 3d] (attn_sm100.cu):
//   fw : P = softmax(alpha Q K^T) -> HBM (for the backward), O = P V  -> o[:, head*64..]
//   bw : dP = dO V^T, D = rowsum(dO o O), dS = alpha P o (dP - D) -> HBM, dQ = dS K -> dqkv
int tc_attn_fwd(const void* qkv, void* P, void* o, int64_t ldo, int64_t m, int64_t S, int64_t d, int64_t H,
                float alpha, cudaStream_t stream);
int tc_attn_bwd(const void* qkv, const void* P, const void* o, int64_t ldo, const void* dout, int64_t lddo,
                void* dS, void* dqkv, int64_t m, int64_t S, int64_t d, int64_t H, float alpha, cudaStream_t stream);
// bf16 operands, tcgen05 + TMA (gemm_sm100.cu).
int tc_gemm(int epi, const void* a, int64_t lda, int a_mn, const void* b, int64_t ldb, int b_mn,
            const EpiParams& ep, int64_t M, int64_t N, int64_t K, cudaStream_t stream);
// fp32 operands, SIMT FFMA (gemm_simt.cu) — exact-fp32 path for the toy config.
int simt_gemm(int epi, const void* a, int64_t lda, int a_mn, const void* b, int64_t ldb,
              int b_mn, const EpiParams& ep, int64_t M, int64_t N, int64_t K,
              cudaStream_t stream);

}  // namespace gpp
