/*
 * gpp_b200.h — C-ABI of the B200 (sm_100a) stage-executor library `libgpp_b200.so`.
 *
 * This is the drop-in boundary below the Python GPP runtime
 * (paper_2406_17145_b200.runtime).  The reference (arXiv 2406.17145, /root/reference)
 * ships NO runtime: its executor was FlexFlow on V100 and
 * SPEC.md:8 puts it out of scope.  The executor's contract is therefore the
 * simulator's task semantics applied to a configured
 * `StageGraph` (reference pkg/src/gpp/model.py:278-345).  Each entry point
 * below replaces one piece of per-task work that the reference models only as
 * an abstract `CostCurve.evaluate` call (model.py:65-92) inside
 * `estimate_tps` (cost.py:56-70) and the sim's task durations:
 *
 *   gpp_linear_fwd / gpp_linear_dgrad / gpp_linear_wgrad
 *        the fw / bw(input) / bw(weight) work of a dense operator
 *        (Operator.fwd_cost / bwd_cost, model.py:100-114; Appendix B
 *        feed-forward layers)
 *   gpp_gemm                    generic layout-flagged GEMM (tests, attention glue)
 *   gpp_rowdot_fwd / _bwd       N=1 regression / CTR heads (CANDLE MSE, DLRM BCE)
 *   gpp_mse_loss / gpp_bce_loss / gpp_ce_loss   fused loss + dLoss kernels
 *   gpp_colsum                  bias gradient
 *   gpp_sgd_step                fused optimizer over a stage's parameters
 *   gpp_layernorm_fwd / _bwd, gpp_softmax_fwd / _bwd, gpp_meanpool_fwd / _bwd,
 *   gpp_gemm_batched            MMT pre-LN transformer layer (attention as batched GEMMs)
 *   gpp_flash_attn_fwd / _bwd         MMT attention, P recomputed (O + LSE forward; dQ, dK, dV backward)
 *   gpp_attn_fwd / gpp_attn_bwd       fused MMT attention (softmax + P.V / softmax-bwd + dS.K)
 *   gpp_attn_softmax / gpp_attn_softmax_bwd  attention scores with the softmax (or its
 *                               backward) fused into the tcgen05 epilogue (S <= 512)
 *   gpp_embbag_fwd / gpp_embbag_sgd        DLRM embedding-bag and its sparse SGD scatter
 *   gpp_interaction_fwd / _bwd  DLRM dot interaction
 *   gpp_copy_rows               strided row-block copy (concat slices, DP re-shard,
 *                               same-device stage edges)
 *   gpp_copy_rows_multi         all slices of one concat / split in one launch
 *
 * Conventions:
 *   - every function returns 0 on success, a nonzero gpp_status otherwise;
 *     gpp_last_error() returns a thread-local message for the last failure;
 *   - all device memory is owned by the caller (PyTorch caching allocator);
 *     the library never allocates or frees user tensors;
 *   - `stream` is a cudaStream_t passed as void*; every launch is async on it;
 *   - row-major matrices; `ld*` are leading dimensions in ELEMENTS;
 *   - dtype: GPP_F32 (SIMT FFMA path, exact fp32) or GPP_BF16 (tcgen05 path,
 *     bf16 operands, fp32 accumulation in TMEM).
 */
#ifndef GPP_B200_H
#define GPP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum gpp_status {
  GPP_OK = 0,
  GPP_ERR_ARG = 1,      /* invalid shape / pointer / alignment */
  GPP_ERR_CUDA = 2,     /* a CUDA runtime call failed */
  GPP_ERR_DRIVER = 3,   /* driver entry point (TMA descriptor encode) failed */
  GPP_ERR_UNSUPPORTED = 4
};

enum gpp_dtype { GPP_F32 = 0, GPP_BF16 = 1 };
enum gpp_act { GPP_ACT_NONE = 0, GPP_ACT_RELU = 1, GPP_ACT_GELU = 2 };

/* ---- library ---------------------------------------------------------- */
int gpp_version(void);
/* "gpp-digest:<sha256>" of the csrc/include sources and nvcc flags the binary was built
 * from: build() rebuilds and lib.load() refuses a binary whose digest is stale. */
const char* gpp_source_digest(void);
const char* gpp_last_error(void);
/* Number of kernels this library has launched since load (evidence counter). */
uint64_t gpp_launch_count(void);

/* One-shot hint: the next GEMM launched from this thread also prefetches
 * [ptr, ptr + bytes) into L2 (spread over its CTAs, overlapping its main loop) — the
 * executor points it at the weights / fp32 master the following kernel will read. */
int gpp_gemm_prefetch_hint(const void* ptr, int64_t bytes);

/* ---- dense operator (Operator fw/bw work, model.py:100-114) ------------- */

/* y[M,N] = act(x[M,K] · w[N,K]^T + bias[N]) (+ residual[M,N] if non-null).
 * If pre_out != NULL it also stores the pre-activation (needed by GELU bw). */
int gpp_linear_fwd(void* y, int64_t ldy, const void* x, int64_t ldx, const void* w, int64_t ldw,
                   const float* bias, const void* residual, int64_t ldres, void* pre_out,
                   int64_t ldpre, int64_t M, int64_t N, int64_t K, int act, int dtype,
                   void* stream);

/* dx[M,K] = (dy[M,N] · w[N,K]) ⊙ act'(saved[M,K]).
 * act is the activation that PRODUCED dx's forward value (the predecessor's):
 * RELU uses saved = that activation's output (mask saved > 0), GELU uses
 * saved = its pre-activation; NONE ignores saved. */
int gpp_linear_dgrad(void* dx, int64_t lddx, const void* dy, int64_t lddy, const void* w,
                     int64_t ldw, const void* saved, int64_t ldsaved, int64_t M, int64_t N,
                     int64_t K, int act, int dtype, void* stream);

/* dw[N,K] (+)= dy[M,N]^T · x[M,K]  (fp32 out);  dbias[N] (+)= sum_m dy[m,:].
 * The bias column sums are read from the dy tiles the GEMM already stages in shared
 * memory (an extra warp of the CTA-pair kernel) -- no second pass over dy -- except for
 * split-K / single-CTA / fp32 launches, which add one column-sum kernel. */
int gpp_linear_wgrad(float* dw, int64_t lddw, float* dbias, const void* dy, int64_t lddy,
                     const void* x, int64_t ldx, int64_t M, int64_t N, int64_t K,
                     int accumulate, int dtype, void* stream);

/* wgrad of the LAST micro-batch fused with SGD (stages without data parallelism):
 *   g = dy[M,N]^T x[M,K] (+ grad if accumulate);  [grad = g if store_grad];
 *   master[N,K] -= lr * g;  shadow = bf16(master)   (shadow ignored for GPP_F32).
 * Replaces gpp_linear_wgrad + the weight part of gpp_sgd_step (saves the fp32
 * gradient round trip through HBM). */
int gpp_linear_wgrad_sgd(float* master, int64_t ldm, void* shadow, int64_t lds, float* grad,
                         int64_t ldg, float lr, int accumulate, int store_grad, const void* dy,
                         int64_t lddy, const void* x, int64_t ldx, int64_t M, int64_t N, int64_t K,
                         float* dbias, int dtype, void* stream);

/* Generic C[M,N] = alpha * sum_k A(m,k) B(n,k) (+ beta*C).
 * a_mn / b_mn = 0: operand stored [rows][ld] with k contiguous (K-major);
 *             = 1: operand stored [k][ld] with the row index contiguous (MN-major).
 * out_f32 selects fp32 vs bf16 C (bf16 inputs); for dtype F32 everything is fp32. */
int gpp_gemm(void* c, int64_t ldc, const void* a, int64_t lda, int a_mn, const void* b,
             int64_t ldb, int b_mn, int64_t M, int64_t N, int64_t K, float alpha, float beta,
             int out_f32, int dtype, void* stream);

/* ---- heads and losses (Appendix B tails; SURVEY.md §2.3 note B) --------- */

/* out[m] = dot(x[m,:K], w[:K]) + bias[0]   (fp32 out; x in dtype; bias may be NULL). */
int gpp_rowdot_fwd(float* out, const void* x, int64_t ldx, const float* w, const float* bias,
                   int64_t M, int64_t K, int dtype, void* stream);
/* dx[m,k] = dout[m] * w[k] * act'(saved[m,k]);  dw[k] (+)= sum_m dout[m] x[m,k];
 * dbias[0] (+)= sum_m dout[m]. */
int gpp_rowdot_bwd(void* dx, int64_t lddx, float* dw, float* dbias, const float* dout,
                   const void* x, int64_t ldx, const float* w, const void* saved,
                   int64_t ldsaved, int act, int64_t M, int64_t K, int accumulate, int dtype,
                   void* stream);
/* The N=1 head and its loss in ONE kernel: z[m] = dot(x[m,:K], w) + bias[0], then
 * kind 0 (MSE): loss_acc[0] += scale sum (z-y)^2, dz = 2 scale (z-y);
 * kind 1 (BCE-with-logits): loss_acc[0] += scale sum l(z,y), dz = scale (sigmoid(z)-y).
 * Deterministic (fixed-order block partials).  Replaces gpp_rowdot_fwd + gpp_mse_loss /
 * gpp_bce_loss on the executor's head stages. */
int gpp_rowdot_loss(float* z, float* dz, float* loss_acc, const void* x, int64_t ldx, const float* w,
                    const float* bias, const float* y, int64_t M, int64_t K, int kind, float scale, int dtype,
                    void* stream);
/* loss_acc[0] += scale * sum (pred-y)^2 ;  dpred = 2*scale*(pred - y). */
int gpp_mse_loss(float* loss_acc, float* dpred, const float* pred, const float* y, int64_t M,
                 float scale, void* stream);
/* BCE-with-logits: loss_acc[0] += scale*sum l(z,y); dz = scale*(sigmoid(z)-y). */
int gpp_bce_loss(float* loss_acc, float* dlogit, const float* logit, const float* y, int64_t M,
                 float scale, void* stream);
/* softmax cross-entropy over C classes: logits [M,C] (dtype), labels int64 [M];
 * loss_acc[0] += scale*sum -log p[label];  dlogits = scale*(p - onehot) (same dtype). */
int gpp_ce_loss(float* loss_acc, void* dlogits, int64_t lddl, const void* logits, int64_t ldl,
                const int64_t* labels, int64_t M, int64_t C, float scale, int dtype,
                void* stream);

/* colsum: out[n] (+)= sum_m x[m,n] (x in dtype, out fp32). */
/* out_i[:N_i] (+)= column sums of x_i [M_i, N_i] for i < n, in as few launches as possible
 * (the bias gradients of a whole backward task: one launch instead of one per layer).
 * Host arrays; each sum is deterministic (fixed-order partials). */
int gpp_colsum_multi(int n, const void* const* x, const int64_t* ldx, const int64_t* M, const int64_t* N,
                     float* const* out, int accumulate, int dtype, void* stream);
int gpp_colsum(float* out, const void* x, int64_t ldx, int64_t M, int64_t N, int accumulate,
               int dtype, void* stream);

/* ---- optimizer ----------------------------------------------------------- */
/* master[i] -= lr * grad[i]; if shadow (bf16) != NULL also shadow[i] = bf16(master[i]). */
int gpp_sgd_step(float* master, void* shadow_bf16, const float* grad, int64_t n, float lr,
                 void* stream);

/* ---- data movement ------------------------------------------------------- */
/* dst[r, :cols] = src[r, :cols] for r < rows (same device; elem_bytes 2 or 4). */
int gpp_copy_rows(void* dst, int64_t lddst, const void* src, int64_t ldsrc, int64_t rows,
                  int64_t cols, int elem_bytes, void* stream);
/* n slices of one concat / split (same rows) in one launch:
 * dst[k][r, :cols[k]] = src[k][r, :cols[k]].  The arrays are read during the call (a
 * captured graph keeps its own copy).  Replaces the per-predecessor slice copies of the
 * reference executor's concat (PAPER.md:589 stage executor; not in the reference code). */
int gpp_copy_rows_multi(int n, void* const* dst, const int64_t* lddst, const void* const* src,
                        const int64_t* ldsrc, int64_t rows, const int64_t* cols, int elem_bytes,
                        void* stream);
/* dst_f32[i] = float(src[i]) or dst_bf16[i] = bf16(src_f32[i]). */
int gpp_cast(void* dst, int dst_dtype, const void* src, int src_dtype, int64_t n, void* stream);

/* ---- MMT transformer layer: pre-LN, attention softmax, mean-pool ---- */
/* y = LN(x) * gamma + beta per row of D (D in {128,256,512,1024}); saves mean / rstd [T]. */
int gpp_layernorm_fwd(void* y, float* mean, float* rstd, const void* x, const float* gamma,
                      const float* beta, int64_t T, int64_t D, float eps, void* stream);
/* dx = LN'(dy) (+ dres, the residual-branch gradient); dgamma/dbeta (+)= column sums. */
int gpp_layernorm_bwd(void* dx, float* dgamma, float* dbeta, const void* dy, const void* x,
                      const float* mean, const float* rstd, const float* gamma, const void* dres,
                      int64_t T, int64_t D, int accumulate, void* stream);
/* P[R, L] = softmax(scores) row-wise (fp32 scores, pre-scaled), bf16 out. */
int gpp_softmax_fwd(void* p, const float* scores, int64_t R, int64_t L, void* stream);
/* dS = scale * P * (dP - rowsum(dP * P)). */
int gpp_softmax_bwd(void* ds, const void* p, const float* dp, int64_t R, int64_t L, float scale,
                    void* stream);
/* out[m, :D] = mean over S token rows of x[m*S : (m+1)*S, :D];  bwd broadcasts dout / S. */
int gpp_meanpool_fwd(void* out, int64_t ldo, const void* x, int64_t M, int64_t S, int64_t D,
                     void* stream);
int gpp_meanpool_bwd(void* dx, const void* dout, int64_t lddo, int64_t M, int64_t S, int64_t D,
                     void* stream);
/* Batched GEMM over batch z = hi*nlo + lo (attention: z = sample*heads + head): each batch
 * multiplies sub-matrices of the same operands at (m,k)/(n,k) coordinate offsets
 * X0 + hi*X_hi + lo*X_lo and writes C at element offset c0 + hi*c_hi + lo*c_lo.
 * spec = {nbatch, nlo, a_m0, a_m_hi, a_m_lo, a_k0, a_k_hi, a_k_lo, b_n0, b_n_hi, b_n_lo,
 *         b_k0, b_k_hi, b_k_lo, c0, c_hi, c_lo};
 * a_rows / b_rows = row counts of the full operands; K % 64 == 0. */
int gpp_gemm_batched(void* c, int64_t ldc, const void* a, int64_t lda, int64_t a_rows, int a_mn,
                     const void* b, int64_t ldb, int64_t b_rows, int b_mn, int64_t M, int64_t N,
                     int64_t K, float alpha, float beta, int out_f32, const int64_t* spec,
                     void* stream);
/* Fused attention softmax over the same batch spec (both operands K-major, keys N <= 512,
 * N % 32 == 0, head dim K % 64 == 0, K <= 256):
 *   gpp_attn_softmax:      p[z] = softmax_rows(scale * q[z] k[z]^T)            (bf16 out)
 *   gpp_attn_softmax_bwd:  ds[z] = scale * p[z] o (g[z] - rowsum(p[z] o g[z])),
 *                          g[z] = dout[z] v[z]^T                              (bf16 out)
 * p / ds rows at c0 + hi*c_hi + lo*c_lo with leading dims ldp / ldc.  Replaces the scores
 * GEMM + softmax (+ backward) pair of the MMT attention without the fp32 scores in HBM. */
int gpp_attn_softmax(void* p, int64_t ldp, const void* q, int64_t ldq, int64_t q_rows, const void* k,
                     int64_t ldk, int64_t k_rows, int64_t M, int64_t N, int64_t K, float scale,
                     const int64_t* spec, void* stream);
int gpp_attn_softmax_bwd(void* ds, int64_t ldc, const void* p, int64_t ldp, const void* dout, int64_t ldo,
                         int64_t o_rows, const void* v, int64_t ldv, int64_t v_rows, int64_t M, int64_t N,
                         int64_t K, float scale, const int64_t* spec, void* stream);

/* Fused MMT attention (one launch per direction; attn_sm100.cu).  Packed QKV [m*S, 3d]
 * (Q | K | V, head h in columns h*64 .. h*64+63), z = sample*H + head, P / ds [m*H*S, S]:
 *   gpp_attn_fwd:  p[z] = softmax(scale q[z] k[z]^T)  (stored for the backward) and
 *                  o[:, h*64..] = p[z] v[z]                                 (bf16)
 *   gpp_attn_bwd:  ds[z] = scale p[z] o (dout[z] v[z]^T - D),  D = rowsum(dout o o),
 *                  dqkv[:, h*64..] (the Q block) = ds[z] k[z]                 (bf16)
 * Requires d == 64 H, S in {128, 256, 384, 512}.  Replaces gpp_attn_softmax + the P.V
 * gpp_gemm_batched (fw) and gpp_attn_softmax_bwd + the dS.K gpp_gemm_batched (bw). */
int gpp_attn_fwd(const void* qkv, void* p, void* o, int64_t ldo, int64_t m, int64_t S, int64_t d, int64_t H,
                 float scale, void* stream);
int gpp_attn_bwd(const void* qkv, const void* p, const void* o, int64_t ldo, const void* dout, int64_t lddo,
                 void* ds, void* dqkv, int64_t m, int64_t S, int64_t d, int64_t H, float scale, void* stream);

/* Recompute-based (FlashAttention-style) MMT attention: nothing of size Z x S x S in HBM.
 *   gpp_flash_attn_fwd: o[:, h*64..] = softmax(scale q k^T) v, and per (z, query row) the
 *       base-2 log-sum-exp lse2 = scale log2(e) max + log2(sum) ([m*H, S] fp32).
 *   gpp_flash_attn_bwd: dvec = scale * rowsum(dout o o) (caller-owned [m*H, S] fp32 scratch), then
 *       with P recomputed from q, k, lse2: per (z, 128-key block) the dK and dV blocks of
 *       dqkv (summed over every query block in TMEM), per (z, 128-query block) dQ (summed
 *       over every key block in TMEM) -- two launches (prep + one persistent kernel), deterministic.
 * Same layouts and requirements (d == 64 H, S in {128, 256, 384, 512}) as gpp_attn_*;
 * they replace gpp_attn_fwd / gpp_attn_bwd and the two dV / dK batched GEMMs. */
int gpp_flash_attn_fwd(const void* qkv, float* lse2, void* o, int64_t ldo, int64_t m, int64_t S, int64_t d,
                       int64_t H, float scale, void* stream);
int gpp_flash_attn_bwd(const void* qkv, const float* lse2, const void* o, int64_t ldo, const void* dout,
                       int64_t lddo, float* dvec, void* dqkv, int64_t m, int64_t S, int64_t d, int64_t H,
                       float scale, void* stream);

/* ---- DLRM: embedding bags and the dot interaction ------------- */
/* pooled[m, :D] = sum_b table[idx[m*ldi + b], :D]; fp32 table [rows, D], bf16 pooled, D = 64.
 * An index outside [0, rows) contributes nothing (gather) / updates nothing (scatter) and
 * is counted; the host reads the count with gpp_embbag_bad_indices and raises (the
 * oracle's torch.nn.functional.embedding_bag raises IndexError on such input). */
int gpp_embbag_bad_indices(uint64_t* count, int reset);
int gpp_embbag_fwd(void* out, int64_t ldo, const float* table, const int64_t* idx, int64_t ldi,
                   int64_t M, int64_t bag, int64_t D, int64_t rows, void* stream);
/* Synchronous sparse SGD: table[idx[m, b], :] -= lr * dpooled[m, :] for all (m, b)
 * (fp32 atomics; applied once per iteration over the whole mini-batch). */
int gpp_embbag_sgd(float* table, const void* dpooled, int64_t ldd, const int64_t* idx, int64_t ldi,
                   int64_t M, int64_t bag, int64_t D, int64_t rows, float lr, void* stream);
/* Deterministic sparse SGD over n tables in one call: for every table t,
 * tables[t][r, :] -= lr * sum over {(m, b): idx[t][m*ldi + b] == r} of dpooled[t][m, :],
 * each row's sum taken in increasing (m, b) order (a counting sort by row, then one warp per
 * touched row) -- bit-reproducible, unlike gpp_embbag_sgd's fp32 atomics. */
int gpp_embbag_sgd_multi(int n, float* const* tables, const int64_t* rows, const void* const* dpooled, int64_t ldd,
                         const int64_t* const* idx, int64_t ldi, int64_t M, int64_t bag, int64_t D, float lr,
                         void* stream);
/* z [M, F*D] (feature 0 = dense/bottom vector): out[:, 0:D] = z_0, then the F(F-1)/2
 * pairwise dots <z_i, z_j> (i > j, row-major lower triangle), zero padding to out_cols. */
int gpp_interaction_fwd(void* out, int64_t ldo, int64_t out_cols, const void* z, int64_t ldz,
                        int64_t M, int64_t F, int64_t D, void* stream);
/* dz from dout; mask_first applies relu'(z_0) to feature 0's gradient. */
int gpp_interaction_bwd(void* dz, int64_t lddz, const void* dout, int64_t lddo, const void* z,
                        int64_t ldz, int64_t M, int64_t F, int64_t D, int mask_first, void* stream);

/* ---- transport (NCCL resolved at run time from the loaded libnccl.so.2) --------------
 * Stage-edge P2P pieces and the per-iteration DP all-reduce; one
 * communicator per ordered rank pair so forward and backward traffic never serialise. */
int gpp_nccl_available(void);
int gpp_nccl_unique_id(void* out128);
/* Initialise n communicators in one NCCL group: comm i has nranks[i] members, this
 * process is rank ranks[i], unique id at ids + 128*i; handles written to comms[i]. */
int gpp_comm_init_group(int n, const void* ids, const int* nranks, const int* ranks, void** comms);
int gpp_comm_destroy(void* comm);
int gpp_send(void* comm, const void* buf, int64_t bytes, int peer, void* stream);
int gpp_recv(void* comm, void* buf, int64_t bytes, int peer, void* stream);
int gpp_allreduce_f32(void* comm, void* buf, int64_t count, void* stream);
/* recv[r*bytes_per_rank ...] = send of DP rank r (embedding-gradient exchange). */
int gpp_allgather(void* comm, const void* send, void* recv, int64_t bytes_per_rank, void* stream);
int gpp_group_start(void);
int gpp_group_end(void);

#ifdef __cplusplus
}
#endif
#endif /* GPP_B200_H */
