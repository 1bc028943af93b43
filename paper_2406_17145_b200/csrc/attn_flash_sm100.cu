// Recompute-based MMT attention for sm_100a (S <= 512 keys, head dim 64).
// Nothing of size Z x S x S ever reaches HBM:
//
//   attn_fwd_lse_kernel : one CTA per (z = sample x head, 128 query rows).  S = Q K^T fills
//       TMEM (128 lanes x S fp32 columns); pass 1 takes the row max, pass 2 writes
//       e = exp2(alpha log2e (s - max)) as bf16 pairs over the consumed score columns and
//       sums them; O = E V (A operand straight from TMEM) is divided by the row sum in its
//       epilogue.  Stores O and the row's log-sum-exp in base 2:
//           lse2 = alpha log2e max + log2(sum),   P = exp2(alpha log2e s - lse2).
//   attn_bwd_prep_kernel: D[q] = rowsum(dO o O) per (z, query) -- the FlashAttention
//       identity rowsum(P o dP) = rowsum(dO o O).
//   attn_bwd_kv_kernel  : one CTA per (z, 128-key block), a cluster of S/128 CTAs per z.
//       For each 128-query block: S^T = K Q^T and dP^T = V dO^T (TMEM, lane = key), the
//       epilogue warps recompute P^T = exp2(alpha log2e s - lse2[q]) and
//       dS^T = alpha P^T o (dP^T - D[q]), write both as bf16 pairs back into TMEM (the A
//       operands of dV += P^T dO and dK += dS^T Q, accumulated in TMEM over all query
//       blocks) and dS^T into shared memory (the MN-major A operand of the partial
//       dQ_kb = dS K_kb).  The S/128 partial dQ blocks are summed across the cluster in a
//       fixed rank order through distributed shared memory (deterministic), by the CTA
//       that owns that query block.  dK, dV go out once, at the end.
//
// Layout: packed QKV [m S, 3d] (Q | K | V, head h at columns h*64), o / dout [m S, d]
// head-interleaved, lse2 / D [Z, S] fp32 with z = sample * H + head.
#include <cuda.h>

#include "gemm.cuh"
#include "tc_ptx.cuh"

namespace gpp {
namespace tc {

int make_map_bf16(CUtensorMap* out, const void* ptr, int64_t inner, int64_t outer, int64_t ld, int box_inner,
                  int box_outer);

namespace {

constexpr int FA_DH = 64;
constexpr int FW_EPI_WARPS = 8;                    // two per TMEM lane quarter (key halves)
constexpr int FW_THREADS = 64 + 32 * FW_EPI_WARPS;  // + TMA warp + MMA warp

__device__ __forceinline__ void fa_mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ uint32_t fa_pack(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

__device__ __forceinline__ void fa_tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

// D(tmem) (+)= A(tmem: lane = row, column j = bf16 elements 2j, 2j+1 along K) x B(smem desc)
__device__ __forceinline__ void fa_umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// per-row value combined across the two key-half warps of a lane quarter
__device__ __forceinline__ float fa_combine(float* red, int hf, int lr, float v, bool is_max) {
  red[hf * 128 + lr] = v;
  asm volatile("bar.sync 1, %0;" ::"n"(32 * FW_EPI_WARPS) : "memory");
  const float o = red[(1 - hf) * 128 + lr];
  asm volatile("bar.sync 1, %0;" ::"n"(32 * FW_EPI_WARPS) : "memory");
  return is_max ? fmaxf(v, o) : v + o;
}

struct FaShape {
  int S, d, H;
  float alpha;
};

// fw smem: Q 16 KB | K (S x 64, two 256-row boxes), then V over it (S/64 MN-major key
// blocks of 8 KB) 64 KB | barriers + row reduction scratch
constexpr uint32_t FW_KV = 16 * 1024;
constexpr uint32_t FW_BAR = 80 * 1024;
constexpr int SMEM_FWL = FW_BAR + 2048 + 1024;

}  // namespace

__global__ void __launch_bounds__(FW_THREADS, 2)
    attn_fwd_lse_kernel(const __grid_constant__ CUtensorMap m_q, const __grid_constant__ CUtensorMap m_k,
                        const __grid_constant__ CUtensorMap m_v, float* __restrict__ lse2,
                        bf16* __restrict__ o, int64_t ldo, FaShape sh) {
  constexpr uint32_t IDESC_S = idesc_bf16<256, false, false>();
  constexpr uint32_t IDESC_O = idesc_bf16<FA_DH, false, true>();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sq = smem;
  uint8_t* skv = smem + FW_KV;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + FW_BAR);
  uint64_t* bar_qk = bar + 0;  // Q + K landed
  uint64_t* bar_v = bar + 1;   // V landed
  uint64_t* bar_s = bar + 2;   // scores MMA done
  uint64_t* bar_p = bar + 3;   // E (bf16) in TMEM (8 epilogue warps)
  uint64_t* bar_o = bar + 4;   // E V MMA done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 8);
  float* red = reinterpret_cast<float*>(smem + FW_BAR + 128);

  const int S = sh.S, d = sh.d, H = sh.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mblocks = S / 128;
  const int z = static_cast<int>(blockIdx.x) / mblocks;
  const int m_blk = static_cast<int>(blockIdx.x) % mblocks;
  const int sample = z / H, head = z % H;
  const int row0 = sample * S;
  const int nkb = S / 64;
  const int nh = (S + 255) / 256;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 5; ++i) mbar_init(&bar[i], i == 3 ? FW_EPI_WARPS : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(bar_qk, 128 * 128 + nh * 256 * 128);
      tma_load_2d(sq, &m_q, bar_qk, head * FA_DH, row0 + m_blk * 128);
      for (int h = 0; h < nh; ++h) tma_load_2d(skv + h * 32768, &m_k, bar_qk, d + head * FA_DH, row0 + h * 256);
      mbar_wait(bar_s, 0);  // K consumed: V (MN-major key blocks) over it
      mbar_expect_tx(bar_v, nkb * 8192);
      for (int kb = 0; kb < nkb; ++kb) tma_load_2d(skv + kb * 8192, &m_v, bar_v, 2 * d + head * FA_DH, row0 + kb * 64);
    }
  } else {
    if (warp == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    asm volatile("bar.sync 2, %0;" ::"n"(32 + 32 * FW_EPI_WARPS) : "memory");
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp == 1) {
      if (lane == 0) {
        mbar_wait(bar_qk, 0);
        tc_fence_after();
        const uint32_t qa = smem_u32(sq), ka = smem_u32(skv);
#pragma unroll
        for (int k = 0; k < FA_DH / 16; ++k)
          for (int h = 0; h < nh; ++h)
            umma_bf16(tmem + h * 256, sdesc_sw128(qa + k * 32, 16, 1024),
                      sdesc_sw128(ka + h * 32768 + k * 32, 16, 1024), IDESC_S, k != 0);
        umma_commit(bar_s);
        mbar_wait(bar_p, 0);
        mbar_wait(bar_v, 0);
        tc_fence_after();
        const uint32_t va = smem_u32(skv);
        for (int kb = 0; kb < nkb; ++kb)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int key = kb * 64 + k * 16;
            const uint32_t acol = (key >> 8) * 256 + ((key & 255) >> 1);
            fa_umma_ts(tmem + 448, tmem + acol, sdesc_sw128(va + kb * 8192 + k * 2048, 8192, 1024), IDESC_O,
                       (kb | k) != 0);
          }
        umma_commit(bar_o);
      }
    } else {
      // epilogue: warp (q, hf) owns TMEM lanes [32q, 32q+32) (query rows) and key half hf
      const int q = warp & 3, hf = (warp - 2) / 4;
      const int lr = q * 32 + lane;
      const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
      const int c_lo = hf * 8, c_hi = min(S / 32, hf * 8 + 8);
      mbar_wait(bar_s, 0);
      tc_fence_after();
      float mx = -INFINITY;
      for (int c = c_lo; c < c_hi; ++c) {
        uint32_t v[32];
        tmem_ld32(trow + c * 32, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) mx = fmaxf(mx, __uint_as_float(v[j]));
      }
      mx = fa_combine(red, hf, lr, mx, true);
      const float sl2 = sh.alpha * 1.4426950408889634f;
      const float mb = mx * sl2;
      float sum = 0.f;
      for (int c = c_lo; c < c_hi; ++c) {
        uint32_t v[32];
        tmem_ld32(trow + c * 32, v);
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float e0 = exp2f(fmaf(__uint_as_float(v[2 * j]), sl2, -mb));
          const float e1 = exp2f(fmaf(__uint_as_float(v[2 * j + 1]), sl2, -mb));
          sum += e0 + e1;
          pk[j] = fa_pack(e0, e1);
        }
        // unnormalised bf16 E over consumed score columns of this half (chunk c -> columns
        // of chunk <= c): key k of half (k >> 8) at column (k >> 8) * 256 + (k & 255) / 2
        fa_tmem_st16(trow + (c >> 3) * 256 + (c & 7) * 16, pk);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      sum = fa_combine(red, hf, lr, sum, false);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) fa_mbar_arrive(bar_p);
      const int64_t grow = static_cast<int64_t>(row0) + m_blk * 128 + lr;
      if (hf == 0) lse2[static_cast<int64_t>(z) * S + m_blk * 128 + lr] = mb + __log2f(sum);
      const float inv = 1.f / sum;
      mbar_wait(bar_o, 0);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld32(trow + 448 + hf * 32, v);
      bf16* dst = o + grow * ldo + head * FA_DH + hf * 32;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 pk;
        pk.x = fa_pack(__uint_as_float(v[8 * i + 0]) * inv, __uint_as_float(v[8 * i + 1]) * inv);
        pk.y = fa_pack(__uint_as_float(v[8 * i + 2]) * inv, __uint_as_float(v[8 * i + 3]) * inv);
        pk.z = fa_pack(__uint_as_float(v[8 * i + 4]) * inv, __uint_as_float(v[8 * i + 5]) * inv);
        pk.w = fa_pack(__uint_as_float(v[8 * i + 6]) * inv, __uint_as_float(v[8 * i + 7]) * inv);
        *reinterpret_cast<uint4*>(dst + 8 * i) = pk;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(*tmem_slot) : "memory");
  }
}

// D[z, s] = sum_c dO[row, head*64 + c] * O[row, head*64 + c]: one warp per (row, head),
// 4 bytes per lane of each operand.
__global__ void __launch_bounds__(256) attn_bwd_prep_kernel(float* __restrict__ dvec, const bf16* __restrict__ o,
                                                            int64_t ldo, const bf16* __restrict__ dout, int64_t lddo,
                                                            int64_t T, int S, int H) {
  const int64_t w = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= T * H) return;
  const int64_t row = w / H;
  const int head = static_cast<int>(w % H);
  const float2 a = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(o + row * ldo + head * FA_DH)[lane]);
  const float2 b = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(dout + row * lddo + head * FA_DH)[lane]);
  float v = fmaf(a.x, b.x, a.y * b.y);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if (lane == 0) {
    const int64_t sample = row / S;
    dvec[(sample * H + head) * S + row % S] = v;
  }
}


// ---------------------------------------------------------------------------------------
// Backward, key-block major (see the file comment).  Warps: 0 TMA, 1 MMA (+ TMEM alloc),
// 2..9 softmax-gradient warps (lane quarter q = warp % 4 = 32 keys, query half hf),
// 10..13 dQ warps (lane quarter = 32 queries of the partial dQ).
namespace {
constexpr int BW_SM_WARPS = 8;
constexpr int BW_DQ_WARPS = 4;
constexpr int BW_THREADS = 64 + 32 * (BW_SM_WARPS + BW_DQ_WARPS);
constexpr uint32_t BW_K = 0, BW_V = 16384;
constexpr uint32_t BW_Q = 32768;      // [2] x 16 KB
constexpr uint32_t BW_DO = 65536;     // [2] x 16 KB
constexpr uint32_t BW_ADS = 98304;    // dS as the MN-major A of dQ = dS K: 2 chunks x 16 KB
constexpr uint32_t BW_DQP = 131072;   // [2] partial dQ, 128 rows x DQ_LD fp32
constexpr int DQ_LD = 68;             // floats per partial row (16-byte stores conflict-free)
constexpr uint32_t DQP_BYTES = 128 * DQ_LD * 4;
constexpr uint32_t BW_VEC = BW_DQP + 2 * DQP_BYTES;   // [2] x (lse2[128] | D[128])
constexpr uint32_t BW_BAR = BW_VEC + 2 * 1024;
constexpr int SMEM_BWKV = BW_BAR + 256 + 1024;
// TMEM columns
constexpr uint32_t T_ST = 0, T_DPT = 128, T_DV = 256, T_DK = 320, T_DQ = 384;  // T_DQ: [2] x 64

__device__ __forceinline__ void fa_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ float4 fa_ld_cluster_f4(uint32_t cluster_addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(cluster_addr)
               : "memory");
  return v;
}
}  // namespace

__global__ void __launch_bounds__(BW_THREADS, 1)
    attn_bwd_kv_kernel(const __grid_constant__ CUtensorMap m_qkv, const __grid_constant__ CUtensorMap m_do,
                       const float* __restrict__ lse2, const float* __restrict__ dvec, bf16* __restrict__ dqkv,
                       int64_t ld_dqkv, FaShape sh) {
  constexpr uint32_t IDESC_ST = idesc_bf16<128, false, false>();   // S^T, dP^T: K-major A and B
  constexpr uint32_t IDESC_DVK = idesc_bf16<FA_DH, false, true>(); // A = TMEM, B = MN-major tile
  constexpr uint32_t IDESC_DQ = idesc_bf16<FA_DH, true, true>();   // A = dS (MN-major smem)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + BW_BAR);
  uint64_t* bar_kv = bar + 0;
  uint64_t* bar_qfull = bar + 1;   // [2]
  uint64_t* bar_qfree = bar + 3;   // [2]
  uint64_t* bar_s = bar + 5;       // S^T, dP^T in TMEM
  uint64_t* bar_p = bar + 6;       // P, dS in TMEM + dS in smem (8 softmax warps)
  uint64_t* bar_mma2 = bar + 7;    // dV, dK, dQ MMAs of the query block done
  uint64_t* bar_dqfree = bar + 8;  // dQ warps have read the dQ accumulator (4 warps)
  uint64_t* bar_dqfull = bar + 9;  // [2] owner: every CTA's partial of the block is in place
  uint64_t* bar_dqempty = bar + 11;  // [2] this CTA's partial buffer may be overwritten
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);

  const int S = sh.S, d = sh.d, H = sh.H;
  const int nq = S / 128;  // query blocks = key blocks = cluster size
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = static_cast<int>(blockIdx.x) % nq;  // == %cluster_ctarank
  const int z = static_cast<int>(blockIdx.x) / nq;
  const int sample = z / H, head = z % H;
  const int row0 = sample * S;
  const float sl2 = sh.alpha * 1.4426950408889634f;

  if (warp == 0 && lane == 0) {
    mbar_init(bar_kv, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_qfull[i], 1);
      mbar_init(&bar_qfree[i], 1);
      mbar_init(&bar_dqfull[i], nq);
      mbar_init(&bar_dqempty[i], 1);
    }
    mbar_init(bar_s, 1);
    mbar_init(bar_p, BW_SM_WARPS);
    mbar_init(bar_mma2, 1);
    mbar_init(bar_dqfree, BW_DQ_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();  // barriers of every CTA initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // K, V of this key block once; Q, dO per query block through a 2-stage ring
      mbar_expect_tx(bar_kv, 2 * 16384);
      tma_load_2d(smem + BW_K, &m_qkv, bar_kv, d + head * FA_DH, row0 + kb * 128);
      tma_load_2d(smem + BW_V, &m_qkv, bar_kv, 2 * d + head * FA_DH, row0 + kb * 128);
      for (int qb = 0; qb < nq; ++qb) {
        const int st = qb & 1;
        mbar_wait(&bar_qfree[st], ((qb >> 1) & 1) ^ 1);
        mbar_expect_tx(&bar_qfull[st], 2 * 16384);
        tma_load_2d(smem + BW_Q + st * 16384, &m_qkv, &bar_qfull[st], head * FA_DH, row0 + qb * 128);
        tma_load_2d(smem + BW_DO + st * 16384, &m_do, &bar_qfull[st], head * FA_DH, row0 + qb * 128);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t ka = smem_u32(smem + BW_K), va = smem_u32(smem + BW_V), dsa = smem_u32(smem + BW_ADS);
      mbar_wait(bar_kv, 0);
      for (int qb = 0; qb < nq; ++qb) {
        const int st = qb & 1;
        const uint32_t qa = smem_u32(smem + BW_Q + st * 16384), da = smem_u32(smem + BW_DO + st * 16384);
        mbar_wait(&bar_qfull[st], (qb >> 1) & 1);
        tc_fence_after();
        // S^T = K Q^T and dP^T = V dO^T (lane = key, column = query)
#pragma unroll
        for (int k = 0; k < FA_DH / 16; ++k) {
          umma_bf16(tmem + T_ST, sdesc_sw128(ka + k * 32, 16, 1024), sdesc_sw128(qa + k * 32, 16, 1024), IDESC_ST, k != 0);
          umma_bf16(tmem + T_DPT, sdesc_sw128(va + k * 32, 16, 1024), sdesc_sw128(da + k * 32, 16, 1024), IDESC_ST, k != 0);
        }
        umma_commit(bar_s);
        mbar_wait(bar_p, qb & 1);  // P^T, dS^T (bf16) in TMEM, dS in smem
        if (qb > 0) mbar_wait(bar_dqfree, (qb - 1) & 1);  // dQ accumulator of qb-1 read out
        tc_fence_after();
        const uint32_t dq = tmem + T_DQ + (qb & 1) * 64;
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // K = 128 queries (dV, dK) / 128 keys (dQ), 16 per MMA
          const uint32_t acol = (k >> 2) * 64 + (k & 3) * 8;  // packed pairs of query half k/4
          const uint32_t acc = (qb | k) != 0;
          fa_umma_ts(tmem + T_DV, tmem + T_ST + acol, sdesc_sw128(da + k * 2048, 8192, 1024), IDESC_DVK, acc);
          fa_umma_ts(tmem + T_DK, tmem + T_DPT + acol, sdesc_sw128(qa + k * 2048, 8192, 1024), IDESC_DVK, acc);
          umma_bf16(dq, sdesc_sw128(dsa + k * 2048, 16384, 1024), sdesc_sw128(ka + k * 2048, 8192, 1024), IDESC_DQ,
                    k != 0);
        }
        umma_commit(bar_mma2);
        umma_commit(&bar_qfree[st]);
      }
    }
  } else if (warp < 2 + BW_SM_WARPS) {
    // ---- softmax-gradient warps: key row lr (TMEM lane), queries [hf*64, hf*64 + 64) ----
    const int q = warp & 3, hf = (warp - 2) / 4;
    const int lr = q * 32 + lane;
    const int tid = threadIdx.x - 64;  // 0..255
    const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
    uint8_t* ads = smem + BW_ADS + hf * 16384 + lr * 128;
    for (int qb = 0; qb < nq; ++qb) {
      float* vec = reinterpret_cast<float*>(smem + BW_VEC + (qb & 1) * 1024);  // lse2[128] | D[128]
      {
        const int64_t base = static_cast<int64_t>(z) * S + qb * 128;
        vec[tid] = tid < 128 ? __ldg(lse2 + base + tid) : __ldg(dvec + base + tid - 128);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * BW_SM_WARPS) : "memory");
      mbar_wait(bar_s, qb & 1);
      if (qb > 0) mbar_wait(bar_mma2, (qb - 1) & 1);  // dQ MMA of qb-1 done reading smem dS
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int q0 = hf * 64 + c * 32;  // first query of this 32-column chunk
        uint32_t sv[32], pv[32];
        tmem_ld32(trow + T_ST + q0, sv);
        tmem_ld32(trow + T_DPT + q0, pv);
        uint32_t pk[16], dk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const float2 ls = *reinterpret_cast<const float2*>(vec + q0 + 2 * j);
          const float2 dd = *reinterpret_cast<const float2*>(vec + 128 + q0 + 2 * j);
          const float p0 = exp2f(fmaf(__uint_as_float(sv[2 * j]), sl2, -ls.x));
          const float p1 = exp2f(fmaf(__uint_as_float(sv[2 * j + 1]), sl2, -ls.y));
          const float g0 = sh.alpha * p0 * (__uint_as_float(pv[2 * j]) - dd.x);
          const float g1 = sh.alpha * p1 * (__uint_as_float(pv[2 * j + 1]) - dd.y);
          pk[j] = fa_pack(p0, p1);
          dk[j] = fa_pack(g0, g1);
        }
        // packed bf16 pairs over this chunk's own (consumed) columns: query pair j of the
        // chunk at column hf*64 + c*16 + j -- the MMA reads A column (k>>2)*64 + (k&3)*8
        fa_tmem_st16(trow + T_ST + hf * 64 + c * 16, pk);
        fa_tmem_st16(trow + T_DPT + hf * 64 + c * 16, dk);
        // dS^T row lr -> MN-major A of dQ: query chunk hf (64 queries), 16-byte units c*4..c*4+3
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int u = c * 4 + i;
          *reinterpret_cast<uint4*>(ads + ((u ^ (lr & 7)) << 4)) = make_uint4(dk[4 * i], dk[4 * i + 1], dk[4 * i + 2], dk[4 * i + 3]);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) fa_mbar_arrive(bar_p);
    }
    // dV (hf = 0) / dK (hf = 1) of key row lr: accumulated over every query block
    mbar_wait(bar_mma2, (nq - 1) & 1);
    tc_fence_after();
    const int64_t krow = static_cast<int64_t>(row0) + kb * 128 + lr;
    bf16* dst = dqkv + krow * ld_dqkv + (hf == 0 ? 2 * d : d) + head * FA_DH;
    const uint32_t src = trow + (hf == 0 ? T_DV : T_DK);
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      uint32_t v[32];
      tmem_ld32(src + h2 * 32, v);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 pkd;
        pkd.x = fa_pack(__uint_as_float(v[8 * i + 0]), __uint_as_float(v[8 * i + 1]));
        pkd.y = fa_pack(__uint_as_float(v[8 * i + 2]), __uint_as_float(v[8 * i + 3]));
        pkd.z = fa_pack(__uint_as_float(v[8 * i + 4]), __uint_as_float(v[8 * i + 5]));
        pkd.w = fa_pack(__uint_as_float(v[8 * i + 6]), __uint_as_float(v[8 * i + 7]));
        *reinterpret_cast<uint4*>(dst + h2 * 32 + 8 * i) = pkd;
      }
    }
  } else {
    // ---- dQ warps: partial dQ of query block qb (row = query r = 32q + lane) -> smem;
    // the owner CTA (rank qb) sums every rank's partial in rank order -> dqkv ----
    const int q = warp & 3;
    const int r = q * 32 + lane;
    const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
    for (int qb = 0; qb < nq; ++qb) {
      const int b = qb & 1;
      float* part = reinterpret_cast<float*>(smem + BW_DQP + b * DQP_BYTES) + r * DQ_LD;
      if (qb >= 2) mbar_wait(&bar_dqempty[b], ((qb >> 1) - 1) & 1);  // owner of qb-2 done reading
      mbar_wait(bar_mma2, qb & 1);
      tc_fence_after();
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        uint32_t v[32];
        tmem_ld32(trow + T_DQ + b * 64 + h2 * 32, v);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          *reinterpret_cast<float4*>(part + h2 * 32 + 4 * i) =
              make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]), __uint_as_float(v[4 * i + 2]),
                          __uint_as_float(v[4 * i + 3]));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) fa_mbar_arrive(bar_dqfree);
      asm volatile("bar.sync 3, %0;" ::"n"(32 * BW_DQ_WARPS) : "memory");
      if (threadIdx.x == 64 + 32 * BW_SM_WARPS) {  // one arrival per CTA on the owner's barrier
        fa_arrive_remote(mapa_shared(smem_u32(&bar_dqfull[b]), static_cast<uint32_t>(qb)));
      }
      if (qb == kb) {  // this CTA owns query block qb
        mbar_wait_cluster(&bar_dqfull[b], 0);  // a CTA owns one query block: one phase
        const uint32_t part_local = smem_u32(smem + BW_DQP + b * DQP_BYTES) + r * DQ_LD * 4;
        float acc[64];
#pragma unroll
        for (int i = 0; i < 64; ++i) acc[i] = 0.f;
        for (int rk = 0; rk < nq; ++rk) {  // fixed rank order: deterministic
          const uint32_t src = mapa_shared(part_local, static_cast<uint32_t>(rk));
          float4 v[16];  // all 16 remote loads in flight before the first add
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = fa_ld_cluster_f4(src + 16 * i);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            acc[4 * i] += v[i].x;
            acc[4 * i + 1] += v[i].y;
            acc[4 * i + 2] += v[i].z;
            acc[4 * i + 3] += v[i].w;
          }
        }
        bf16* dst = dqkv + (static_cast<int64_t>(row0) + qb * 128 + r) * ld_dqkv + head * FA_DH;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          uint4 pkd;
          pkd.x = fa_pack(acc[8 * i + 0], acc[8 * i + 1]);
          pkd.y = fa_pack(acc[8 * i + 2], acc[8 * i + 3]);
          pkd.z = fa_pack(acc[8 * i + 4], acc[8 * i + 5]);
          pkd.w = fa_pack(acc[8 * i + 6], acc[8 * i + 7]);
          *reinterpret_cast<uint4*>(dst + 8 * i) = pkd;
        }
        asm volatile("bar.sync 3, %0;" ::"n"(32 * BW_DQ_WARPS) : "memory");  // all rows read
        if (threadIdx.x == 64 + 32 * BW_SM_WARPS) {
          for (int rk = 0; rk < nq; ++rk)  // every rank may now overwrite its buffer b
            fa_arrive_remote(mapa_shared(smem_u32(&bar_dqempty[b]), static_cast<uint32_t>(rk)));
        }
      }
    }
  }
  tc_fence_before();
  cluster_sync();  // no CTA leaves while a peer may still read its partial dQ
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

}  // namespace tc

namespace {
int flash_checks(const void* qkv, int64_t m, int64_t S, int64_t d, int64_t H) {
  GPP_ARG_CHECK(qkv != nullptr, "null qkv");
  GPP_ARG_CHECK(m >= 1 && H >= 1 && d == H * 64, "flash attention needs head dim 64 (d == 64 H)");
  GPP_ARG_CHECK(S >= 128 && S <= 512 && S % 128 == 0, "flash attention needs S in {128, 256, 384, 512}");
  GPP_ARG_CHECK((reinterpret_cast<uintptr_t>(qkv) & 15) == 0, "16-byte aligned qkv");
  return GPP_OK;
}
}  // namespace

}  // namespace gpp

using namespace gpp;

extern "C" {

int gpp_flash_attn_fwd(const void* qkv, float* lse2, void* o, int64_t ldo, int64_t m, int64_t S, int64_t d,
                       int64_t H, float scale, void* stream) {
  int rc = flash_checks(qkv, m, S, d, H);
  if (rc) return rc;
  GPP_ARG_CHECK(lse2 && o && ldo % 8 == 0 && (reinterpret_cast<uintptr_t>(o) & 15) == 0, "16-byte aligned o");
  GPP_ARG_CHECK(scale > 0.f, "softmax scale must be positive");
  const int64_t T = m * S, Z = m * H;
  CUtensorMap mq, mk, mv;
  if ((rc = tc::make_map_bf16(&mq, qkv, 3 * d, T, 3 * d, 64, 128))) return rc;
  if ((rc = tc::make_map_bf16(&mk, qkv, 3 * d, T, 3 * d, 64, 256))) return rc;
  if ((rc = tc::make_map_bf16(&mv, qkv, 3 * d, T, 3 * d, 64, 64))) return rc;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc::attn_fwd_lse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM_FWL);
    attr = true;
  }
  tc::FaShape sh{static_cast<int>(S), static_cast<int>(d), static_cast<int>(H), scale};
  tc::attn_fwd_lse_kernel<<<static_cast<unsigned>(Z * (S / 128)), tc::FW_THREADS, tc::SMEM_FWL,
                            static_cast<cudaStream_t>(stream)>>>(mq, mk, mv, lse2, static_cast<bf16*>(o), ldo, sh);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_flash_attn_bwd(const void* qkv, const float* lse2, const void* o, int64_t ldo, const void* dout,
                       int64_t lddo, float* dvec, void* dqkv, int64_t m, int64_t S, int64_t d, int64_t H,
                       float scale, void* stream) {
  int rc = flash_checks(qkv, m, S, d, H);
  if (rc) return rc;
  GPP_ARG_CHECK(lse2 && o && dout && dvec && dqkv, "null pointer");
  GPP_ARG_CHECK(ldo % 8 == 0 && lddo % 8 == 0 && (reinterpret_cast<uintptr_t>(dqkv) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(dout) & 15) == 0, "16-byte alignment");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t T = m * S, Z = m * H;
  tc::attn_bwd_prep_kernel<<<static_cast<unsigned>((T * H + 7) / 8), 256, 0, s>>>(
      dvec, static_cast<const bf16*>(o), ldo, static_cast<const bf16*>(dout), lddo, T, static_cast<int>(S),
      static_cast<int>(H));
  GPP_LAUNCH_CHECK();
  CUtensorMap mqkv, mdo;
  if ((rc = tc::make_map_bf16(&mqkv, qkv, 3 * d, T, 3 * d, 64, 128))) return rc;
  if ((rc = tc::make_map_bf16(&mdo, dout, d, T, lddo, 64, 128))) return rc;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc::attn_bwd_kv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM_BWKV);
    cudaFuncSetAttribute(tc::attn_bwd_kv_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  tc::FaShape sh{static_cast<int>(S), static_cast<int>(d), static_cast<int>(H), scale};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(Z * (S / 128)));
  cfg.blockDim = dim3(tc::BW_THREADS);
  cfg.dynamicSmemBytes = tc::SMEM_BWKV;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = static_cast<unsigned>(S / 128);  // the key blocks of one (sample, head)
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, tc::attn_bwd_kv_kernel, mqkv, mdo, lse2, static_cast<const float*>(dvec),
                                     static_cast<bf16*>(dqkv), 3 * d, sh);
  if (e != cudaSuccess) {
    set_error(std::string("attn_bwd_kv launch: ") + cudaGetErrorString(e));
    return GPP_ERR_CUDA;
  }
  count_launch();
  return GPP_OK;
}

}  // extern "C"
