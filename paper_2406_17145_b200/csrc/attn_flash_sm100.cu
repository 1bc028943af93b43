// Recompute-based MMT attention for sm_100a (S <= 512 keys, head dim 64).
// Nothing of size Z x S x S ever reaches HBM:
//
//   attn_fwd_lse_kernel : one CTA per (z = sample x head, 128 query rows).  S = Q K^T fills
//       TMEM (128 lanes x S fp32 columns); pass 1 takes the row max, pass 2 writes
//       e = exp2(alpha log2e (s - max)) as bf16 pairs over the consumed score columns and
//       sums them; O = E V (A operand straight from TMEM) is divided by the row sum in its
//       epilogue.  Stores O and the row's log-sum-exp in base 2:
//           lse2 = alpha log2e max + log2(sum),   P = exp2(alpha log2e s - lse2).
//   attn_bwd_prep_kernel: D[q] = alpha rowsum(dO o O) per (z, query) -- the FlashAttention
//       identity rowsum(P o dP) = rowsum(dO o O).
//   attn_bwd_kernel     : ONE persistent launch, two CTA roles (one CTA of each per SM).
//       dK/dV role, items (z, 128-key block), looping over 32-query blocks: S^T = K Q^T and
//       dP^T = V dO^T in TMEM (lane = key); the softmax warps recompute
//       P^T = exp2(alpha log2e s - lse2[q]) and dS^T = P^T o (alpha dP^T - D[q]) and write
//       both as bf16 pairs back over the consumed columns -- the TMEM A operands of
//       dV += P^T dO and dK += dS^T Q, accumulated in TMEM over every query block.
//       dQ role, items (z, 128-query block), looping over 32-key blocks: S, dP recomputed
//       (lane = query, lse2 / D row constants), dS in place, dQ += dS K.
//       S / dP TMEM tiles in two (dK/dV) / three (dQ) buffers turned by two ping-pong groups
//       of softmax warps, the 32 KB first tiles double-buffered across items, 256 TMEM
//       columns per CTA.
//       (A single kernel reducing per-key-block dQ partials across a 4-CTA cluster through
//       DSMEM measured 363 us vs 149 us without the exchange -- the owner-CTA reductions
//       serialised the cluster; recomputing S and dP in the dQ role costs less.)
//
// Layout: packed QKV [m S, 3d] (Q | K | V, head h at columns h*64), o / dout [m S, d]
// head-interleaved, lse2 / D [Z, S] fp32 with z = sample * H + head.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#define GPP_PDL_CLASS 2  // programmatic-dependent-launch family: flash attention
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

// 2^x on the SFU without exp2f's denormal range fix-up (results below 2^-126 flush to 0;
// softmax terms that small are far below bf16 resolution of the row sum).
__device__ __forceinline__ float fa_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
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
  pdl_wait();  // qkv is the previous kernel's output
  pdl_trigger();

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
          const float e0 = fa_ex2(fmaf(__uint_as_float(v[2 * j]), sl2, -mb));
          const float e1 = fa_ex2(fmaf(__uint_as_float(v[2 * j + 1]), sl2, -mb));
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

// Streamed forward (default): 256 TMEM columns and ~83 KB of shared memory per CTA, so TWO
// CTAs run per SM and one's softmax overlaps the other's MMAs (the kernel above holds the
// whole 128 x S score block in 512 columns: one CTA computes per SM at a time).  K / V
// arrive as 64-key tiles through a 4-slot TMA ring.  Pass 1: S_j = Q K_j^T per 64-key block
// (double-buffered in TMEM) -> row max.  Pass 2: S_j recomputed, e = exp2(alpha log2e (s -
// max)) packed bf16 over the consumed columns (the TMEM A operand), O += E_j V_j; the row
// sum, O / sum and the base-2 LSE at the end.  Warps: 0 TMA, 1 MMA, 2..9 two per TMEM lane
// quarter, each taking 32 of a block's 64 keys.
namespace {
constexpr int F2_SLOTS = 4;
constexpr uint32_t F2_TILE = 64 * 128;            // 64 keys x 64 dims bf16, 128B-swizzled: 8 KB
constexpr uint32_t F2_RING = 16 * 1024;           // after Q (16 KB)
constexpr uint32_t F2_BAR = F2_RING + F2_SLOTS * F2_TILE;
constexpr int SMEM_FW2 = F2_BAR + 2048 + 1024;
constexpr uint32_t F2_O = 128;                     // O accumulator columns [128, 192)
}  // namespace

__global__ void __launch_bounds__(FW_THREADS, 2)
    attn_fwd_stream_kernel(const __grid_constant__ CUtensorMap m_q, const __grid_constant__ CUtensorMap m_kv,
                           float* __restrict__ lse2, bf16* __restrict__ o, int64_t ldo, FaShape sh) {
  constexpr uint32_t IDESC_S = idesc_bf16<64, false, false>();
  constexpr uint32_t IDESC_O = idesc_bf16<FA_DH, false, true>();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sq = smem;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + F2_BAR);
  uint64_t* b_q = bar + 0;                  // Q landed
  uint64_t* b_full = bar + 1;               // [F2_SLOTS]
  uint64_t* b_empty = b_full + F2_SLOTS;    // [F2_SLOTS]
  uint64_t* b_s = b_empty + F2_SLOTS;       // [2] S of TMEM buffer b complete
  uint64_t* b_c = b_s + 2;                  // [2] softmax warps done with buffer b (max read / E written)
  uint64_t* b_o = b_c + 2;                  // all E V MMAs complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(b_o + 1);
  float* red = reinterpret_cast<float*>(smem + F2_BAR + 128);

  const int S = sh.S, d = sh.d, H = sh.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mblocks = S / 128;
  const int z = static_cast<int>(blockIdx.x) / mblocks;
  const int m_blk = static_cast<int>(blockIdx.x) % mblocks;
  const int sample = z / H, head = z % H;
  const int row0 = sample * S;
  const int nb = S / 64;  // 64-key blocks
  const int ntiles = 3 * nb;  // pass 1: K_0..K_{nb-1}; pass 2: K_0, V_0, K_1, V_1, ...

  if (warp == 0 && lane == 0) {
    mbar_init(b_q, 1);
    for (int i = 0; i < F2_SLOTS; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&b_s[i], 1);
      mbar_init(&b_c[i], FW_EPI_WARPS);
    }
    mbar_init(b_o, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // qkv is the previous kernel's output
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(b_q, 128 * 128);
      tma_load_2d(sq, &m_q, b_q, head * FA_DH, row0 + m_blk * 128);
      for (int t = 0; t < ntiles; ++t) {
        const int sl = t % F2_SLOTS;
        mbar_wait(&b_empty[sl], ((t / F2_SLOTS) & 1) ^ 1);
        const int u = t - nb;  // pass-2 index
        const int key_blk = t < nb ? t : u >> 1;
        const int col = (t >= nb && (u & 1)) ? 2 * d : d;  // V or K columns of the head
        mbar_expect_tx(&b_full[sl], F2_TILE);
        tma_load_2d(smem + F2_RING + sl * F2_TILE, &m_kv, &b_full[sl], col + head * FA_DH, row0 + key_blk * 64);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      mbar_wait(b_q, 0);
      const uint32_t qa = smem_u32(sq);
      // S of block g (g < nb: pass 1 block g; else pass 2 block g - nb) from ring tile t
      auto issue_s = [&](int g, int t) {
        const int b = g & 1, sl = t % F2_SLOTS;
        if (g >= 2) mbar_wait(&b_c[b], ((g - 2) >> 1) & 1);  // softmax warps done with the buffer
        mbar_wait(&b_full[sl], (t / F2_SLOTS) & 1);
        tc_fence_after();
        const uint32_t ka = smem_u32(smem + F2_RING + sl * F2_TILE);
#pragma unroll
        for (int k = 0; k < FA_DH / 16; ++k)
          umma_bf16(tmem + b * 64, sdesc_sw128(qa + k * 32, 16, 1024), sdesc_sw128(ka + k * 32, 16, 1024), IDESC_S,
                    k != 0);
        umma_commit(&b_s[b]);
        umma_commit(&b_empty[sl]);
      };
      for (int g = 0; g < nb; ++g) issue_s(g, g);  // pass 1
      // pass 2: S of block j + 1 is issued before E_j V_j
      issue_s(nb, nb);
      for (int j = 0; j < nb; ++j) {
        const int g = nb + j;
        if (j + 1 < nb) issue_s(g + 1, nb + 2 * (j + 1));
        const int b = g & 1, tv = nb + 2 * j + 1, sl = tv % F2_SLOTS;
        mbar_wait(&b_c[b], (g >> 1) & 1);  // E_j in TMEM
        mbar_wait(&b_full[sl], (tv / F2_SLOTS) & 1);
        tc_fence_after();
        const uint32_t va = smem_u32(smem + F2_RING + sl * F2_TILE);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {  // keys 16 kk..: packed E of warp half kk / 2 at b*64 + hf*32 + (kk&1)*8
          const uint32_t acol = b * 64 + (kk >> 1) * 32 + (kk & 1) * 8;
          fa_umma_ts(tmem + F2_O, tmem + acol, sdesc_sw128(va + kk * 2048, 8192, 1024), IDESC_O, (j | kk) != 0);
        }
        umma_commit(&b_empty[sl]);
      }
      umma_commit(b_o);
    }
  } else {
    const int q = warp & 3, hf = (warp - 2) / 4;
    const int lr = q * 32 + lane;
    const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
    float mx = -INFINITY;
    for (int g = 0; g < nb; ++g) {
      const int b = g & 1;
      mbar_wait(&b_s[b], (g >> 1) & 1);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld32(trow + b * 64 + hf * 32, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) mx = fmaxf(mx, __uint_as_float(v[i]));
      tc_fence_before();
      __syncwarp();
      if (lane == 0) fa_mbar_arrive(&b_c[b]);
    }
    mx = fa_combine(red, hf, lr, mx, true);
    const float sl2 = sh.alpha * 1.4426950408889634f;
    const float mb = mx * sl2;
    float sum = 0.f;
    for (int j = 0; j < nb; ++j) {
      const int g = nb + j, b = g & 1;
      mbar_wait(&b_s[b], (g >> 1) & 1);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld32(trow + b * 64 + hf * 32, v);
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float e0 = fa_ex2(fmaf(__uint_as_float(v[2 * i]), sl2, -mb));
        const float e1 = fa_ex2(fmaf(__uint_as_float(v[2 * i + 1]), sl2, -mb));
        sum += e0 + e1;
        pk[i] = fa_pack(e0, e1);
      }
      fa_tmem_st16(trow + b * 64 + hf * 32, pk);  // over this warp's consumed columns
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) fa_mbar_arrive(&b_c[b]);
    }
    sum = fa_combine(red, hf, lr, sum, false);
    const int64_t grow = static_cast<int64_t>(row0) + m_blk * 128 + lr;
    if (hf == 0) lse2[static_cast<int64_t>(z) * S + m_blk * 128 + lr] = mb + __log2f(sum);
    const float inv = 1.f / sum;
    mbar_wait(b_o, 0);
    tc_fence_after();
    uint32_t v[32];
    tmem_ld32(trow + F2_O + hf * 32, v);
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
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}

// Online forward (one pass over the keys): the eight softmax warps form two ping-pong groups
// of one warp per TMEM lane quarter; group g owns 64-key blocks j = g, g + 2, ... of every
// row, keeps its own running max / sum per row in registers and its own O accumulator in TMEM
// (O_g += E_j V_j), and rescales O_g only when a block raises its row max by more than 2^8
// (waiting for its previous E V MMA first).  The two groups' (max, sum, O) are merged once at
// the end.  TMEM: S buffers [0, 64) / [64, 128) (group 0 / 1), O_0 [128, 192), O_1 [192, 256).
namespace {
constexpr float F3_SLACK = 8.f;  // log2 units a row max may grow before O is rescaled
}  // namespace

__global__ void __launch_bounds__(FW_THREADS, 2)
    attn_fwd_online_kernel(const __grid_constant__ CUtensorMap m_q, const __grid_constant__ CUtensorMap m_kv,
                           float* __restrict__ lse2, bf16* __restrict__ o, int64_t ldo, FaShape sh) {
  constexpr uint32_t IDESC_S = idesc_bf16<64, false, false>();
  constexpr uint32_t IDESC_O = idesc_bf16<FA_DH, false, true>();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sq = smem;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + F2_BAR);
  uint64_t* b_q = bar + 0;                  // Q landed
  uint64_t* b_full = bar + 1;               // [F2_SLOTS]
  uint64_t* b_empty = b_full + F2_SLOTS;    // [F2_SLOTS]
  uint64_t* b_s = b_empty + F2_SLOTS;       // [2] S of group g's buffer complete
  uint64_t* b_c = b_s + 2;                  // [2] group g's E written (buffer consumed)
  uint64_t* b_pv = b_c + 2;                 // [2] group g's E V MMAs complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(b_pv + 2);
  float* red = reinterpret_cast<float*>(smem + F2_BAR + 128);  // [2 groups][2][128] max, sum

  const int S = sh.S, d = sh.d, H = sh.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mblocks = S / 128;
  const int z = static_cast<int>(blockIdx.x) / mblocks;
  const int m_blk = static_cast<int>(blockIdx.x) % mblocks;
  const int sample = z / H, head = z % H;
  const int row0 = sample * S;
  const int nb = S / 64;  // 64-key blocks (even)
  const int ntiles = 2 * nb;  // K_0, V_0, K_1, V_1, ...

  if (warp == 0 && lane == 0) {
    mbar_init(b_q, 1);
    for (int i = 0; i < F2_SLOTS; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&b_s[i], 1);
      mbar_init(&b_c[i], FW_EPI_WARPS / 2);
      mbar_init(&b_pv[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // qkv is the previous kernel's output
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(b_q, 128 * 128);
      tma_load_2d(sq, &m_q, b_q, head * FA_DH, row0 + m_blk * 128);
      for (int t = 0; t < ntiles; ++t) {
        const int sl = t % F2_SLOTS;
        mbar_wait(&b_empty[sl], ((t / F2_SLOTS) & 1) ^ 1);
        const int col = (t & 1) ? 2 * d : d;  // V or K columns of the head
        mbar_expect_tx(&b_full[sl], F2_TILE);
        tma_load_2d(smem + F2_RING + sl * F2_TILE, &m_kv, &b_full[sl], col + head * FA_DH, row0 + (t >> 1) * 64);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      mbar_wait(b_q, 0);
      const uint32_t qa = smem_u32(sq);
      auto issue_s = [&](int j) {  // S_j = Q K_j^T into group (j & 1)'s buffer
        const int b = j & 1, t = 2 * j, sl = t % F2_SLOTS;
        if (j >= 2) mbar_wait(&b_c[b], ((j - 2) >> 1) & 1);  // E_{j-2} written (and its E V issued)
        mbar_wait(&b_full[sl], (t / F2_SLOTS) & 1);
        tc_fence_after();
        const uint32_t ka = smem_u32(smem + F2_RING + sl * F2_TILE);
#pragma unroll
        for (int k = 0; k < FA_DH / 16; ++k)
          umma_bf16(tmem + b * 64, sdesc_sw128(qa + k * 32, 16, 1024), sdesc_sw128(ka + k * 32, 16, 1024), IDESC_S,
                    k != 0);
        umma_commit(&b_s[b]);
        umma_commit(&b_empty[sl]);
      };
      issue_s(0);
      for (int j = 0; j < nb; ++j) {
        if (j + 1 < nb) issue_s(j + 1);
        const int b = j & 1, tv = 2 * j + 1, sl = tv % F2_SLOTS;
        mbar_wait(&b_c[b], (j >> 1) & 1);  // E_j in TMEM (and O_b rescaled if it had to be)
        mbar_wait(&b_full[sl], (tv / F2_SLOTS) & 1);
        tc_fence_after();
        const uint32_t va = smem_u32(smem + F2_RING + sl * F2_TILE);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // keys 16 kk.. : packed E columns 8 kk.. of the buffer
          fa_umma_ts(tmem + 128 + b * 64, tmem + b * 64 + kk * 8, sdesc_sw128(va + kk * 2048, 8192, 1024), IDESC_O,
                     (j >= 2 || kk != 0) ? 1u : 0u);
        umma_commit(&b_pv[b]);
        umma_commit(&b_empty[sl]);
      }
    }
  } else {
    const int q = warp & 3, g = (warp - 2) / 4;  // lane quarter, group
    const int lr = q * 32 + lane;
    const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
    const uint32_t tb = trow + g * 64, to = trow + 128 + g * 64;
    const float sl2 = sh.alpha * 1.4426950408889634f;
    float mrun = -INFINITY;  // running row max (raw score units) of this group's blocks
    float sum = 0.f;
    int kth = 0;  // blocks of this group processed
    for (int j = g; j < nb; j += 2, ++kth) {
      mbar_wait(&b_s[g], kth & 1);
      tc_fence_after();
      float mx = mrun;
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // row max over the block's 64 columns, 32 at a time
        uint32_t v[32];
        tmem_ld32(tb + h * 32, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) mx = fmaxf(mx, __uint_as_float(v[i]));
      }
      if (kth == 0) {
        mrun = mx;
      } else if (__any_sync(0xffffffffu, (mx - mrun) * sl2 > F3_SLACK)) {
        // warp-uniform (tcgen05.ld / st are .sync.aligned): every lane moves its max up to the
        // block's and rescales its O_g row and sum; the last E V MMA of the group must be done
        mbar_wait(&b_pv[g], (kth - 1) & 1);
        tc_fence_after();
        const float f = fa_ex2((mrun - mx) * sl2);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t ov[32];
          tmem_ld32(to + h * 32, ov);
#pragma unroll
          for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(__uint_as_float(ov[i]) * f);
          fa_tmem_st16(to + h * 32, *reinterpret_cast<uint32_t(*)[16]>(&ov[0]));
          fa_tmem_st16(to + h * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(&ov[16]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        sum *= f;
        mrun = mx;
      }
      const float mb = mrun * sl2;
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // exponentials 32 columns at a time; bf16 pairs of half h -> columns 16 h..
        uint32_t v[32], pk[16];
        tmem_ld32(tb + h * 32, v);  // (half 0's pairs only overwrite half 0's consumed columns)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float e0 = fa_ex2(fmaf(__uint_as_float(v[2 * i]), sl2, -mb));
          const float e1 = fa_ex2(fmaf(__uint_as_float(v[2 * i + 1]), sl2, -mb));
          sum += e0 + e1;
          pk[i] = fa_pack(e0, e1);
        }
        fa_tmem_st16(tb + h * 16, pk);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) fa_mbar_arrive(&b_c[g]);
    }
    // merge the two groups: (max, sum) through shared memory, O from both TMEM accumulators
    red[(g * 2 + 0) * 128 + lr] = mrun;
    red[(g * 2 + 1) * 128 + lr] = sum;
    mbar_wait(&b_pv[g], (kth - 1) & 1);  // this group's last E V MMA complete
    asm volatile("bar.sync 1, %0;" ::"n"(32 * FW_EPI_WARPS) : "memory");
    tc_fence_after();
    const float m0 = red[0 * 128 + lr], s0 = red[1 * 128 + lr];
    const float m1 = red[2 * 128 + lr], s1 = red[3 * 128 + lr];
    const float mm = fmaxf(m0, m1);
    const float f0 = fa_ex2((m0 - mm) * sl2), f1 = fa_ex2((m1 - mm) * sl2);
    const float tot = s0 * f0 + s1 * f1;
    const float inv = 1.f / tot;
    const int64_t grow = static_cast<int64_t>(row0) + m_blk * 128 + lr;
    if (g == 0) lse2[static_cast<int64_t>(z) * S + m_blk * 128 + lr] = mm * sl2 + __log2f(tot);
    uint32_t a[32], bb[32];  // this group's half of the 64 output dims from both accumulators
    tmem_ld32(trow + 128 + g * 32, a);
    tmem_ld32(trow + 192 + g * 32, bb);
    bf16* dst = o + grow * ldo + head * FA_DH + g * 32;
    const float c0 = f0 * inv, c1 = f1 * inv;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float w[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) w[t] = fmaf(__uint_as_float(a[8 * i + t]), c0, __uint_as_float(bb[8 * i + t]) * c1);
      uint4 pkk;
      pkk.x = fa_pack(w[0], w[1]);
      pkk.y = fa_pack(w[2], w[3]);
      pkk.z = fa_pack(w[4], w[5]);
      pkk.w = fa_pack(w[6], w[7]);
      *reinterpret_cast<uint4*>(dst + 8 * i) = pkk;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}

// D[z, s] = alpha sum_c dO[row, head*64 + c] * O[row, head*64 + c] (pre-scaled by the softmax
// scale so that dS = P (alpha dP - D) is one FFMA + one FMUL): eight lanes per (row, head),
// one 16-byte vector of each operand per lane (every warp load is 512 contiguous bytes),
// reduced with three shuffles.
__global__ void __launch_bounds__(256) attn_bwd_prep_kernel(float* __restrict__ dvec, const bf16* __restrict__ o,
                                                            int64_t ldo, const bf16* __restrict__ dout, int64_t lddo,
                                                            int64_t T, int S, int H, float alpha) {
  pdl_wait();
  pdl_trigger();
  const int64_t t = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
  const int64_t pair = t >> 3;  // (row, head)
  const int part = static_cast<int>(t & 7);
  float acc = 0.f;
  if (pair < T * H) {
    const int64_t row = pair / H;
    const int head = static_cast<int>(pair % H);
    const uint4 va = __ldg(reinterpret_cast<const uint4*>(o + row * ldo + head * FA_DH) + part);
    const uint4 vb = __ldg(reinterpret_cast<const uint4*>(dout + row * lddo + head * FA_DH) + part);
    const uint32_t* ua = reinterpret_cast<const uint32_t*>(&va);
    const uint32_t* ub = reinterpret_cast<const uint32_t*>(&vb);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ua[k]));
      const float2 y = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ub[k]));
      acc = fmaf(x.x, y.x, fmaf(x.y, y.y, acc));
    }
  }
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  acc += __shfl_xor_sync(0xffffffffu, acc, 4);
  if (pair < T * H && part == 0) {
    const int64_t row = pair / H;
    const int head = static_cast<int>(pair % H);
    dvec[(row / S * H + head) * S + row % S] = alpha * acc;
  }
}

// ---------------------------------------------------------------------------------------
// Backward: a PERSISTENT launch of two CTA roles, one CTA of each per SM (256 TMEM columns
// each), no cross-CTA reduction.  CTAs [0, P) loop over the dK/dV items (z, 128-key block),
// CTAs [P, 2P) over the dQ items (z, 128-query block); CTA b of a role takes items b, b + P,
// ...  Warps: 0 TMA, 1 MMA (+ TMEM alloc), 2..9 eight softmax warps in two ping-pong groups
// (one warp per TMEM lane quarter each, one row per lane).  The loop dimension runs in
// blocks of BB = 32; block g's S / dP tiles live in TMEM buffer g % NBUF and are turned into
// P / dS by group g & 1, so one group's TMEM load / store latencies overlap the other's math.
// The MMA warp issues S / dP NBUF - 1 blocks ahead within an item before it waits for block
// g's P / dS and issues its accumulating MMAs (NBUF = 2 for dK/dV, whose two accumulators
// take half the columns; 3 for dQ).  The 32 KB "first" tiles (K, V or Q, dO) are
// double-buffered across items and the accumulators are handed back to the MMA warp by an
// mbarrier once read out, so per-item launch / barrier-init / TMEM-alloc / first-load
// latencies are paid once per CTA.  (Issuing ahead ACROSS item boundaries measured 150 us
// vs 124 us: the MMA warp then stalls on the next item's first tiles before it has issued
// the current item's last accumulating MMAs.)
namespace {
constexpr int BB = 32;                              // loop block (queries for dK/dV, keys for dQ)
constexpr int BW_SMW = 8;                           // softmax warps per role
constexpr int BW_ROLE_WARPS = 2 + BW_SMW;
constexpr int BW_THREADS = 32 * BW_ROLE_WARPS;      // one role per CTA: 320 threads
constexpr int BW_STAGES = 4;
constexpr uint32_t TILEB = BB * 128;     // 32 rows x 64 bf16 (128B-swizzled): 4 KB
constexpr uint32_t TILE128 = 128 * 128;  // 16 KB
constexpr uint32_t FIRST_BYTES = 2 * TILE128;  // K + V, or Q + dO

__device__ __forceinline__ void fa_bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void fa_tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void fa_tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

// 32 fp32 values -> bf16 -> 64 contiguous bytes
__device__ __forceinline__ void fa_store_row32(bf16* dst, const uint32_t (&v)[32]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint4 pk;
    pk.x = fa_pack(__uint_as_float(v[8 * i + 0]), __uint_as_float(v[8 * i + 1]));
    pk.y = fa_pack(__uint_as_float(v[8 * i + 2]), __uint_as_float(v[8 * i + 3]));
    pk.z = fa_pack(__uint_as_float(v[8 * i + 4]), __uint_as_float(v[8 * i + 5]));
    pk.w = fa_pack(__uint_as_float(v[8 * i + 6]), __uint_as_float(v[8 * i + 7]));
    *reinterpret_cast<uint4*>(dst + 8 * i) = pk;
  }
}

// smem per role (1024-aligned): first tiles [2] x 32 KB | stages [BW_STAGES] of 9 KB (two
// 32-row tiles + 2 x 128 B of per-query lse2 / D, used by the dK/dV role) | barriers
constexpr uint32_t BW_STAGE_STRIDE = 9 * 1024;
constexpr uint32_t BW_RING = 2 * FIRST_BYTES;
constexpr uint32_t BW_BAR = BW_RING + BW_STAGES * BW_STAGE_STRIDE;
constexpr uint32_t BW_ROLE_SMEM = (BW_BAR + 256 + 1023) & ~1023u;
constexpr int SMEM_BW = BW_ROLE_SMEM + 1024;

// TMEM columns (256 per CTA, two CTAs per SM).  dK/dV role: S[2] at 0 / 32, dP[2] at 64 / 96,
// dV at 128, dK at 192.  dQ role (one accumulator): S[3] at 0 / 32 / 64, dP[3] at 96 / 128 / 160,
// dQ at 192.
template <bool DQ>
struct BwTmem {
  static constexpr int NBUF = DQ ? 3 : 2;
  static constexpr uint32_t S = 0;
  static constexpr uint32_t P = S + NBUF * BB;
  static constexpr uint32_t A0 = P + NBUF * BB;  // dV (dK/dV role) or dQ
  static constexpr uint32_t A1 = A0 + FA_DH;     // dK
};
static_assert(BwTmem<false>::A1 + FA_DH == 256 && BwTmem<true>::A0 + FA_DH == 256, "TMEM plan");
}  // namespace

// DQ = false: dK, dV of items (z, 128-key block), looping over the S/32 query blocks:
//   S^T = K Q_j^T, dP^T = V dO_j^T (lane = key); P^T = exp2(alpha log2e S^T - lse2[q]),
//   dS^T = P^T o (alpha dP^T - D[q]) -> bf16 pairs in place; dV += P^T dO_j, dK += dS^T Q_j.
// DQ = true: dQ of items (z, 128-query block), looping over the S/32 key blocks:
//   S = Q K_j^T, dP = dO V_j^T (lane = query, lse2 / D row constants); dS in place;
//   dQ += dS K_j.
// smem: this role's region; w: role-local warp; qw: the CTA warp index (TMEM lane quarter).
#ifdef GPP_ATTN_TRACE
// Phase timestamps (SM clock) of the first 64 blocks of CTA 0's dK/dV role (probe builds only).
__device__ long long g_attn_trace[6 * 64];
#define ATR(ev, gb, on)                                                       \
  do {                                                                        \
    if ((on) && blockIdx.x == 0 && (gb) < 64) g_attn_trace[(ev) * 64 + (gb)] = clock64(); \
  } while (0)
#else
#define ATR(ev, gb, on) \
  do {                  \
  } while (0)
#endif

template <bool DQ>
__device__ __forceinline__ void attn_bwd_role(uint8_t* smem, uint32_t tmem, int w, int qw, int lane,
                                              const CUtensorMap& m_qkv128, const CUtensorMap& m_qkvb,
                                              const CUtensorMap& m_do128, const CUtensorMap& m_dob,
                                              const float* __restrict__ lse2, const float* __restrict__ dvec,
                                              bf16* __restrict__ dqkv, int64_t ld_dqkv, const FaShape& sh,
                                              int first_item, int item_step, int n_items) {
  using L = BwTmem<DQ>;
  constexpr int NB = L::NBUF;
  constexpr uint32_t IDESC_S = idesc_bf16<BB, false, false>();
  constexpr uint32_t IDESC_AC = idesc_bf16<FA_DH, false, true>();
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + BW_BAR);
  uint64_t* b_ffull = bar + 0;                 // [2] first tiles landed
  uint64_t* b_ffree = bar + 2;                 // [2] first tiles free (item's MMAs done)
  uint64_t* b_full = bar + 4;                  // [BW_STAGES]
  uint64_t* b_free = b_full + BW_STAGES;       // [BW_STAGES]
  uint64_t* b_s = b_free + BW_STAGES;          // [NB] S, dP of the buffer in TMEM
  uint64_t* b_p = b_s + NB;                    // [NB] bf16 P / dS of the buffer in TMEM
  uint64_t* b_done = b_p + NB;                 // the item's accumulators complete
  uint64_t* b_acc = b_done + 1;                // accumulators read out (8 warps)

  const int S = sh.S, d = sh.d, H = sh.H;
  const int per_z = S / 128, nb = S / BB;
  const float sl2 = sh.alpha * 1.4426950408889634f;
  // my items: first_item, first_item + item_step, ... < n_items
  const int my_items = first_item < n_items ? (n_items - 1 - first_item) / item_step + 1 : 0;

  if (w == 0) {
    if (lane == 0) {
      uint32_t g = 0;  // global stage counter (continues across items)
      for (int it = 0; it < my_items; ++it) {
        const int item = first_item + it * item_step;
        const int z = item / per_z, blk = item % per_z;
        const int row0 = (z / H) * S, head = z % H;
        const int fb = it & 1;
        mbar_wait(&b_ffree[fb], ((it >> 1) & 1) ^ 1);
        uint8_t* first = smem + fb * FIRST_BYTES;
        mbar_expect_tx(&b_ffull[fb], FIRST_BYTES);
        if (DQ) {
          tma_load_2d(first, &m_qkv128, &b_ffull[fb], head * FA_DH, row0 + blk * 128);
          tma_load_2d(first + TILE128, &m_do128, &b_ffull[fb], head * FA_DH, row0 + blk * 128);
        } else {
          tma_load_2d(first, &m_qkv128, &b_ffull[fb], d + head * FA_DH, row0 + blk * 128);
          tma_load_2d(first + TILE128, &m_qkv128, &b_ffull[fb], 2 * d + head * FA_DH, row0 + blk * 128);
        }
        const float* lz = lse2 + static_cast<int64_t>(z) * S;
        const float* dz = dvec + static_cast<int64_t>(z) * S;
        for (int j = 0; j < nb; ++j, ++g) {
          const int st = g % BW_STAGES;
          mbar_wait(&b_free[st], ((g / BW_STAGES) & 1) ^ 1);
          ATR(5, g, !DQ);
          uint8_t* sb = smem + BW_RING + st * BW_STAGE_STRIDE;
          if (DQ) {
            mbar_expect_tx(&b_full[st], 2 * TILEB);
            tma_load_2d(sb, &m_qkvb, &b_full[st], d + head * FA_DH, row0 + j * BB);
            tma_load_2d(sb + TILEB, &m_qkvb, &b_full[st], 2 * d + head * FA_DH, row0 + j * BB);
          } else {
            mbar_expect_tx(&b_full[st], 2 * TILEB + 2 * BB * 4);
            tma_load_2d(sb, &m_qkvb, &b_full[st], head * FA_DH, row0 + j * BB);
            tma_load_2d(sb + TILEB, &m_dob, &b_full[st], head * FA_DH, row0 + j * BB);
            fa_bulk_load(sb + 2 * TILEB, lz + j * BB, BB * 4, &b_full[st]);
            fa_bulk_load(sb + 2 * TILEB + 128, dz + j * BB, BB * 4, &b_full[st]);
          }
        }
      }
    }
  } else if (w == 1) {
    if (lane == 0) {
      uint32_t g = 0;  // global block counter: stage g % BW_STAGES, TMEM buffer g % NB
      for (int it = 0; it < my_items; ++it) {
        const int fb = it & 1;
        const uint32_t fa = smem_u32(smem + fb * FIRST_BYTES), fa2 = fa + TILE128;
        mbar_wait(&b_ffull[fb], (it >> 1) & 1);
        auto issue_sp = [&](uint32_t gg) {  // S / dP of block gg into buffer gg % NB
          const int st = gg % BW_STAGES, b = gg % NB;
          const uint32_t ta = smem_u32(smem + BW_RING + st * BW_STAGE_STRIDE), tb = ta + TILEB;
          mbar_wait(&b_full[st], (gg / BW_STAGES) & 1);
          ATR(0, gg, !DQ);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < FA_DH / 16; ++k) {
            // dK/dV: S^T = K Q_j^T, dP^T = V dO_j^T;  dQ: S = Q K_j^T, dP = dO V_j^T
            umma_bf16(tmem + L::S + b * BB, sdesc_sw128(fa + k * 32, 16, 1024), sdesc_sw128(ta + k * 32, 16, 1024),
                      IDESC_S, k != 0);
            umma_bf16(tmem + L::P + b * BB, sdesc_sw128(fa2 + k * 32, 16, 1024), sdesc_sw128(tb + k * 32, 16, 1024),
                      IDESC_S, k != 0);
          }
          umma_commit(&b_s[b]);
          ATR(1, gg, !DQ);
        };
        for (int j = 0; j + 1 < NB && j < nb; ++j) issue_sp(g + j);
        for (int j = 0; j < nb; ++j, ++g) {
          const int st = g % BW_STAGES, b = g % NB;
          // buffer (g + NB - 1) % NB last held block g - 1, whose MMAs were issued last iteration
          if (j + NB - 1 < nb) issue_sp(g + NB - 1);
          mbar_wait(&b_p[b], (g / NB) & 1);
          ATR(4, g, !DQ);
          if (j == 0 && it > 0) mbar_wait(b_acc, (it - 1) & 1);  // previous item's accumulators read out
          tc_fence_after();
          const uint32_t ta = smem_u32(smem + BW_RING + st * BW_STAGE_STRIDE), tb = ta + TILEB;
#pragma unroll
          for (int k = 0; k < BB / 16; ++k) {  // K = 32 rows of the block, 16 per MMA (8 packed columns)
            const uint32_t acc = (j | k) != 0;
            if (DQ) {  // B = K_j as the MN-major (key rows) operand
              fa_umma_ts(tmem + L::A0, tmem + L::S + b * BB + k * 8, sdesc_sw128(ta + k * 2048, 8192, 1024), IDESC_AC,
                         acc);
            } else {
              fa_umma_ts(tmem + L::A0, tmem + L::S + b * BB + k * 8, sdesc_sw128(tb + k * 2048, 8192, 1024), IDESC_AC,
                         acc);
              fa_umma_ts(tmem + L::A1, tmem + L::P + b * BB + k * 8, sdesc_sw128(ta + k * 2048, 8192, 1024), IDESC_AC,
                         acc);
            }
          }
          umma_commit(&b_free[st]);
        }
        umma_commit(b_done);
        umma_commit(&b_ffree[fb]);
      }
    }
  } else {
    const int q = qw & 3, c = (w - 2) >> 2;  // lane quarter, ping-pong group
    const int lr = q * 32 + lane;            // key row (dK/dV) or query row (dQ)
    const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
    for (int it = 0; it < my_items; ++it) {
      const int item = first_item + it * item_step;
      const int z = item / per_z, blk = item % per_z;
      const int row0 = (z / H) * S, head = z % H;
      float mls = 0.f, dq = 0.f;
      if (DQ) {
        const int64_t zq = static_cast<int64_t>(z) * S + blk * 128 + lr;
        mls = -__ldg(lse2 + zq);
        dq = __ldg(dvec + zq);
      }
      for (int j = c; j < nb; j += 2) {  // nb is even: block gb goes to group gb & 1 == c
        const uint32_t gb = static_cast<uint32_t>(it * nb + j);
        const int st = gb % BW_STAGES, b = gb % NB;
        const uint32_t ts = trow + L::S + b * BB, tp = trow + L::P + b * BB;
        const float* vec = reinterpret_cast<const float*>(smem + BW_RING + st * BW_STAGE_STRIDE + 2 * TILEB);
        if (!DQ) mbar_wait(&b_full[st], (gb / BW_STAGES) & 1);  // lse2 / D of the stage (TMA-written)
        mbar_wait(&b_s[b], (gb / NB) & 1);
        ATR(2, gb, !DQ && lane == 0 && q == 0);
        tc_fence_after();
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // 16 columns at a time; bf16 pairs of half h -> columns 8h..8h+7
          uint32_t sv[16], pv[16];
          fa_tmem_ld16(ts + h * 16, sv);
          fa_tmem_ld16(tp + h * 16, pv);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          uint32_t pk[8], dk[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float m0 = mls, m1 = mls, d0 = dq, d1 = dq;
            if (!DQ) {
              const float2 ls = *reinterpret_cast<const float2*>(vec + h * 16 + 2 * i);
              const float2 dd = *reinterpret_cast<const float2*>(vec + 32 + h * 16 + 2 * i);
              m0 = -ls.x;
              m1 = -ls.y;
              d0 = dd.x;
              d1 = dd.y;
            }
            const float p0 = fa_ex2(fmaf(__uint_as_float(sv[2 * i]), sl2, m0));
            const float p1 = fa_ex2(fmaf(__uint_as_float(sv[2 * i + 1]), sl2, m1));
            pk[i] = fa_pack(p0, p1);
            dk[i] = fa_pack(p0 * fmaf(__uint_as_float(pv[2 * i]), sh.alpha, -d0),
                            p1 * fmaf(__uint_as_float(pv[2 * i + 1]), sh.alpha, -d1));
          }
          // half 0's pairs land in columns 0..7 (already read); half 1 reads 16..31
          if (!DQ) fa_tmem_st8(ts + h * 8, pk);
          fa_tmem_st8((DQ ? ts : tp) + h * 8, dk);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        ATR(3, gb, !DQ && lane == 0 && q == 0);
        if (lane == 0) fa_mbar_arrive(&b_p[b]);
      }
      // the item's accumulators -> bf16 rows of dqkv, then hand them back to the MMA warp
      mbar_wait(b_done, it & 1);
      tc_fence_after();
      const int64_t row = static_cast<int64_t>(row0) + blk * 128 + lr;
      if (DQ) {
        uint32_t v[32];
        tmem_ld32(trow + L::A0 + c * 32, v);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) fa_mbar_arrive(b_acc);
        fa_store_row32(dqkv + row * ld_dqkv + head * FA_DH + c * 32, v);
      } else {
        // group 0 writes dV, group 1 dK
        const uint32_t src = trow + (c == 0 ? L::A0 : L::A1);
        uint32_t v0[32], v1[32];
        tmem_ld32(src, v0);
        tmem_ld32(src + 32, v1);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) fa_mbar_arrive(b_acc);
        bf16* dst = dqkv + row * ld_dqkv + (c == 0 ? 2 * d : d) + head * FA_DH;
        fa_store_row32(dst, v0);
        fa_store_row32(dst + 32, v1);
      }
    }
  }
}

template <bool DQ>
__device__ __forceinline__ void attn_bwd_init_barriers(uint8_t* smem) {
  constexpr int NB = BwTmem<DQ>::NBUF;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + BW_BAR);
  for (int i = 0; i < 4 + 2 * BW_STAGES; ++i) mbar_init(&bar[i], 1);  // ffull, ffree, full, free
  uint64_t* b_s = bar + 4 + 2 * BW_STAGES;
  for (int i = 0; i < NB; ++i) {
    mbar_init(&b_s[i], 1);
    mbar_init(&b_s[NB + i], BW_SMW / 2);  // b_p: the four warps of one group
  }
  mbar_init(&b_s[2 * NB], 1);           // b_done
  mbar_init(&b_s[2 * NB + 1], BW_SMW);  // b_acc
}

// CTAs [0, P) run the dK/dV role, [P, 2P) the dQ role (one of each per SM).
__global__ void __launch_bounds__(BW_THREADS, 2)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap m_qkv128, const __grid_constant__ CUtensorMap m_qkvb,
                    const __grid_constant__ CUtensorMap m_do128, const __grid_constant__ CUtensorMap m_dob,
                    const float* __restrict__ lse2, const float* __restrict__ dvec, bf16* __restrict__ dqkv,
                    int64_t ld_dqkv, FaShape sh, int n, int P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + BW_BAR + 248);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = static_cast<int>(blockIdx.x);
  const bool dq_role = b >= P;
  if (threadIdx.x == 0) {
    if (dq_role)
      attn_bwd_init_barriers<true>(smem);
    else
      attn_bwd_init_barriers<false>(smem);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // prologue above overlaps the previous kernel's tail
  pdl_trigger();
#ifdef GPP_ATTN_TRACE_SOLO  // probe builds: the dK/dV role alone
  if (dq_role) {
  } else
#endif
  if (dq_role)
    attn_bwd_role<true>(smem, tmem, warp, warp, lane, m_qkv128, m_qkvb, m_do128, m_dob, lse2, dvec, dqkv, ld_dqkv,
                        sh, b - P, P, n);
  else
    attn_bwd_role<false>(smem, tmem, warp, warp, lane, m_qkv128, m_qkvb, m_do128, m_dob, lse2, dvec, dqkv, ld_dqkv,
                         sh, b, P, n);
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
  }
}

}  // namespace tc

#ifdef GPP_ATTN_TRACE
extern "C" int gpp_attn_trace_read(long long* out) {
  return cudaMemcpyFromSymbol(out, tc::g_attn_trace, sizeof(tc::g_attn_trace)) == cudaSuccess ? 0 : 1;
}
#endif

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
  tc::FaShape sh{static_cast<int>(S), static_cast<int>(d), static_cast<int>(H), scale};
  // GPP_ATTN_FWD=resident: the 512-column kernel (whole score block in TMEM) for A/B runs
  // default: the online kernel; GPP_ATTN_FWD=stream (two-pass streamed) / resident for A/B runs
  static const char fwd_kind = [] { const char* e = std::getenv("GPP_ATTN_FWD"); return e ? e[0] : 'o'; }();
  const bool resident = fwd_kind == 'r';
  if (fwd_kind == 'o') {  // one pass, two ping-pong groups, conditional rescale
    CUtensorMap mkv;
    if ((rc = tc::make_map_bf16(&mkv, qkv, 3 * d, T, 3 * d, 64, 64))) return rc;
    static bool attr3 = false;
    if (!attr3) {
      cudaFuncSetAttribute(tc::attn_fwd_online_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM_FW2);
      attr3 = true;
    }
    launch_pdl(tc::attn_fwd_online_kernel, dim3(static_cast<unsigned>(Z * (S / 128))), dim3(tc::FW_THREADS),
               tc::SMEM_FW2, static_cast<cudaStream_t>(stream), mq, mkv, lse2, static_cast<bf16*>(o), ldo, sh);
    GPP_LAUNCH_CHECK();
    return GPP_OK;
  }
  if (!resident) {
    CUtensorMap mkv;
    if ((rc = tc::make_map_bf16(&mkv, qkv, 3 * d, T, 3 * d, 64, 64))) return rc;
    static bool attr2 = false;
    if (!attr2) {
      cudaFuncSetAttribute(tc::attn_fwd_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM_FW2);
      attr2 = true;
    }
    launch_pdl(tc::attn_fwd_stream_kernel, dim3(static_cast<unsigned>(Z * (S / 128))), dim3(tc::FW_THREADS),
               tc::SMEM_FW2, static_cast<cudaStream_t>(stream), mq, mkv, lse2, static_cast<bf16*>(o), ldo, sh);
    GPP_LAUNCH_CHECK();
    return GPP_OK;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc::attn_fwd_lse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM_FWL);
    attr = true;
  }
  launch_pdl(tc::attn_fwd_lse_kernel, dim3(static_cast<unsigned>(Z * (S / 128))), dim3(tc::FW_THREADS), tc::SMEM_FWL,
             static_cast<cudaStream_t>(stream), mq, mk, mv, lse2, static_cast<bf16*>(o), ldo, sh);
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
  GPP_ARG_CHECK(ldo % 8 == 0 && (reinterpret_cast<uintptr_t>(o) & 15) == 0, "16-byte aligned o");
  launch_pdl(tc::attn_bwd_prep_kernel, dim3(static_cast<unsigned>((T * H * 8 + 255) / 256)), dim3(256), 0, s, dvec,
             static_cast<const bf16*>(o), ldo, static_cast<const bf16*>(dout), lddo, T, static_cast<int>(S),
             static_cast<int>(H), scale);
  GPP_LAUNCH_CHECK();
  CUtensorMap mk128, mq64, mdo64, mdo128;  // qkv maps serve Q, K and V by coordinates
  if ((rc = tc::make_map_bf16(&mk128, qkv, 3 * d, T, 3 * d, 64, 128))) return rc;
  if ((rc = tc::make_map_bf16(&mq64, qkv, 3 * d, T, 3 * d, 64, tc::BB))) return rc;
  if ((rc = tc::make_map_bf16(&mdo64, dout, d, T, lddo, 64, tc::BB))) return rc;
  if ((rc = tc::make_map_bf16(&mdo128, dout, d, T, lddo, 64, 128))) return rc;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc::attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM_BW);
    attr = true;
  }
  tc::FaShape sh{static_cast<int>(S), static_cast<int>(d), static_cast<int>(H), scale};
  const int n = static_cast<int>(Z * (S / 128));
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int P = std::min(n, sms > 0 ? sms : 148);  // one CTA of each role per SM
  launch_pdl(tc::attn_bwd_kernel, dim3(static_cast<unsigned>(2 * P)), dim3(tc::BW_THREADS), tc::SMEM_BW, s, mk128,
             mq64, mdo128, mdo64, lse2, dvec, static_cast<bf16*>(dqkv), 3 * d, sh, n, P);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

}  // extern "C"
