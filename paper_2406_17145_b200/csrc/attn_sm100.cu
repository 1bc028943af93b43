// Fused MMT attention for sm_100a (S <= 512 keys, head dim 64).
//
// One CTA per (z = sample x head, 128 query rows); the whole 128 x S score block lives
// in TMEM (512 fp32 columns), so the thread owning a query row sees every key of it.
//
//   attn_fwd2_kernel (default): as below, but P stays in TMEM (bf16 pairs over the consumed
//                     score columns) as the A operand of O = P V, and goes to HBM through a
//                     small row staging buffer: ~103 KB of smem, two CTAs per SM.
//   attn_fwd_kernel : S = Q K^T (tcgen05, TMEM)  ->  P = softmax(alpha S)  (3 TMEM passes:
//                     max, exp parked back with tcgen05.st, normalise) written as bf16 into
//                     shared memory in the 128B-swizzled K-major operand layout, from where
//                     (a) TMA stores it to HBM (the backward's P) and (b) it is the A operand
//                     of O = P V (second tcgen05 MMA into TMEM columns 0..63).
//   attn_bwd_kernel : dP = dO V^T (TMEM) with the P tile streamed into shared memory by TMA
//                     meanwhile;  D = rowsum(dO o O) (= rowsum(P o dP), the FlashAttention
//                     identity, from two 128 x 64 tiles instead of a second pass over P);
//                     one pass dS = alpha P o (dP - D) written in place over P in shared
//                     memory, TMA-stored to HBM (for dK = dS^T Q) and used as the A operand of
//                     dQ = dS K (tcgen05 into TMEM columns 0..63).
//
// Versus the previous path (scores+softmax kernel, then a P.V GEMM; softmax-backward kernel
// reading P twice, then a dS.K GEMM) this removes one launch and one full Z S^2 bf16 read
// per direction, makes every P / dS transfer a TMA bulk copy, and halves the backward's
// TMEM and P passes.  Layout: packed QKV [m S, 3d] (Q | K | V, head h at columns h*64),
// o / dout [m S, d] head-interleaved, P / dS [Z S, S] with z = sample * H + head.
#include <cuda.h>

#include <cstdlib>

#include "gemm.cuh"
#include "tc_ptx.cuh"

namespace gpp {
namespace tc {

int make_map_bf16(CUtensorMap* out, const void* ptr, int64_t inner, int64_t outer, int64_t ld, int box_inner,
                  int box_outer);

namespace {

constexpr int AT_EPI_WARPS = 8;                      // two per TMEM lane quarter (key halves)
constexpr int AT_THREADS = 64 + 32 * AT_EPI_WARPS;   // + TMA warp + MMA warp
constexpr int AT_DH = 64;
constexpr uint32_t P_TILE = 128 * 64 * 2;            // one 64-key block of P: 16 KB

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}

__device__ __forceinline__ void tma_store_commit_wait() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Byte offset of the 16-byte chunk j (0..7, 8 bf16 each) of row r inside a 128B-swizzled
// [rows x 64] bf16 tile (what TMA SWIZZLE_128B writes and the UMMA descriptor reads).
__device__ __forceinline__ uint32_t sw128(int r, int j) {
  return static_cast<uint32_t>(r * 128 + ((j ^ (r & 7)) << 4));
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

__device__ __forceinline__ float2 unpack_bf16(uint32_t u) {
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u));
}

// Combine a per-row value across the two key-half warps of a quarter through smem.
__device__ __forceinline__ float combine_halves(float* red, int hf, int lr, float v, bool is_max) {
  red[hf * 128 + lr] = v;
  asm volatile("bar.sync 1, %0;" ::"n"(32 * AT_EPI_WARPS) : "memory");
  const float o = red[(1 - hf) * 128 + lr];
  asm volatile("bar.sync 1, %0;" ::"n"(32 * AT_EPI_WARPS) : "memory");
  return is_max ? fmaxf(v, o) : v + o;
}

// 32 fp32 accumulator columns of this thread's row -> bf16 -> 64 contiguous bytes in global.
__device__ __forceinline__ void store_row32(bf16* dst, const uint32_t (&v)[32]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint4 pk;
    pk.x = pack_bf16(__uint_as_float(v[8 * i + 0]), __uint_as_float(v[8 * i + 1]));
    pk.y = pack_bf16(__uint_as_float(v[8 * i + 2]), __uint_as_float(v[8 * i + 3]));
    pk.z = pack_bf16(__uint_as_float(v[8 * i + 4]), __uint_as_float(v[8 * i + 5]));
    pk.w = pack_bf16(__uint_as_float(v[8 * i + 6]), __uint_as_float(v[8 * i + 7]));
    *reinterpret_cast<uint4*>(dst + 8 * i) = pk;
  }
}

// 16 consecutive 32-bit TMEM columns of this warp's 32 lanes (one per thread), then wait
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

// D(tmem) (+)= A(tmem, K-major bf16 pairs: lane = row, column j = elements 2j, 2j+1) x B(smem)
__device__ __forceinline__ void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

struct AttnShape {
  int S, d, H;
  float alpha;
};

// shared-memory plan (bytes from the 1024-aligned base)
constexpr uint32_t SM_P = 0;               // [0, 128K): P / dS tile (8 x 16 KB key blocks)
constexpr uint32_t SM_FW_V = 128 * 1024;   // fw: V, 8 x 8 KB MN-major key blocks
constexpr uint32_t SM_FW_BAR = 192 * 1024;
constexpr uint32_t SM_BW_A = 128 * 1024;   // bw: dO (16 KB) + V (2 x 32 KB), then K (8 x 8 KB)
constexpr uint32_t SM_BW_O = 208 * 1024;   // bw: O tile (16 KB)
constexpr uint32_t SM_BW_BAR = 224 * 1024;
constexpr int SMEM_FW = SM_FW_BAR + 1024 + 1024;
// fw2 (P kept in TMEM): Q 16 KB | K, then V, 64 KB | per-warp P row staging | barriers
constexpr uint32_t SM2_KV = 16 * 1024;
constexpr uint32_t SM2_STG = 80 * 1024;
constexpr int STG_LD = 80;  // bytes per staged 32-key row (64 + pad: conflict-free)
constexpr uint32_t SM2_BAR = SM2_STG + AT_EPI_WARPS * 32 * STG_LD;
constexpr int SMEM_FW2 = SM2_BAR + 1024 + 1024;  // ~103 KB: two CTAs per SM
constexpr int SMEM_BW = SM_BW_BAR + 1024 + 1024;

}  // namespace

// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(AT_THREADS, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap m_q, const __grid_constant__ CUtensorMap m_k,
                    const __grid_constant__ CUtensorMap m_v, const __grid_constant__ CUtensorMap m_p,
                    bf16* __restrict__ o, int64_t ldo, AttnShape sh) {
  constexpr uint32_t IDESC_S = idesc_bf16<256, false, false>();
  constexpr uint32_t IDESC_O = idesc_bf16<AT_DH, false, true>();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sp = smem + SM_P;
  uint8_t* sv = smem + SM_FW_V;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SM_FW_BAR);
  uint64_t* bar_qk = bar + 0;  // Q + K landed
  uint64_t* bar_v = bar + 1;   // V landed
  uint64_t* bar_s = bar + 2;   // scores MMA done
  uint64_t* bar_p = bar + 3;   // P written to smem (8 epilogue warps)
  uint64_t* bar_o = bar + 4;   // P V MMA done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 8);
  float* red = reinterpret_cast<float*>(smem + SM_FW_BAR + 128);

  const int S = sh.S, d = sh.d, H = sh.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mblocks = S / 128;
  const int z = static_cast<int>(blockIdx.x) / mblocks;
  const int m_blk = static_cast<int>(blockIdx.x) % mblocks;
  const int sample = z / H, head = z % H;
  const int row0 = sample * S;          // first token row of this sample
  const int nkb = S / 64;               // 64-key blocks
  const int nh = (S + 255) / 256;       // N=256 score MMAs

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 5; ++i) mbar_init(&bar[i], i == 3 ? AT_EPI_WARPS : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&m_q)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&m_p)) : "memory");
      mbar_expect_tx(bar_qk, 128 * 128 + nh * 256 * 128);
      tma_load_2d(sp, &m_q, bar_qk, head * AT_DH, row0 + m_blk * 128);
      for (int h = 0; h < nh; ++h)
        tma_load_2d(sp + 16384 + h * 32768, &m_k, bar_qk, d + head * AT_DH, row0 + h * 256);
      mbar_expect_tx(bar_v, nkb * 8192);
      for (int kb = 0; kb < nkb; ++kb) tma_load_2d(sv + kb * 8192, &m_v, bar_v, 2 * d + head * AT_DH, row0 + kb * 64);
      // P tile -> HBM once the epilogue has written it
      mbar_wait(bar_p, 0);
      for (int kb = 0; kb < nkb; ++kb) tma_store_2d(&m_p, sp + kb * P_TILE, kb * 64, z * S + m_blk * 128);
      tma_store_commit_wait();
    }
  } else {
    if (warp == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    asm volatile("bar.sync 2, %0;" ::"n"(32 + 32 * AT_EPI_WARPS) : "memory");  // warps 1..9
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp == 1) {
      if (lane == 0) {
        mbar_wait(bar_qk, 0);
        tc_fence_after();
        const uint32_t qa = smem_u32(sp), ka = smem_u32(sp + 16384);
#pragma unroll
        for (int k = 0; k < AT_DH / 16; ++k)
          for (int h = 0; h < nh; ++h)
            umma_bf16(tmem + h * 256, sdesc_sw128(qa + k * 32, 16, 1024),
                      sdesc_sw128(ka + h * 32768 + k * 32, 16, 1024), IDESC_S, k != 0);
        umma_commit(bar_s);
        mbar_wait(bar_p, 0);
        mbar_wait(bar_v, 0);
        tc_fence_after();
        const uint32_t pa = smem_u32(sp), va = smem_u32(sv);
        for (int kb = 0; kb < nkb; ++kb)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(tmem, sdesc_sw128(pa + kb * P_TILE + k * 32, 16, 1024),
                      sdesc_sw128(va + kb * 8192 + k * 2048, 8192, 1024), IDESC_O, (kb | k) != 0);
        umma_commit(bar_o);
      }
    } else {
      // epilogue warps 2..9: quarter q (32 query rows), key half hf
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
      mx = combine_halves(red, hf, lr, mx, true);
      const float sl2 = sh.alpha * 1.4426950408889634f;
      const float mb = mx * sl2;
      float sum = 0.f;
      for (int c = c_lo; c < c_hi; ++c) {
        uint32_t v[32];
        tmem_ld32(trow + c * 32, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float e = exp2f(fmaf(__uint_as_float(v[j]), sl2, -mb));
          sum += e;
          v[j] = __float_as_uint(e);
        }
        tmem_st32(trow + c * 32, v);
      }
      const float inv = 1.f / combine_halves(red, hf, lr, sum, false);
      for (int c = c_lo; c < c_hi; ++c) {
        uint32_t v[32];
        tmem_ld32(trow + c * 32, v);
        uint8_t* blk = sp + (c >> 1) * P_TILE;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint4 pk;
          pk.x = pack_bf16(__uint_as_float(v[8 * i + 0]) * inv, __uint_as_float(v[8 * i + 1]) * inv);
          pk.y = pack_bf16(__uint_as_float(v[8 * i + 2]) * inv, __uint_as_float(v[8 * i + 3]) * inv);
          pk.z = pack_bf16(__uint_as_float(v[8 * i + 4]) * inv, __uint_as_float(v[8 * i + 5]) * inv);
          pk.w = pack_bf16(__uint_as_float(v[8 * i + 6]) * inv, __uint_as_float(v[8 * i + 7]) * inv);
          *reinterpret_cast<uint4*>(blk + sw128(lr, (c & 1) * 4 + i)) = pk;
        }
      }
      fence_proxy_async_smem();  // generic-proxy smem writes -> visible to TMA / tcgen05
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_p);
      // O = P V: columns [hf*32, hf*32+32) of this warp's rows
      mbar_wait(bar_o, 0);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld32(trow + hf * 32, v);
      store_row32(o + static_cast<int64_t>(row0 + m_blk * 128 + lr) * ldo + head * AT_DH + hf * 32, v);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(*tmem_slot) : "memory");
  }
}

// ---------------------------------------------------------------------------------------
// Forward with P kept in TMEM: the normalised bf16 P is written back over the consumed
// score columns (keys [0,256) -> columns [0,128), keys [256,512) -> [256,384)) and is the
// A operand of O = P V straight from TMEM (tcgen05.mma [d], [a_tmem], b_desc); O goes to
// columns [448, 512).  Shared memory drops to Q + K/V (V loaded over K once the scores
// MMA is done) + row staging for the P stores to HBM, so two CTAs fit per SM: the second
// issues its Q/K loads (before its TMEM allocation) while the first runs its softmax.
__global__ void __launch_bounds__(AT_THREADS, 2)
    attn_fwd2_kernel(const __grid_constant__ CUtensorMap m_q, const __grid_constant__ CUtensorMap m_k,
                     const __grid_constant__ CUtensorMap m_v, bf16* __restrict__ P, bf16* __restrict__ o,
                     int64_t ldo, AttnShape sh) {
  constexpr uint32_t IDESC_S = idesc_bf16<256, false, false>();
  constexpr uint32_t IDESC_O = idesc_bf16<AT_DH, false, true>();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sq = smem;
  uint8_t* skv = smem + SM2_KV;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SM2_BAR);
  uint64_t* bar_qk = bar + 0;
  uint64_t* bar_v = bar + 1;
  uint64_t* bar_s = bar + 2;
  uint64_t* bar_p = bar + 3;   // P in TMEM (8 epilogue warps)
  uint64_t* bar_o = bar + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 8);
  float* red = reinterpret_cast<float*>(smem + SM2_BAR + 128);

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
    for (int i = 0; i < 5; ++i) mbar_init(&bar[i], i == 3 ? AT_EPI_WARPS : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(bar_qk, 128 * 128 + nh * 256 * 128);
      tma_load_2d(sq, &m_q, bar_qk, head * AT_DH, row0 + m_blk * 128);
      for (int h = 0; h < nh; ++h)
        tma_load_2d(skv + h * 32768, &m_k, bar_qk, d + head * AT_DH, row0 + h * 256);
      mbar_wait(bar_s, 0);  // K consumed: V (MN-major key blocks) over it
      mbar_expect_tx(bar_v, nkb * 8192);
      for (int kb = 0; kb < nkb; ++kb) tma_load_2d(skv + kb * 8192, &m_v, bar_v, 2 * d + head * AT_DH, row0 + kb * 64);
    }
  } else {
    if (warp == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    asm volatile("bar.sync 2, %0;" ::"n"(32 + 32 * AT_EPI_WARPS) : "memory");
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp == 1) {
      if (lane == 0) {
        mbar_wait(bar_qk, 0);
        tc_fence_after();
        const uint32_t qa = smem_u32(sq), ka = smem_u32(skv);
#pragma unroll
        for (int k = 0; k < AT_DH / 16; ++k)
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
            umma_ts(tmem + 448, tmem + acol, sdesc_sw128(va + kb * 8192 + k * 2048, 8192, 1024), IDESC_O,
                    (kb | k) != 0);
          }
        umma_commit(bar_o);
      }
    } else {
      const int q = warp & 3, hf = (warp - 2) / 4;
      const int lr = q * 32 + lane;
      const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
      const int c_lo = hf * 8, c_hi = min(S / 32, hf * 8 + 8);
      uint8_t* stg = smem + SM2_STG + (warp - 2) * 32 * STG_LD;
      const int row_base = m_blk * 128 + q * 32;  // within z
      bf16* pz = P + static_cast<int64_t>(z) * S * S;
      mbar_wait(bar_s, 0);
      tc_fence_after();
      float mx = -INFINITY;
      for (int c = c_lo; c < c_hi; ++c) {
        uint32_t v[32];
        tmem_ld32(trow + c * 32, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) mx = fmaxf(mx, __uint_as_float(v[j]));
      }
      mx = combine_halves(red, hf, lr, mx, true);
      const float sl2 = sh.alpha * 1.4426950408889634f;
      const float mb = mx * sl2;
      float sum = 0.f;
      for (int c = c_lo; c < c_hi; ++c) {
        uint32_t v[32];
        tmem_ld32(trow + c * 32, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float e = exp2f(fmaf(__uint_as_float(v[j]), sl2, -mb));
          sum += e;
          v[j] = __float_as_uint(e);
        }
        tmem_st32(trow + c * 32, v);
      }
      const float inv = 1.f / combine_halves(red, hf, lr, sum, false);
      for (int c = c_lo; c < c_hi; ++c) {
        uint32_t v[32];
        tmem_ld32(trow + c * 32, v);
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          pk[j] = pack_bf16(__uint_as_float(v[2 * j]) * inv, __uint_as_float(v[2 * j + 1]) * inv);
        // packed P over consumed score columns of this half (chunk c -> columns of chunk <= c)
        tmem_st16(trow + (c >> 3) * 256 + (c & 7) * 16, pk);
        // and to HBM: this thread's 64 B -> smem -> 4 lanes per row, 16 B each (coalesced)
#pragma unroll
        for (int i = 0; i < 4; ++i)
          *reinterpret_cast<uint4*>(stg + lane * STG_LD + i * 16) = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = (lane >> 2) + 8 * i, seg = lane & 3;
          const uint4 val = *reinterpret_cast<const uint4*>(stg + r * STG_LD + seg * 16);
          *reinterpret_cast<uint4*>(pz + static_cast<int64_t>(row_base + r) * S + c * 32 + seg * 8) = val;
        }
        __syncwarp();
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_p);
      mbar_wait(bar_o, 0);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld32(trow + 448 + hf * 32, v);
      store_row32(o + static_cast<int64_t>(row0 + m_blk * 128 + lr) * ldo + head * AT_DH + hf * 32, v);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(*tmem_slot) : "memory");
  }
}

// ---------------------------------------------------------------------------------------
__global__ void __launch_bounds__(AT_THREADS, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap m_do, const __grid_constant__ CUtensorMap m_kv,
                    const __grid_constant__ CUtensorMap m_kmn, const __grid_constant__ CUtensorMap m_o,
                    const __grid_constant__ CUtensorMap m_p, const __grid_constant__ CUtensorMap m_ds,
                    bf16* __restrict__ dqkv, int64_t ld_dqkv, AttnShape sh) {
  constexpr uint32_t IDESC_S = idesc_bf16<256, false, false>();
  constexpr uint32_t IDESC_Q = idesc_bf16<AT_DH, false, true>();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sp = smem + SM_P;        // P, overwritten in place by dS
  uint8_t* sa = smem + SM_BW_A;     // dO | V halves, later K (MN-major blocks)
  uint8_t* so = smem + SM_BW_O;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SM_BW_BAR);
  uint64_t* bar_a = bar + 0;     // dO + V landed
  uint64_t* bar_o = bar + 1;     // O landed
  uint64_t* bar_pl = bar + 2;    // P landed
  uint64_t* bar_s = bar + 3;     // dP MMA done
  uint64_t* bar_free = bar + 4;  // epilogue finished reading dO (8 warps)
  uint64_t* bar_k = bar + 5;     // K landed
  uint64_t* bar_ds = bar + 6;    // dS written to smem (8 warps)
  uint64_t* bar_q = bar + 7;     // dQ MMA done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 8);

  const int S = sh.S, d = sh.d, H = sh.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mblocks = S / 128;
  const int z = static_cast<int>(blockIdx.x) / mblocks;
  const int m_blk = static_cast<int>(blockIdx.x) % mblocks;
  const int sample = z / H, head = z % H;
  const int row0 = sample * S;
  const int qrow0 = row0 + m_blk * 128;
  const int prow0 = z * S + m_blk * 128;
  const int nkb = S / 64;
  const int nh = (S + 255) / 256;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bar[i], (i == 4 || i == 6) ? AT_EPI_WARPS : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(bar_a, 128 * 128 + nh * 256 * 128);
      tma_load_2d(sa, &m_do, bar_a, head * AT_DH, qrow0);
      for (int h = 0; h < nh; ++h)
        tma_load_2d(sa + 16384 + h * 32768, &m_kv, bar_a, 2 * d + head * AT_DH, row0 + h * 256);
      mbar_expect_tx(bar_o, 128 * 128);
      tma_load_2d(so, &m_o, bar_o, head * AT_DH, qrow0);
      mbar_expect_tx(bar_pl, nkb * P_TILE);
      for (int kb = 0; kb < nkb; ++kb) tma_load_2d(sp + kb * P_TILE, &m_p, bar_pl, kb * 64, prow0);
      // K (MN-major, for dQ = dS K) replaces dO / V once the dP MMA and the D pass are done
      mbar_wait(bar_s, 0);
      mbar_wait(bar_free, 0);
      mbar_expect_tx(bar_k, nkb * 8192);
      for (int kb = 0; kb < nkb; ++kb) tma_load_2d(sa + kb * 8192, &m_kmn, bar_k, d + head * AT_DH, row0 + kb * 64);
      mbar_wait(bar_ds, 0);
      for (int kb = 0; kb < nkb; ++kb) tma_store_2d(&m_ds, sp + kb * P_TILE, kb * 64, prow0);
      tma_store_commit_wait();
    }
  } else {
    if (warp == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    asm volatile("bar.sync 2, %0;" ::"n"(32 + 32 * AT_EPI_WARPS) : "memory");
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp == 1) {
      if (lane == 0) {
        mbar_wait(bar_a, 0);
        tc_fence_after();
        const uint32_t aa = smem_u32(sa), va = smem_u32(sa + 16384);
#pragma unroll
        for (int k = 0; k < AT_DH / 16; ++k)
          for (int h = 0; h < nh; ++h)
            umma_bf16(tmem + h * 256, sdesc_sw128(aa + k * 32, 16, 1024),
                      sdesc_sw128(va + h * 32768 + k * 32, 16, 1024), IDESC_S, k != 0);
        umma_commit(bar_s);
        mbar_wait(bar_ds, 0);
        mbar_wait(bar_k, 0);
        tc_fence_after();
        const uint32_t pa = smem_u32(sp), ka = smem_u32(sa);
        for (int kb = 0; kb < nkb; ++kb)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(tmem, sdesc_sw128(pa + kb * P_TILE + k * 32, 16, 1024),
                      sdesc_sw128(ka + kb * 8192 + k * 2048, 8192, 1024), IDESC_Q, (kb | k) != 0);
        umma_commit(bar_q);
      }
    } else {
      const int q = warp & 3, hf = (warp - 2) / 4;
      const int lr = q * 32 + lane;
      const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
      const int c_lo = hf * 8, c_hi = min(S / 32, hf * 8 + 8);
      // D = rowsum(dO o O) over the 64 head columns (both swizzled 128 x 64 tiles)
      mbar_wait(bar_a, 0);
      mbar_wait(bar_o, 0);
      float D = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint4 a = *reinterpret_cast<const uint4*>(sa + sw128(lr, j));
        const uint4 b = *reinterpret_cast<const uint4*>(so + sw128(lr, j));
        const uint32_t* ua = reinterpret_cast<const uint32_t*>(&a);
        const uint32_t* ub = reinterpret_cast<const uint32_t*>(&b);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float2 x = unpack_bf16(ua[t]), y = unpack_bf16(ub[t]);
          D = fmaf(x.x, y.x, fmaf(x.y, y.y, D));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_free);
      mbar_wait(bar_s, 0);
      mbar_wait(bar_pl, 0);
      tc_fence_after();
      const float alpha = sh.alpha;
      for (int c = c_lo; c < c_hi; ++c) {
        uint32_t v[32];
        tmem_ld32(trow + c * 32, v);
        uint8_t* blk = sp + (c >> 1) * P_TILE;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint4* ptr = reinterpret_cast<uint4*>(blk + sw128(lr, (c & 1) * 4 + i));
          uint4 pk = *ptr;
          uint32_t* w = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float2 p = unpack_bf16(w[t]);
            const float g0 = __uint_as_float(v[8 * i + 2 * t]) - D;
            const float g1 = __uint_as_float(v[8 * i + 2 * t + 1]) - D;
            w[t] = pack_bf16(alpha * p.x * g0, alpha * p.y * g1);
          }
          *ptr = pk;
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_ds);
      mbar_wait(bar_q, 0);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld32(trow + hf * 32, v);
      store_row32(dqkv + static_cast<int64_t>(qrow0 + lr) * ld_dqkv + head * AT_DH + hf * 32, v);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(*tmem_slot) : "memory");
  }
}

}  // namespace tc

namespace {
int attn_checks(const void* qkv, int64_t m, int64_t S, int64_t d, int64_t H) {
  GPP_ARG_CHECK(qkv != nullptr, "null qkv");
  GPP_ARG_CHECK(m >= 1 && H >= 1 && d == H * 64, "fused attention needs head dim 64 (d == 64 H)");
  GPP_ARG_CHECK(S >= 128 && S <= 512 && S % 128 == 0, "fused attention needs S in {128, 256, 384, 512}");
  GPP_ARG_CHECK((reinterpret_cast<uintptr_t>(qkv) & 15) == 0, "16-byte aligned qkv");
  return GPP_OK;
}
}  // namespace

int tc_attn_fwd(const void* qkv, void* P, void* o, int64_t ldo, int64_t m, int64_t S, int64_t d, int64_t H,
                float alpha, cudaStream_t stream) {
  int rc = attn_checks(qkv, m, S, d, H);
  if (rc) return rc;
  GPP_ARG_CHECK(P && o && ldo % 8 == 0 && (reinterpret_cast<uintptr_t>(o) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(P) & 15) == 0, "16-byte aligned P / o");
  GPP_ARG_CHECK(alpha > 0.f, "softmax scale must be positive");
  const int64_t T = m * S, Z = m * H;
  CUtensorMap mq, mk, mv, mp;
  if ((rc = tc::make_map_bf16(&mq, qkv, 3 * d, T, 3 * d, 64, 128))) return rc;
  if ((rc = tc::make_map_bf16(&mk, qkv, 3 * d, T, 3 * d, 64, 256))) return rc;
  if ((rc = tc::make_map_bf16(&mv, qkv, 3 * d, T, 3 * d, 64, 64))) return rc;
  if ((rc = tc::make_map_bf16(&mp, P, S, Z * S, S, 64, 128))) return rc;
  tc::AttnShape sh{static_cast<int>(S), static_cast<int>(d), static_cast<int>(H), alpha};
  // P kept in TMEM (two CTAs per SM) by default; GPP_ATTN_FWD2=0 selects the smem-P kernel
  static const bool p_in_tmem = [] { const char* e = std::getenv("GPP_ATTN_FWD2"); return !(e && e[0] == '0'); }();
  if (p_in_tmem) {
    static bool attr2 = false;
    if (!attr2) {
      cudaFuncSetAttribute(tc::attn_fwd2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM_FW2);
      attr2 = true;
    }
    tc::attn_fwd2_kernel<<<static_cast<unsigned>(Z * (S / 128)), tc::AT_THREADS, tc::SMEM_FW2, stream>>>(
        mq, mk, mv, static_cast<bf16*>(P), static_cast<bf16*>(o), ldo, sh);
    GPP_LAUNCH_CHECK();
    return GPP_OK;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc::attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM_FW);
    attr = true;
  }
  tc::attn_fwd_kernel<<<static_cast<unsigned>(Z * (S / 128)), tc::AT_THREADS, tc::SMEM_FW, stream>>>(
      mq, mk, mv, mp, static_cast<bf16*>(o), ldo, sh);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int tc_attn_bwd(const void* qkv, const void* P, const void* o, int64_t ldo, const void* dout, int64_t lddo,
                void* dS, void* dqkv, int64_t m, int64_t S, int64_t d, int64_t H, float alpha, cudaStream_t stream) {
  int rc = attn_checks(qkv, m, S, d, H);
  if (rc) return rc;
  GPP_ARG_CHECK(P && o && dout && dS && dqkv, "null pointer");
  GPP_ARG_CHECK(ldo % 8 == 0 && lddo % 8 == 0 && (reinterpret_cast<uintptr_t>(dqkv) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(o) & 15) == 0 && (reinterpret_cast<uintptr_t>(dout) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(P) & 15) == 0 && (reinterpret_cast<uintptr_t>(dS) & 15) == 0,
                "16-byte alignment");
  const int64_t T = m * S, Z = m * H;
  CUtensorMap mdo, mkv, mkmn, mo, mp, mds;
  if ((rc = tc::make_map_bf16(&mdo, dout, d, T, lddo, 64, 128))) return rc;
  if ((rc = tc::make_map_bf16(&mkv, qkv, 3 * d, T, 3 * d, 64, 256))) return rc;
  if ((rc = tc::make_map_bf16(&mkmn, qkv, 3 * d, T, 3 * d, 64, 64))) return rc;
  if ((rc = tc::make_map_bf16(&mo, o, d, T, ldo, 64, 128))) return rc;
  if ((rc = tc::make_map_bf16(&mp, P, S, Z * S, S, 64, 128))) return rc;
  if ((rc = tc::make_map_bf16(&mds, dS, S, Z * S, S, 64, 128))) return rc;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc::attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::SMEM_BW);
    attr = true;
  }
  tc::AttnShape sh{static_cast<int>(S), static_cast<int>(d), static_cast<int>(H), alpha};
  tc::attn_bwd_kernel<<<static_cast<unsigned>(Z * (S / 128)), tc::AT_THREADS, tc::SMEM_BW, stream>>>(
      mdo, mkv, mkmn, mo, mp, mds, static_cast<bf16*>(dqkv), 3 * d, sh);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

}  // namespace gpp

extern "C" {

int gpp_attn_fwd(const void* qkv, void* p, void* o, int64_t ldo, int64_t m, int64_t S, int64_t d, int64_t H,
                 float scale, void* stream) {
  return gpp::tc_attn_fwd(qkv, p, o, ldo, m, S, d, H, scale, static_cast<cudaStream_t>(stream));
}

int gpp_attn_bwd(const void* qkv, const void* p, const void* o, int64_t ldo, const void* dout, int64_t lddo,
                 void* ds, void* dqkv, int64_t m, int64_t S, int64_t d, int64_t H, float scale, void* stream) {
  return gpp::tc_attn_bwd(qkv, p, o, ldo, dout, lddo, ds, dqkv, m, S, d, H, scale,
                          static_cast<cudaStream_t>(stream));
}

}  // extern "C"
