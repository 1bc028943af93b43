// tcgen05 / TMEM / TMA GEMM for sm_100a — the dense-operator hot path of the
// GPP stage executor (fw, dgrad and wgrad of every Linear in MMT / CANDLE-Uno /
// DLRM MLP stages).
//
// C[M,N] = epilogue( sum_k A(m,k) * B(n,k) )
//   A is K-major ([M][lda], k contiguous) or MN-major ([K][lda], m contiguous);
//   B likewise with n.  The three training GEMMs of y = x W^T map to:
//     fw    : A = x  (K-major),  B = W  (K-major)
//     dgrad : A = dy (K-major),  B = W  (MN-major: W is [N_out][K_in], n = K_in)
//     wgrad : A = dy (MN-major), B = x  (MN-major)  -> fp32 dW, optional accumulate
//
// Structure (warp-specialised, one output tile of 128 x BN per CTA, 192 threads):
//   warp 0 (one lane)  : TMA producer, STAGES-deep smem ring (full/empty mbarriers)
//   warp 1             : TMEM allocator; one lane issues tcgen05.mma (M=128, N=BN, K=16)
//                        and tcgen05.commit's the ring slots / the accumulator
//   warps 2..5         : epilogue: tcgen05.ld 32x32b -> registers -> fused
//                        bias / activation / residual / act'-mask -> global
// Operand tiles are 128B-swizzled (TMA SWIZZLE_128B == UMMA SWIZZLE_128B).
#include <cuda.h>
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <unordered_map>

#define GPP_PDL_CLASS 1  // programmatic-dependent-launch family: tcgen05 GEMMs
#include "gemm.cuh"
#include "tc_ptx.cuh"

namespace gpp {
namespace tc {

constexpr int NUM_THREADS = 192;
#ifndef GPP_SGD_DEPTH
#define GPP_SGD_DEPTH 2
#endif
constexpr int SGD_DEPTH = GPP_SGD_DEPTH;  // master chunks in flight per warp (3 with a 3-stage ring measured slower)
constexpr int SGD_STAGES256 = SGD_DEPTH >= 3 ? 3 : 4;     // operand ring of the 256-wide SGD GEMM
constexpr int PAIR_EPI_WARPS = 8;                          // two epilogue warpgroups
constexpr int PAIR_THREADS = 64 + 32 * PAIR_EPI_WARPS;     // + TMA warp + MMA warp

// L2 prefetch of this CTA's share of the hinted buffer (64 KB bulk pieces), issued by an
// otherwise idle lane so it overlaps the tensor-bound main loop.
__device__ __forceinline__ void l2_prefetch_share(const EpiParams& ep, int cta, int ncta) {
  if (ep.pf_ptr == nullptr || ep.pf_bytes <= 0) return;
  const int64_t total = ep.pf_bytes & ~static_cast<int64_t>(15);
  const int64_t share = ((total / ncta) + 65535) & ~static_cast<int64_t>(65535);
  const int64_t beg = static_cast<int64_t>(cta) * share;
  const int64_t end = beg + share < total ? beg + share : total;
  const char* base = static_cast<const char*>(ep.pf_ptr);
  for (int64_t off = beg; off < end; off += 65536) {
    const uint32_t n = static_cast<uint32_t>(end - off < 65536 ? end - off : 65536);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + off), "r"(n) : "memory");
  }
}

// 32 bf16 from global (16-byte vector loads when aligned and in bounds).
__device__ __forceinline__ void load_bf16x32(const bf16* p, bool vec, int n_valid, float (&o)[32]) {
  if (vec) {
    uint4 r[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) r[i] = __ldg(reinterpret_cast<const uint4*>(p) + i);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 f = __bfloat1622float2(h[j]);
        o[i * 8 + 2 * j] = f.x;
        o[i * 8 + 2 * j + 1] = f.y;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) o[j] = j < n_valid ? __bfloat162float(p[j]) : 0.f;
  }
}

__device__ __forceinline__ void store_bf16x32(bf16* p, bool vec, int n_valid, const float (&f)[32]) {
  if (vec) {
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
      uint4 pk;
      __nv_bfloat162 h0 = __floats2bfloat162_rn(f[j + 0], f[j + 1]);
      __nv_bfloat162 h1 = __floats2bfloat162_rn(f[j + 2], f[j + 3]);
      __nv_bfloat162 h2 = __floats2bfloat162_rn(f[j + 4], f[j + 5]);
      __nv_bfloat162 h3 = __floats2bfloat162_rn(f[j + 6], f[j + 7]);
      pk.x = *reinterpret_cast<uint32_t*>(&h0);
      pk.y = *reinterpret_cast<uint32_t*>(&h1);
      pk.z = *reinterpret_cast<uint32_t*>(&h2);
      pk.w = *reinterpret_cast<uint32_t*>(&h3);
      *reinterpret_cast<uint4*>(p + j) = pk;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < n_valid) p[j] = __float2bfloat16_rn(f[j]);
  }
}

__device__ __forceinline__ bool al16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15) == 0;
}

// Warp-collective bf16 store of a 32 x 32 chunk (lane = row) through a 2 KB smem tile in the
// 64B-swizzled layout of the aux tiles: each lane writes its row's 64 B, then every store
// instruction moves 8 rows x 64 contiguous bytes (4 lanes per row) instead of 32 rows x
// 16 B -- a quarter of the L1/L2 store transactions.  Rows >= rows_valid are not stored.
__device__ __forceinline__ void store_bf16x32_staged(bf16* base, int64_t ld, const float (&f)[32], uint8_t* stage,
                                                     int lane, int rows_valid) {
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    uint4 pk;
    const int j = 8 * u;
    __nv_bfloat162 h0 = __floats2bfloat162_rn(f[j + 0], f[j + 1]);
    __nv_bfloat162 h1 = __floats2bfloat162_rn(f[j + 2], f[j + 3]);
    __nv_bfloat162 h2 = __floats2bfloat162_rn(f[j + 4], f[j + 5]);
    __nv_bfloat162 h3 = __floats2bfloat162_rn(f[j + 6], f[j + 7]);
    pk.x = *reinterpret_cast<uint32_t*>(&h0);
    pk.y = *reinterpret_cast<uint32_t*>(&h1);
    pk.z = *reinterpret_cast<uint32_t*>(&h2);
    pk.w = *reinterpret_cast<uint32_t*>(&h3);
    *reinterpret_cast<uint4*>(stage + lane * 64 + ((u ^ ((lane >> 1) & 3)) << 4)) = pk;
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = (lane >> 2) + 8 * i, u = lane & 3;
    const uint4 v = *reinterpret_cast<const uint4*>(stage + r * 64 + ((u ^ ((r >> 1) & 3)) << 4));
    if (r < rows_valid) *reinterpret_cast<uint4*>(base + static_cast<int64_t>(r) * ld + u * 8) = v;
  }
  __syncwarp();
}

// Epilogue of one thread: 32 consecutive columns [col0, col0+32) of one row.
// `aux` (residual / act'-saved, 32 values) is loaded by the caller BEFORE the TMEM
// load so its global latency overlaps tcgen05.ld.
template <int EPI>
// `sbias`: the chunk's 32 bias values already staged in shared memory (or null: global).
__device__ __forceinline__ void epilogue_chunk(const EpiParams& ep, const uint32_t (&v)[32],
                                               const float (&aux)[32], int row, int col0, int M,
                                               int N, uint8_t* stage = nullptr, int lane = 0,
                                               const float* sbias = nullptr) {
  // staged (warp-collective, coalesced) bf16 stores: whole 32-column chunks of a FWD / DGRAD
  // epilogue with 16-byte-aligned rows; every lane of the warp takes part
  const int row0 = row - lane;
  bool staged = false;
  if constexpr (EPI == EPI_FWD || EPI == EPI_DGRAD) {
    staged = stage != nullptr && col0 + 32 <= N && row0 < M && ep.ldo % 8 == 0 &&
             al16(static_cast<bf16*>(ep.out) + static_cast<int64_t>(row0) * ep.ldo + col0) &&
             (ep.pre == nullptr || (ep.ldpre % 8 == 0 &&
                                    al16(static_cast<bf16*>(ep.pre) + static_cast<int64_t>(row0) * ep.ldpre + col0)));
  }
  if (!staged && (row >= M || col0 >= N)) return;
  const int rows_valid = M - row0 < 32 ? M - row0 : 32;
  const int n_valid = N - col0 < 32 ? N - col0 : 32;
  const bool full = n_valid == 32;
  float f[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]) * ep.alpha;

  if constexpr (EPI == EPI_SGD) {
    float* master = reinterpret_cast<float*>(ep.out) + static_cast<int64_t>(row) * ep.ldo + col0;
    float* grad = ep.grad + static_cast<int64_t>(row) * ep.ldgrad + col0;
    bf16* shadow = static_cast<bf16*>(ep.pre) + static_cast<int64_t>(row) * ep.ldpre + col0;
    if (full && al16(master) && al16(grad) && al16(shadow)) {
      float m[32];
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        const float4 mv = *reinterpret_cast<const float4*>(master + j);
        m[j] = mv.x; m[j + 1] = mv.y; m[j + 2] = mv.z; m[j + 3] = mv.w;
      }
      if (ep.beta != 0.f) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const float4 g = *reinterpret_cast<const float4*>(grad + j);
          f[j] += g.x; f[j + 1] += g.y; f[j + 2] += g.z; f[j + 3] += g.w;
        }
      }
      if (ep.store_grad) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(grad + j) = make_float4(f[j], f[j + 1], f[j + 2], f[j + 3]);
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) m[j] -= ep.lr * f[j];
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(master + j) = make_float4(m[j], m[j + 1], m[j + 2], m[j + 3]);
      store_bf16x32(shadow, true, 32, m);
    } else {
      for (int j = 0; j < n_valid; ++j) {
        float g = f[j] + (ep.beta != 0.f ? grad[j] : 0.f);
        if (ep.store_grad) grad[j] = g;
        const float mj = master[j] - ep.lr * g;
        master[j] = mj;
        shadow[j] = __float2bfloat16_rn(mj);
      }
    }
    return;
  } else if constexpr (EPI == EPI_F32) {
    float* out = reinterpret_cast<float*>(ep.out) + static_cast<int64_t>(row) * ep.ldo + col0;
    if (full && al16(out)) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 o = make_float4(f[j], f[j + 1], f[j + 2], f[j + 3]);
        if (ep.beta != 0.f) {
          const float4 c = *reinterpret_cast<const float4*>(out + j);
          o.x += ep.beta * c.x; o.y += ep.beta * c.y; o.z += ep.beta * c.z; o.w += ep.beta * c.w;
        }
        *reinterpret_cast<float4*>(out + j) = o;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < n_valid) out[j] = ep.beta != 0.f ? f[j] + ep.beta * out[j] : f[j];
    }
    return;
  } else {
    if constexpr (EPI == EPI_FWD) {
      if (ep.bias != nullptr) {
        if (sbias != nullptr) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 b = *reinterpret_cast<const float4*>(sbias + j);
            f[j] += b.x; f[j + 1] += b.y; f[j + 2] += b.z; f[j + 3] += b.w;
          }
        } else if (full && al16(ep.bias + col0)) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 b = __ldg(reinterpret_cast<const float4*>(ep.bias + col0 + j));
            f[j] += b.x; f[j + 1] += b.y; f[j + 2] += b.z; f[j + 3] += b.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) f[j] += j < n_valid ? __ldg(ep.bias + col0 + j) : 0.f;
        }
      }
      if (ep.pre != nullptr) {
        if (staged) {
          store_bf16x32_staged(static_cast<bf16*>(ep.pre) + static_cast<int64_t>(row0) * ep.ldpre + col0, ep.ldpre, f,
                               stage, lane, rows_valid);
        } else {
          bf16* pre = static_cast<bf16*>(ep.pre) + static_cast<int64_t>(row) * ep.ldpre + col0;
          store_bf16x32(pre, full && al16(pre), n_valid, f);
        }
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) f[j] = act_fwd(f[j], ep.act);
      if (ep.aux != nullptr) {
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] += aux[j];
      }
    } else if constexpr (EPI == EPI_DGRAD) {
      if (ep.act != GPP_ACT_NONE) {
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] *= act_bwd(aux[j], ep.act);
      }
    }
    bf16* out = reinterpret_cast<bf16*>(ep.out) + static_cast<int64_t>(row) * ep.ldo + col0;
    if constexpr (EPI == EPI_BF16) {
      if (ep.beta != 0.f) {
        float c[32];
        load_bf16x32(out, full && al16(out), n_valid, c);
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] += ep.beta * c[j];
      }
    }
    if (staged) {
      store_bf16x32_staged(static_cast<bf16*>(ep.out) + static_cast<int64_t>(row0) * ep.ldo + col0, ep.ldo, f, stage,
                           lane, rows_valid);
    } else {
      store_bf16x32(out, full && al16(out), n_valid, f);
    }
  }
}


// fp32-output epilogues (EPI_F32 / EPI_SGD) through a per-warp 32x32 smem transpose:
// each thread owns one accumulator ROW, but global fp32 rows are written (and the
// master weights read) 128 B per 8 lanes, 4 rows per warp instruction.
constexpr int STAGE_LD = 36;  // floats per staged row (16 B aligned, conflict-free phases)

template <int EPI>
__device__ __forceinline__ void epilogue_f32_coalesced(const EpiParams& ep, const uint32_t (&v)[32],
                                                       float* stage, int row0, int col0, int M,
                                                       int N, int lane) {
  const int sub = lane >> 3;
  const int c4 = (lane & 7) * 4;
  const int col = col0 + c4;
  const int nv = N - col < 4 ? N - col : 4;
  // Issue every global read of this lane's 8 row-pieces up front (one memory latency
  // per chunk instead of one per row): master (+ old grad) for SGD, old out for beta.
  float4 mres[8], gres[8];
  bool vec[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int grow = row0 + 4 * i + sub;
    vec[i] = false;
    if (grow >= M || col >= N) continue;
    if constexpr (EPI == EPI_SGD) {
      const float* master = reinterpret_cast<const float*>(ep.out) + static_cast<int64_t>(grow) * ep.ldo + col;
      const float* grad = ep.grad + static_cast<int64_t>(grow) * ep.ldgrad + col;
      const bf16* shadow = static_cast<const bf16*>(ep.pre) + static_cast<int64_t>(grow) * ep.ldpre + col;
      vec[i] = nv == 4 && al16(master) && al16(grad) && ((reinterpret_cast<uintptr_t>(shadow) & 7) == 0);
      if (vec[i]) {
        mres[i] = *reinterpret_cast<const float4*>(master);
        if (ep.beta != 0.f) gres[i] = *reinterpret_cast<const float4*>(grad);
      }
    } else {
      const float* out = reinterpret_cast<const float*>(ep.out) + static_cast<int64_t>(grow) * ep.ldo + col;
      vec[i] = nv == 4 && al16(out);
      if (vec[i] && ep.beta != 0.f) gres[i] = *reinterpret_cast<const float4*>(out);
    }
  }
  float* mine = stage + lane * STAGE_LD;
#pragma unroll
  for (int j = 0; j < 32; j += 4)
    *reinterpret_cast<float4*>(mine + j) =
        make_float4(__uint_as_float(v[j]) * ep.alpha, __uint_as_float(v[j + 1]) * ep.alpha,
                    __uint_as_float(v[j + 2]) * ep.alpha, __uint_as_float(v[j + 3]) * ep.alpha);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = 4 * i + sub;
    const int grow = row0 + r;
    if (grow >= M || col >= N) continue;
    const float4 a = *reinterpret_cast<const float4*>(stage + r * STAGE_LD + c4);
    float g[4] = {a.x, a.y, a.z, a.w};
    if constexpr (EPI == EPI_SGD) {
      float* master = reinterpret_cast<float*>(ep.out) + static_cast<int64_t>(grow) * ep.ldo + col;
      float* grad = ep.grad + static_cast<int64_t>(grow) * ep.ldgrad + col;
      bf16* shadow = static_cast<bf16*>(ep.pre) + static_cast<int64_t>(grow) * ep.ldpre + col;
      if (vec[i]) {
        if (ep.beta != 0.f) {
          g[0] += gres[i].x; g[1] += gres[i].y; g[2] += gres[i].z; g[3] += gres[i].w;
        }
        if (ep.store_grad) *reinterpret_cast<float4*>(grad) = make_float4(g[0], g[1], g[2], g[3]);
        float4 m = mres[i];
        m.x -= ep.lr * g[0]; m.y -= ep.lr * g[1]; m.z -= ep.lr * g[2]; m.w -= ep.lr * g[3];
        *reinterpret_cast<float4*>(master) = m;
        __nv_bfloat162 lo = __floats2bfloat162_rn(m.x, m.y);
        __nv_bfloat162 hi = __floats2bfloat162_rn(m.z, m.w);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&lo);
        pk.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(shadow) = pk;
      } else {
        for (int t = 0; t < nv; ++t) {
          float gt = g[t] + (ep.beta != 0.f ? grad[t] : 0.f);
          if (ep.store_grad) grad[t] = gt;
          const float mt = master[t] - ep.lr * gt;
          master[t] = mt;
          shadow[t] = __float2bfloat16_rn(mt);
        }
      }
    } else {
      float* out = reinterpret_cast<float*>(ep.out) + static_cast<int64_t>(grow) * ep.ldo + col;
      if (vec[i]) {
        if (ep.beta != 0.f) {
          g[0] += ep.beta * gres[i].x; g[1] += ep.beta * gres[i].y;
          g[2] += ep.beta * gres[i].z; g[3] += ep.beta * gres[i].w;
        }
        *reinterpret_cast<float4*>(out) = make_float4(g[0], g[1], g[2], g[3]);
      } else {
        for (int t = 0; t < nv; ++t) out[t] = ep.beta != 0.f ? g[t] + ep.beta * out[t] : g[t];
      }
    }
  }
  __syncwarp();
}

// ---- fused-SGD fast path (beta == 0, no grad store, aligned rows, N % 4 == 0) ----
// The master chunk does not depend on the accumulator, so it is copied global -> smem
// with cp.async (no registers held) two chunks ahead -- for a tile's first two chunks
// before the accumulator is even ready.  Lane = row then updates its row in place
// (m -= lr * alpha * acc), and the warp writes master + bf16 shadow back coalesced.
__device__ __forceinline__ bool sgd_fast_ok(const EpiParams& ep, int N) {
  const uintptr_t mo = reinterpret_cast<uintptr_t>(ep.out), so = reinterpret_cast<uintptr_t>(ep.pre);
  return ep.beta == 0.f && !ep.store_grad && (N & 3) == 0 && (mo & 15) == 0 && (ep.ldo & 3) == 0 &&
         (so & 7) == 0 && (ep.ldpre & 3) == 0;
}

__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Issue the copy of a 32 x 32 fp32 master chunk (rows row0.., columns col0..) into buf.
__device__ __forceinline__ void sgd_fast_issue(const EpiParams& ep, float* buf, int row0, int col0,
                                               int M, int N, int lane) {
  const int sub = lane >> 3, c4 = (lane & 7) * 4;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = 4 * i + sub, grow = row0 + r;
    if (grow < M && col0 + c4 < N)
      cp_async16(buf + r * STAGE_LD + c4,
                 reinterpret_cast<const float*>(ep.out) + static_cast<int64_t>(grow) * ep.ldo + col0 + c4);
  }
  cp_async_commit();
}

// buf holds the chunk's master (copy complete for this lane); update and write back.
__device__ __forceinline__ void sgd_fast_update(const EpiParams& ep, const uint32_t (&v)[32], float* buf,
                                                int row0, int col0, int M, int N, int lane) {
  __syncwarp();  // every lane's cp.async data visible warp-wide
  const float s = -ep.lr * ep.alpha;
  float* mine = buf + lane * STAGE_LD;
#pragma unroll
  for (int j = 0; j < 32; j += 4) {
    float4 m = *reinterpret_cast<float4*>(mine + j);
    m.x = fmaf(s, __uint_as_float(v[j]), m.x);
    m.y = fmaf(s, __uint_as_float(v[j + 1]), m.y);
    m.z = fmaf(s, __uint_as_float(v[j + 2]), m.z);
    m.w = fmaf(s, __uint_as_float(v[j + 3]), m.w);
    *reinterpret_cast<float4*>(mine + j) = m;
  }
  __syncwarp();
  const int sub = lane >> 3, c4 = (lane & 7) * 4, col = col0 + c4;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = 4 * i + sub, grow = row0 + r;
    if (grow >= M || col >= N) continue;
    const float4 nm = *reinterpret_cast<const float4*>(buf + r * STAGE_LD + c4);
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(ep.out) + static_cast<int64_t>(grow) * ep.ldo + col) = nm;
    __nv_bfloat162 lo = __floats2bfloat162_rn(nm.x, nm.y);
    __nv_bfloat162 hi = __floats2bfloat162_rn(nm.z, nm.w);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&lo);
    pk.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(static_cast<bf16*>(ep.pre) + static_cast<int64_t>(grow) * ep.ldpre + col) = pk;
  }
  __syncwarp();  // buf may be refilled next
}

// Prefetch the chunk's aux operand (residual for EPI_FWD, act'-saved for EPI_DGRAD).
template <int EPI>
__device__ __forceinline__ void epilogue_aux(const EpiParams& ep, int row, int col0, int M, int N,
                                             float (&aux)[32]) {
  const bool need = (EPI == EPI_FWD && ep.aux != nullptr) ||
                    (EPI == EPI_DGRAD && ep.act != GPP_ACT_NONE);
  if (!need || row >= M || col0 >= N) return;
  const int n_valid = N - col0 < 32 ? N - col0 : 32;
  const bf16* p = static_cast<const bf16*>(ep.aux) + static_cast<int64_t>(row) * ep.ldaux + col0;
  load_bf16x32(p, n_valid == 32 && al16(p), n_valid, aux);
}

template <int BN, int STAGES, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tma_a,
                   const __grid_constant__ CUtensorMap tma_b, EpiParams ep, int M, int N, int K,
                   int k_splits, BatchSpec bs) {
  constexpr int A_BYTES = BM * BK * 2;
  constexpr int B_BYTES = BN * BK * 2;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = BN;  // power of two >= 32
  constexpr uint32_t IDESC = idesc_bf16<BN, A_MN, B_MN>();

  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned via an offset (not pointer-integer casts) so smem accesses stay STS/LDS
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* accum_bar = empty_bar + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum_bar + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_blocks = (N + BN - 1) / BN;
  const int m_blocks = (M + BM - 1) / BM;
  const int per_batch = m_blocks * n_blocks * k_splits;
  const int z = static_cast<int>(blockIdx.x) / per_batch;
  const int z_hi = z / bs.nlo, z_lo = z % bs.nlo;
  const int unit = static_cast<int>(blockIdx.x) % per_batch;
  const int tile = unit / k_splits;
  const int split = unit % k_splits;
  const int am_off = bs.a_m0 + z_hi * bs.a_m_hi + z_lo * bs.a_m_lo;
  const int ak_off = bs.a_k0 + z_hi * bs.a_k_hi + z_lo * bs.a_k_lo;
  const int bn_off = bs.b_n0 + z_hi * bs.b_n_hi + z_lo * bs.b_n_lo;
  const int bk_off = bs.b_k0 + z_hi * bs.b_k_hi + z_lo * bs.b_k_lo;
  const int m_blk = tile / n_blocks;
  const int n_blk = tile % n_blocks;
  const int kb_per = ((K + BK - 1) / BK + k_splits - 1) / k_splits;
  const int kb0 = split * kb_per;
  const int num_kb = min((K + BK - 1) / BK, kb0 + kb_per) - kb0;
  EpiParams epu = ep;
  if (k_splits > 1) epu.out = reinterpret_cast<float*>(ep.out) + split * ep.split_stride;
  if (bs.nbatch > 1 || bs.c0 != 0) {
    const int64_t c_off = bs.c0 + z_hi * bs.c_hi + z_lo * bs.c_lo;
    const int esz = (EPI == EPI_F32 || EPI == EPI_SGD) ? 4 : 2;
    epu.out = static_cast<char*>(epu.out) + c_off * esz;
    if (ep.aux) epu.aux = static_cast<const char*>(ep.aux) + c_off * 2;
    if (ep.pre) epu.pre = static_cast<char*>(ep.pre) + c_off * 2;
  }

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(accum_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // prologue above overlaps the previous kernel's tail
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&empty_bar[s], ph ^ 1);
        uint8_t* a_dst = smem + s * STAGE_BYTES;
        uint8_t* b_dst = a_dst + A_BYTES;
        mbar_expect_tx(&full_bar[s], STAGE_BYTES);
        if constexpr (!A_MN) {
          tma_load_2d(a_dst, &tma_a, &full_bar[s], (kb0 + kb) * BK + ak_off, m_blk * BM + am_off);
        } else {
#pragma unroll
          for (int c = 0; c < BM / 64; ++c)
            tma_load_2d(a_dst + c * 8192, &tma_a, &full_bar[s], m_blk * BM + c * 64 + am_off, (kb0 + kb) * BK + ak_off);
        }
        if constexpr (!B_MN) {
          tma_load_2d(b_dst, &tma_b, &full_bar[s], (kb0 + kb) * BK + bk_off, n_blk * BN + bn_off);
        } else {
#pragma unroll
          for (int c = 0; c < BN / 64; ++c)
            tma_load_2d(b_dst + c * 8192, &tma_b, &full_bar[s], n_blk * BN + c * 64 + bn_off, (kb0 + kb) * BK + bk_off);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 1) l2_prefetch_share(ep, static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x));
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&full_bar[s], ph);
        tc_fence_after();
        const uint32_t a_base = smem_u32(smem + s * STAGE_BYTES);
        const uint32_t b_base = a_base + A_BYTES;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          // K-major: advance 16 elements (32 B) inside the 128 B swizzle row.
          // MN-major: advance 16 k-rows of 128 B.
          const uint32_t a_off = A_MN ? k * 2048 : k * 32;
          const uint32_t b_off = B_MN ? k * 2048 : k * 32;
          const uint64_t adesc = sdesc_sw128(a_base + a_off, A_MN ? 8192 : 16, 1024);
          const uint64_t bdesc = sdesc_sw128(b_base + b_off, B_MN ? 8192 : 16, 1024);
          umma_bf16(tmem_base, adesc, bdesc, IDESC, (kb | k) != 0 ? 1u : 0u);
        }
        umma_commit(&empty_bar[s]);
      }
      umma_commit(accum_bar);
    }
  } else {
    // ---------------- epilogue (warps 2..5) ----------------
    mbar_wait(accum_bar, 0);
    tc_fence_after();
    const int q = warp & 3;  // TMEM lane quarter accessible to this warp
    const int row = m_blk * BM + q * 32 + lane;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      uint32_t v[32];
      float aux[32];
      epilogue_aux<EPI>(epu, row, n_blk * BN + c * 32, M, N, aux);
      tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + c * 32, v);
      epilogue_chunk<EPI>(epu, v, aux, row, n_blk * BN + c * 32, M, N);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS)
                 : "memory");
  }
}


// ---- aux tiles by TMA (bf16 epilogues with a residual / act'-saved operand) ----
#define AUX_TMA_EPI(E) ((E) == EPI_FWD || (E) == EPI_DGRAD)

// this lane's row of a 64B-swizzled [32 x 32] bf16 tile -> 32 floats (conflict-free)
__device__ __forceinline__ void read_aux_tile(const uint8_t* tile, int lane, float (&a)[32]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint4 r = *reinterpret_cast<const uint4*>(tile + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4));
    const uint32_t* u = reinterpret_cast<const uint32_t*>(&r);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u[t]));
      a[8 * j + 2 * t] = x.x;
      a[8 * j + 2 * t + 1] = x.y;
    }
  }
}

// ------------------------------------------------------------------------
// Persistent CTA-pair GEMM: cluster (2,1,1), tcgen05.mma.cta_group::2 with
// M = 256 (128 rows per CTA) x N = BN, TMEM accumulators double-buffered
// (2 x BN columns) so the epilogue of tile t overlaps the MMAs of tile t+1.
//   CTA rank r loads A rows [m0 + 128 r, +128) and B rows [n0 + r BN/2, +BN/2);
//   both CTAs' TMA bytes complete on the leader's full barrier; the leader's
//   single MMA thread commits (multicast) to both CTAs' empty / accum-full
//   barriers; all 8 epilogue warps arrive on the leader's accum-empty barrier.
// ------------------------------------------------------------------------
// wgrad epilogues (A = dy^T, MN-major) carry one more warp: the bias-gradient column sums
template <int EPI, bool A_MN>
constexpr bool pair_colsum_epi() { return (EPI == EPI_F32 || EPI == EPI_SGD) && A_MN; }

__device__ __forceinline__ void mbar_arrive_local(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int BN, int STAGES, bool A_MN, bool B_MN, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PAIR_THREADS + 32, 1)
    gemm_tc_pair_kernel(const __grid_constant__ CUtensorMap tma_a,
                        const __grid_constant__ CUtensorMap tma_b, EpiParams ep, int M, int N,
                        int K, int k_splits, int m_fast, const __grid_constant__ CUtensorMap tma_aux,
                        int aux_tma) {
  constexpr int A_BYTES = BM * BK * 2;            // 16 KB: this CTA's 128 rows of A
  constexpr int B_BYTES = (BN / 2) * BK * 2;      // this CTA's BN/2 rows of B
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = 2 * BN;          // two accumulators
  constexpr uint32_t IDESC = idesc_bf16<BN, A_MN, B_MN, 2 * BM>();

  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned via an offset (not pointer-integer casts) so smem accesses stay STS/LDS
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;       // [2]
  uint64_t* tempty_bar = tfull_bar + 2;           // [2] (leader's copy is the live one)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  uint64_t* cs_bar = tempty_bar + 3;              // [STAGES] peer CTA: "leader saw this stage full"
  float* epi_stage = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256);  // per warp 32 x 36 (x2 SGD)
  // bf16 epilogues: per-warp double-buffered 64B-swizzled 32 x 32 aux tiles filled by TMA
  uint64_t* aux_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES + 512);
  uint8_t* aux_tiles = smem + STAGES * STAGE_BYTES + 1024;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = (rank == 0);
  const int cluster_id = blockIdx.x >> 1;
  const int num_clusters = gridDim.x >> 1;
  const int m_tiles = (M + 2 * BM - 1) / (2 * BM);
  const int n_tiles = (N + BN - 1) / BN;
  const int num_units = m_tiles * n_tiles * k_splits;   // (tile, K-split) work units
  const int kb_total = (K + BK - 1) / BK;
  const int kb_per = (kb_total + k_splits - 1) / k_splits;
  // fused bias gradient: a 12th warp per CTA sums this CTA's A tile of every stage over K
  // (both CTAs: the leader's warp tells the peer's when the pair's TMA bytes landed) and
  // releases the stage as a second arrival on its empty barrier
  const bool cs = pair_colsum_epi<EPI, A_MN>() && ep.colsum != nullptr && k_splits == 1;
  static_assert(3 * STAGES + 5 <= 32, "barrier block overflows its 256 bytes");

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], cs ? 2 : 1);
      mbar_init(&cs_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 2 * PAIR_EPI_WARPS);
    }
    if (AUX_TMA_EPI(EPI))
      for (int i = 0; i < 2 * PAIR_EPI_WARPS; ++i) mbar_init(&aux_bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // prologue above overlaps the previous kernel's tail
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs) ----------------
      uint32_t it = 0;
      for (int u = cluster_id; u < num_units; u += num_clusters) {
        const int tile = u / k_splits, kb0 = (u % k_splits) * kb_per;
        const int num_kb = min(kb_total, kb0 + kb_per) - kb0;
        // raster: concurrently running pairs share the larger operand's tiles through L2
        const int m_blk = m_fast ? tile % m_tiles : tile / n_tiles;
        const int n_blk = m_fast ? tile / m_tiles : tile % n_tiles;
        const int a_row = m_blk * 2 * BM + static_cast<int>(rank) * BM;
        const int b_row = n_blk * BN + static_cast<int>(rank) * (BN / 2);
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty_bar[s], ph ^ 1);
          uint8_t* a_dst = smem + s * STAGE_BYTES;
          uint8_t* b_dst = a_dst + A_BYTES;
          if (leader) mbar_expect_tx(&full_bar[s], 2 * STAGE_BYTES);
          if constexpr (!A_MN) {
            tma_load_2d_pair(a_dst, &tma_a, &full_bar[s], (kb0 + kb) * BK, a_row);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c)
              tma_load_2d_pair(a_dst + c * 8192, &tma_a, &full_bar[s], a_row + c * 64, (kb0 + kb) * BK);
          }
          if constexpr (!B_MN) {
            tma_load_2d_pair(b_dst, &tma_b, &full_bar[s], (kb0 + kb) * BK, b_row);
          } else {
#pragma unroll
            for (int c = 0; c < (BN / 2) / 64; ++c)
              tma_load_2d_pair(b_dst + c * 8192, &tma_b, &full_bar[s], b_row + c * 64, (kb0 + kb) * BK);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 1) l2_prefetch_share(ep, static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x));
    if (leader && lane == 0) {
      // ---------------- MMA issuer (leader CTA only) ----------------
      uint32_t it = 0, lt = 0;
      for (int u = cluster_id; u < num_units; u += num_clusters, ++lt) {
        const int kb0 = (u % k_splits) * kb_per;
        const int num_kb = min(kb_total, kb0 + kb_per) - kb0;
        const uint32_t acc = lt & 1, aph = (lt >> 1) & 1;
        mbar_wait_cluster(&tempty_bar[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full_bar[s], ph);
          tc_fence_after();
          const uint32_t a_base = smem_u32(smem + s * STAGE_BYTES);
          const uint32_t b_base = a_base + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint32_t a_off = A_MN ? k * 2048 : k * 32;
            const uint32_t b_off = B_MN ? k * 2048 : k * 32;
            const uint64_t adesc = sdesc_sw128(a_base + a_off, A_MN ? 8192 : 16, 1024);
            const uint64_t bdesc = sdesc_sw128(b_base + b_off, B_MN ? 8192 : 16, 1024);
            umma_bf16_pair(d_tmem, adesc, bdesc, IDESC, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit_pair(&empty_bar[s], 0x3);
        }
        umma_commit_pair(&tfull_bar[acc], 0x3);
      }
    }
  } else if (warp >= 2 + PAIR_EPI_WARPS) {
    // ---------------- bias-gradient column sums (wgrad: A = dy^T, MN-major) ----------------
    // A stage holds this CTA's 128 m x 64 k as two 8 KB chunks of 64 k-rows x 64 m (128B
    // swizzle); lane = (chunk, 16-byte unit, half): 4 m columns, summed over the 64 rows.
    if (cs) {
      const uint32_t peer_cs0 = mapa_shared(smem_u32(&cs_bar[0]), 1);
      const int ch = lane >> 4, j = (lane & 15) >> 1, half = lane & 1;
      uint32_t it = 0;
      for (int u = cluster_id; u < num_units; u += num_clusters) {
        const int m_blk = m_fast ? u % m_tiles : u / n_tiles;
        const int n_blk = m_fast ? u / m_tiles : u % n_tiles;
        const bool mine = n_blk == 0;  // one tile column sums each m block
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
        for (int kb = 0; kb < kb_total; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          // default (.release.cta) remote arrive + CTA-scope wait: a .release.cluster arrive
          // costs a cluster-scope fence per stage (measured: 4x slower wgrad); the peer's A tile
          // was written by the pair TMA before the leader's full barrier could complete
          if (leader) {
            mbar_wait(&full_bar[s], ph);
            if (lane == 0) mbar_arrive_cluster(peer_cs0 + s * 8);
          } else {
            mbar_wait(&cs_bar[s], ph);
          }
          if (mine) {
            const uint8_t* base = smem + s * STAGE_BYTES + ch * 8192 + half * 8;
#pragma unroll 16
            for (int r = 0; r < 64; ++r) {
              const uint2 v = *reinterpret_cast<const uint2*>(base + r * 128 + ((j ^ (r & 7)) << 4));
              const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.x));
              const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v.y));
              a0 += lo.x;
              a1 += lo.y;
              a2 += hi.x;
              a3 += hi.y;
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive_local(&empty_bar[s]);
        }
        if (mine) {
          const int m = m_blk * 2 * BM + static_cast<int>(rank) * BM + ch * 64 + j * 8 + half * 4;
          const float sums[4] = {a0, a1, a2, a3};
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (m + t < M) ep.colsum[m + t] = ep.colsum_acc ? ep.colsum[m + t] + sums[t] : sums[t];
        }
      }
    }
  } else {
    // ---------------- epilogue (warps 2..9 of both CTAs) ----------------
    const int q = warp & 3;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty_bar[0]), 0);
    uint32_t lt = 0, aux_it = 0;
    for (int u = cluster_id; u < num_units; u += num_clusters, ++lt) {
      const int tile = u / k_splits;
      EpiParams epu = ep;
      if (k_splits > 1) epu.out = reinterpret_cast<float*>(ep.out) + (u % k_splits) * ep.split_stride;
      const uint32_t acc = lt & 1, aph = (lt >> 1) & 1;
      const int m_blk = m_fast ? tile % m_tiles : tile / n_tiles;
      const int n_blk = m_fast ? tile / m_tiles : tile % n_tiles;
      const int row0 = m_blk * 2 * BM + static_cast<int>(rank) * BM + q * 32;
      const int row = row0 + lane;
      const int group = (warp - 2) / 4;  // epilogue warpgroup: takes every other 32-col chunk
      constexpr int GSTEP = PAIR_EPI_WARPS / 4;
      constexpr int CH = BN / 32 / GSTEP;  // chunks per warp per tile (even)
      if constexpr (EPI == EPI_SGD) {
        if (sgd_fast_ok(epu, N) && k_splits == 1) {
          // SGD_DEPTH master chunks in flight per warp, issued before the accumulator is ready
          float* b0 = epi_stage + (warp - 2) * SGD_DEPTH * 32 * STAGE_LD;
          auto col_of = [&](int p) { return n_blk * BN + (group + p * GSTEP) * 32; };
#pragma unroll
          for (int p = 0; p < SGD_DEPTH && p < CH; ++p) sgd_fast_issue(epu, b0 + p * 32 * STAGE_LD, row0, col_of(p), M, N, lane);
          mbar_wait(&tfull_bar[acc], aph);
          tc_fence_after();
#pragma unroll
          for (int p = 0; p < CH; ++p) {
            float* buf = b0 + (p % SGD_DEPTH) * 32 * STAGE_LD;
            uint32_t v[32];
            tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + (group + p * GSTEP) * 32, v);
            // groups committed after chunk p's: min(SGD_DEPTH, CH - p) - 1
            const int after = (CH - p < SGD_DEPTH ? CH - p : SGD_DEPTH) - 1;
            if (after >= 2) cp_async_wait<2>(); else if (after == 1) cp_async_wait<1>(); else cp_async_wait<0>();
            sgd_fast_update(epu, v, buf, row0, col_of(p), M, N, lane);
            if (p + SGD_DEPTH < CH) sgd_fast_issue(epu, buf, row0, col_of(p + SGD_DEPTH), M, N, lane);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tempty_leader0 + acc * 8);
          continue;
        }
      }
      // The aux tile (residual / act'-saved) of a bf16 epilogue arrives by TMA, 32 x 32 per
      // chunk, one chunk ahead, into this warp's double buffer (row-per-lane global loads
      // touched 32 lines per instruction and exposed a DRAM latency per chunk).
      uint8_t* my_aux = aux_tiles + (warp - 2) * 4096;
      uint64_t* my_bar = aux_bar + 2 * (warp - 2);
      auto issue_aux = [&](int c) {
        if (lane == 0) {
          const uint32_t b = aux_it & 1;
          mbar_expect_tx(&my_bar[b], 2048);
          tma_load_2d(my_aux + b * 2048, &tma_aux, &my_bar[b], n_blk * BN + c * 32, row0);
        }
      };
      if (AUX_TMA_EPI(EPI) && aux_tma) issue_aux(group);
      // bias of this warp's CH chunks -> the unused second half of its aux tile, loaded before
      // the accumulator wait (a per-chunk global load exposed its latency in every chunk)
      const float* sbias = nullptr;
      if constexpr (EPI == EPI_FWD) {
        if (!aux_tma && ep.bias != nullptr) {
          static_assert(CH * 32 <= 32 * 4 * 4, "one float4 per lane");
          float* sb = reinterpret_cast<float*>(my_aux + 2048);
          const int p = lane >> 3;
          if (p < CH) {
            const int col = n_blk * BN + (group + p * GSTEP) * 32 + (lane & 7) * 4;
            float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
            if (col + 4 <= N && al16(ep.bias + col)) {
              b = __ldg(reinterpret_cast<const float4*>(ep.bias + col));
            } else {
              if (col < N) b.x = __ldg(ep.bias + col);
              if (col + 1 < N) b.y = __ldg(ep.bias + col + 1);
              if (col + 2 < N) b.z = __ldg(ep.bias + col + 2);
              if (col + 3 < N) b.w = __ldg(ep.bias + col + 3);
            }
            *reinterpret_cast<float4*>(sb + p * 32 + (lane & 7) * 4) = b;
          }
          __syncwarp();
          sbias = sb;
        }
      }
      mbar_wait(&tfull_bar[acc], aph);
      tc_fence_after();
#pragma unroll 1
      for (int c = group; c < BN / 32; c += GSTEP) {
        uint32_t v[32];
        if constexpr (EPI == EPI_F32 || EPI == EPI_SGD) {
          tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + c * 32, v);
          epilogue_f32_coalesced<EPI>(epu, v, epi_stage + (warp - 2) * 32 * STAGE_LD, row0,
                                      n_blk * BN + c * 32, M, N, lane);
        } else {
          float aux[32];
          uint8_t* stage = nullptr;  // the chunk's store staging tile (2 KB of this warp's aux pair)
          if (AUX_TMA_EPI(EPI) && aux_tma) {
            const uint32_t b = aux_it & 1, ph = (aux_it >> 1) & 1;
            ++aux_it;
            if (c + GSTEP < BN / 32) issue_aux(c + GSTEP);  // into the other buffer (consumed)
            mbar_wait(&my_bar[b], ph);
            read_aux_tile(my_aux + b * 2048, lane, aux);
            __syncwarp();  // every lane done with buffer b before it is reused / refilled
            stage = my_aux + b * 2048;  // free until the next chunk's TMA refills it
          } else {
            epilogue_aux<EPI>(epu, row, n_blk * BN + c * 32, M, N, aux);
            if (AUX_TMA_EPI(EPI)) stage = my_aux;  // aux tiles unused by this launch
          }
          tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + c * 32, v);
          epilogue_chunk<EPI>(epu, v, aux, row, n_blk * BN + c * 32, M, N, stage, lane,
                              sbias != nullptr ? sbias + ((c - group) / GSTEP) * 32 : nullptr);
          if (stage != nullptr) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader0 + acc * 8);
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS)
                 : "memory");
  }
}

// ------------------------------------------------------------------------
// Host side: TMA descriptors (cached) and dispatch.
// ------------------------------------------------------------------------

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

struct MapKey {
  const void* ptr;
  int64_t inner, outer, ld;
  int box_inner, box_outer, swz;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && inner == o.inner && outer == o.outer && ld == o.ld &&
           box_inner == o.box_inner && box_outer == o.box_outer && swz == o.swz;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = std::hash<const void*>()(k.ptr);
    h ^= std::hash<int64_t>()(k.inner * 1315423911LL + k.outer) + 0x9e3779b9 + (h << 6) + (h >> 2);
    h ^= std::hash<int64_t>()(k.ld * 31 + k.box_inner * 7 + k.box_outer * 3 + k.swz) + (h << 6) + (h >> 2);
    return h;
  }
};

// 2-D bf16 tensor map over a row-major buffer: `outer` rows of `inner` elements, row pitch ld.
static int make_map(CUtensorMap* out, const void* ptr, int64_t inner, int64_t outer, int64_t ld,
                    int box_inner, int box_outer, int swizzle_bytes = 128) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  MapKey key{ptr, inner, outer, ld, box_inner, box_outer, swizzle_bytes};
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
      *out = it->second;
      return GPP_OK;
    }
  }
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled entry point unavailable");
    return GPP_ERR_DRIVER;
  }
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed with code " + std::to_string(static_cast<int>(r)));
    return GPP_ERR_DRIVER;
  }
  std::lock_guard<std::mutex> g(mu);
  if (cache.size() > 65536) cache.clear();
  cache.emplace(key, *out);
  return GPP_OK;
}

int make_map_bf16(CUtensorMap* out, const void* ptr, int64_t inner, int64_t outer, int64_t ld, int box_inner,
                  int box_outer) {
  return make_map(out, ptr, inner, outer, ld, box_inner, box_outer);
}

template <int BN, int STAGES, bool A_MN, bool B_MN, int EPI>
static int launch_tc(const void* a, int64_t lda, const void* b, int64_t ldb, const EpiParams& ep,
                     int64_t M, int64_t N, int64_t K, int k_splits, cudaStream_t stream,
                     const BatchSpec& bs = BatchSpec(), int64_t a_inner = -1, int64_t a_outer = -1,
                     int64_t b_inner = -1, int64_t b_outer = -1) {
  CUtensorMap ma, mb;
  int rc;
  // K-major operand: inner = K, outer = rows;  MN-major: inner = rows, outer = K.
  // Batched calls pass the full operand extents (a_inner/outer...) so per-batch offsets
  // stay inside one descriptor.
  if (!A_MN) rc = make_map(&ma, a, a_inner > 0 ? a_inner : K, a_outer > 0 ? a_outer : M, lda, BK, BM);
  else rc = make_map(&ma, a, a_inner > 0 ? a_inner : M, a_outer > 0 ? a_outer : K, lda, 64, BK);
  if (rc) return rc;
  if (!B_MN) rc = make_map(&mb, b, b_inner > 0 ? b_inner : K, b_outer > 0 ? b_outer : N, ldb, BK, BN);
  else rc = make_map(&mb, b, b_inner > 0 ? b_inner : N, b_outer > 0 ? b_outer : K, ldb, 64, BK);
  if (rc) return rc;

  constexpr int STAGE_BYTES = (BM + BN) * BK * 2;
  constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_tc_kernel<BN, STAGES, A_MN, B_MN, EPI>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    attr_set = true;
  }
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  cudaError_t e = launch_pdl(gemm_tc_kernel<BN, STAGES, A_MN, B_MN, EPI>,
                             dim3(static_cast<unsigned>(tiles * k_splits * bs.nbatch)), dim3(NUM_THREADS), SMEM,
                             stream, ma, mb, ep, static_cast<int>(M), static_cast<int>(N), static_cast<int>(K),
                             k_splits, bs);
  if (e != cudaSuccess) {
    set_error(std::string("gemm_tc launch: ") + cudaGetErrorString(e));
    return GPP_ERR_CUDA;
  }
  count_launch();
  return GPP_OK;
}


static bool aux_tma_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("GPP_AUX_TMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

static bool pair_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("GPP_GEMM_PAIR");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static int max_splits_env() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("GPP_GEMM_MAX_SPLITS");
    v = e ? atoi(e) : 16;
    if (v < 1) v = 1;
  }
  return v;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, int STAGES, bool A_MN, bool B_MN, int EPI>
static int launch_tc_pair(const void* a, int64_t lda, const void* b, int64_t ldb,
                          const EpiParams& ep, int64_t M, int64_t N, int64_t K, int k_splits,
                          cudaStream_t stream) {
  CUtensorMap ma, mb;
  int rc;
  if (!A_MN) rc = make_map(&ma, a, K, M, lda, BK, BM);
  else rc = make_map(&ma, a, M, K, lda, 64, BK);
  if (rc) return rc;
  if (!B_MN) rc = make_map(&mb, b, K, N, ldb, BK, BN / 2);
  else rc = make_map(&mb, b, N, K, ldb, 64, BK);
  if (rc) return rc;
  constexpr int STAGE_BYTES = (BM + BN / 2) * BK * 2;
  // fp32 epilogues stage through smem (fused SGD double-buffers its master chunks);
  // the bf16 epilogues write straight from registers and give that space to the ring
  constexpr int EPI_BUFS = EPI == EPI_SGD ? SGD_DEPTH : (EPI == EPI_F32 ? 1 : 0);
  constexpr int SMEM = AUX_TMA_EPI(EPI) ? STAGES * STAGE_BYTES + 1024 + 1024 + PAIR_EPI_WARPS * 4096
                                        : STAGES * STAGE_BYTES + 1024 + 256 + PAIR_EPI_WARPS * 32 * STAGE_LD * 4 * EPI_BUFS;
  CUtensorMap mx = ma;
  int aux_tma = 0;
  if constexpr (AUX_TMA_EPI(EPI)) {
    const bool need = (EPI == EPI_FWD && ep.aux != nullptr) || (EPI == EPI_DGRAD && ep.act != GPP_ACT_NONE);
    aux_tma = need && k_splits == 1 && (reinterpret_cast<uintptr_t>(ep.aux) & 15) == 0 && ep.ldaux % 8 == 0 &&
              aux_tma_enabled();
    if (aux_tma && (rc = make_map(&mx, ep.aux, N, M, ep.ldaux, 32, 32, 64))) return rc;
  }
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_tc_pair_kernel<BN, STAGES, A_MN, B_MN, EPI>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    attr_set = true;
  }
  const int64_t units = ((M + 2 * BM - 1) / (2 * BM)) * ((N + BN - 1) / BN) * k_splits;
  int64_t clusters = num_sms() / 2;
  if (units < clusters) clusters = units;
  constexpr int THREADS = PAIR_THREADS + (pair_colsum_epi<EPI, A_MN>() ? 32 : 0);
  cudaError_t e = launch_pdl(gemm_tc_pair_kernel<BN, STAGES, A_MN, B_MN, EPI>, dim3(static_cast<unsigned>(2 * clusters)),
                             dim3(THREADS), SMEM, stream, ma, mb, ep, static_cast<int>(M), static_cast<int>(N),
                             static_cast<int>(K), k_splits, M < N ? 1 : 0, mx, aux_tma);
  if (e != cudaSuccess) {
    set_error(std::string("gemm_tc_pair launch: ") + cudaGetErrorString(e));
    return GPP_ERR_CUDA;
  }
  count_launch();
  return GPP_OK;
}

// ---- split-K: fp32 partials in a per-device workspace, then one reduce + epilogue ----

static float* splitk_workspace(size_t floats, cudaStream_t stream) {
  static float* bufs[64] = {nullptr};
  static size_t caps[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (caps[dev] >= floats) return bufs[dev];
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &st);
  if (st != cudaStreamCaptureStatusNone) {
    set_error("split-K workspace must be sized before CUDA-graph capture (run one eager step first)");
    return nullptr;
  }
  size_t want = floats < (size_t(16) << 20) ? (size_t(16) << 20) : floats;
  // the old buffer is retired, not freed: graphs captured earlier may still reference it
  if (cudaMalloc(&bufs[dev], want * sizeof(float)) != cudaSuccess) {
    bufs[dev] = nullptr;
    caps[dev] = 0;
    set_error("split-K workspace allocation failed");
    return nullptr;
  }
  caps[dev] = want;
  return bufs[dev];
}

template <int EPI>
__device__ __forceinline__ void epi_elem(const EpiParams& ep, float acc, int64_t row, int64_t col) {
  float v = acc * ep.alpha;
  if constexpr (EPI == EPI_FWD) {
    if (ep.bias) v += ep.bias[col];
    if (ep.pre) static_cast<bf16*>(ep.pre)[row * ep.ldpre + col] = __float2bfloat16_rn(v);
    v = act_fwd(v, ep.act);
    if (ep.aux) v += __bfloat162float(static_cast<const bf16*>(ep.aux)[row * ep.ldaux + col]);
    static_cast<bf16*>(ep.out)[row * ep.ldo + col] = __float2bfloat16_rn(v);
  } else if constexpr (EPI == EPI_DGRAD) {
    if (ep.act != GPP_ACT_NONE)
      v *= act_bwd(__bfloat162float(static_cast<const bf16*>(ep.aux)[row * ep.ldaux + col]), ep.act);
    static_cast<bf16*>(ep.out)[row * ep.ldo + col] = __float2bfloat16_rn(v);
  } else if constexpr (EPI == EPI_F32) {
    float* o = static_cast<float*>(ep.out) + row * ep.ldo + col;
    *o = ep.beta != 0.f ? v + ep.beta * *o : v;
  } else if constexpr (EPI == EPI_BF16) {
    bf16* o = static_cast<bf16*>(ep.out) + row * ep.ldo + col;
    *o = __float2bfloat16_rn(ep.beta != 0.f ? v + ep.beta * __bfloat162float(*o) : v);
  } else {  // EPI_SGD
    float* g = ep.grad + row * ep.ldgrad + col;
    const float gv = v + (ep.beta != 0.f ? *g : 0.f);
    if (ep.store_grad) *g = gv;
    float* m = static_cast<float*>(ep.out) + row * ep.ldo + col;
    const float mv = *m - ep.lr * gv;
    *m = mv;
    static_cast<bf16*>(ep.pre)[row * ep.ldpre + col] = __float2bfloat16_rn(mv);
  }
}

template <int EPI>
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float* __restrict__ ws, int splits,
                                                            int64_t stride, EpiParams ep, int M,
                                                            int N) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = static_cast<int64_t>(M) * N;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float acc = 0.f;
    for (int sp = 0; sp < splits; ++sp) acc += ws[sp * stride + i];
    epi_elem<EPI>(ep, acc, i / N, i % N);
  }
}

// How many K-slices: fill idle SMs when the tile count is small, keep >= 2 k-blocks each.
static int choose_splits(int64_t tiles, int64_t slots, int64_t num_kb) {
  if (tiles * 2 > slots) return 1;
  int64_t s = slots / tiles;
  if (s > num_kb / 2) s = num_kb / 2;
  if (s > max_splits_env()) s = max_splits_env();
  if (s < 1) s = 1;
  // every split must own >= 1 k-block: kernels split K as ceil(num_kb / s) blocks each, so
  // e.g. 64 blocks over 9 splits would leave the 9th empty (an uncommitted accumulator)
  const int64_t per = (num_kb + s - 1) / s;
  return static_cast<int>((num_kb + per - 1) / per);
}

template <bool A_MN, bool B_MN, int EPI>
static int dispatch_bn(const void* a, int64_t lda, const void* b, int64_t ldb,
                       const EpiParams& ep, int64_t M, int64_t N, int64_t K,
                       cudaStream_t stream) {
  const int64_t num_kb = (K + BK - 1) / BK;
  const bool pair = M > BM && pair_enabled();
  int bn;
  int64_t tiles, slots;
  if (pair) {
    // CTA-pair 256 x BN tiles; BN=128 when 256-wide tiles leave most pairs idle.
    const int64_t pairs256 = ((M + 255) / 256) * ((N + 255) / 256);
    bn = (N > 128 && pairs256 >= 48) ? 256 : 128;
    // small output, long K: split-K fills the GPU anyway, and 256-wide tiles cut the
    // L2 -> SM operand traffic per FLOP by a third (the CANDLE tail: 1024 x 1024 x 28672)
    if (bn == 128 && N > 128 && pairs256 * std::min<int64_t>(max_splits_env(), num_kb / 2) >= 48) bn = 256;
    tiles = ((M + 255) / 256) * ((N + bn - 1) / bn);
    slots = num_sms() / 2;
  } else {
    const int64_t tiles256 = ((M + BM - 1) / BM) * ((N + 255) / 256);
    bn = (N > 128 && tiles256 >= 96) ? 256 : 128;
    tiles = ((M + BM - 1) / BM) * ((N + bn - 1) / bn);
    slots = num_sms();
  }
  const int splits = choose_splits(tiles, slots, num_kb);
  // bias gradient: fused into the pair kernel's A-tile reads when it runs unsplit; else
  // one column-sum kernel over A ([K, M] row-major for the MN-major dy^T) after the GEMM
  // Off by default (GPP_FUSED_COLSUM=1 enables it): measured at the MMT shapes the column-sum
  // warp shares its SM sub-partition with the SGD epilogue warps and stretches the tiles it
  // sums (wgrad+SGD 3072x1024x8192: 128 us fused vs 54 + 15 us GEMM + column-sum kernel;
  // CANDLE 4096^2 x 1024: 54 vs 49 + 5 us) -- tools/bench_wgrad_sgd.py, DESIGN.md section 7b
  static const bool cs_enabled = [] { const char* e = std::getenv("GPP_FUSED_COLSUM"); return e && e[0] == '1'; }();
  const bool fuse_cs = cs_enabled && ep.colsum != nullptr && pair && splits == 1 && pair_colsum_epi<EPI, A_MN>();
  if (ep.colsum != nullptr && !fuse_cs) {
    GPP_ARG_CHECK(A_MN, "fused column sum needs the MN-major (wgrad) A operand");
    EpiParams e2 = ep;
    e2.colsum = nullptr;
    int rc = dispatch_bn<A_MN, B_MN, EPI>(a, lda, b, ldb, e2, M, N, K, stream);
    if (rc) return rc;
    return gpp_colsum(ep.colsum, a, lda, K, M, ep.colsum_acc, GPP_BF16, stream);
  }

  auto run = [&](auto epi_tag, const EpiParams& e, int ks) -> int {
    constexpr int E = decltype(epi_tag)::value;
    if (pair) {
      // EPI_SGD gives one smem stage to its double-buffered master chunks
      constexpr int S256 = E == EPI_SGD ? SGD_STAGES256 : (E == EPI_F32 ? 5 : 6);
      constexpr int S128 = E == EPI_SGD ? (SGD_DEPTH >= 3 ? 4 : 6) : (E == EPI_F32 ? 7 : 8);
      if (bn == 256) return launch_tc_pair<256, S256, A_MN, B_MN, E>(a, lda, b, ldb, e, M, N, K, ks, stream);
      return launch_tc_pair<128, S128, A_MN, B_MN, E>(a, lda, b, ldb, e, M, N, K, ks, stream);
    }
    if (bn == 256) return launch_tc<256, 4, A_MN, B_MN, E>(a, lda, b, ldb, e, M, N, K, ks, stream);
    return launch_tc<128, 6, A_MN, B_MN, E>(a, lda, b, ldb, e, M, N, K, ks, stream);
  };
  if (splits == 1) return run(std::integral_constant<int, EPI>{}, ep, 1);

  float* ws = splitk_workspace(static_cast<size_t>(splits) * M * N, stream);
  if (!ws) return GPP_ERR_CUDA;
  EpiParams part{};
  part.out = ws;
  part.ldo = N;
  part.alpha = 1.f;
  part.beta = 0.f;
  part.split_stride = M * N;
  int rc = run(std::integral_constant<int, EPI_F32>{}, part, splits);
  if (rc) return rc;
  const int64_t total = M * N;
  int64_t grid = (total + 255) / 256;
  if (grid > 148 * 8) grid = 148 * 8;
  cudaError_t e = launch_pdl(splitk_reduce_kernel<EPI>, dim3(static_cast<unsigned>(grid)), dim3(256), 0, stream, ws,
                             splits, M * N, ep, static_cast<int>(M), static_cast<int>(N));
  if (e != cudaSuccess) {
    set_error(std::string("splitk_reduce launch: ") + cudaGetErrorString(e));
    return GPP_ERR_CUDA;
  }
  count_launch();
  return GPP_OK;
}

template <int EPI>
static int dispatch_layout(const void* a, int64_t lda, int a_mn, const void* b, int64_t ldb,
                           int b_mn, const EpiParams& ep, int64_t M, int64_t N, int64_t K,
                           cudaStream_t stream) {
  if (!a_mn && !b_mn) return dispatch_bn<false, false, EPI>(a, lda, b, ldb, ep, M, N, K, stream);
  if (!a_mn && b_mn) return dispatch_bn<false, true, EPI>(a, lda, b, ldb, ep, M, N, K, stream);
  if (a_mn && !b_mn) return dispatch_bn<true, false, EPI>(a, lda, b, ldb, ep, M, N, K, stream);
  return dispatch_bn<true, true, EPI>(a, lda, b, ldb, ep, M, N, K, stream);
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int check_operands(const void* a, int64_t lda, int a_mn, const void* b, int64_t ldb, int b_mn,
                   int64_t M, int64_t N, int64_t K) {
  GPP_ARG_CHECK(M > 0 && N > 0 && K > 0, "M, N, K must be positive");
  GPP_ARG_CHECK(M < (1LL << 31) && N < (1LL << 31) && K < (1LL << 31), "dimension too large");
  GPP_ARG_CHECK(aligned16(a) && aligned16(b), "TMA operands must be 16-byte aligned");
  GPP_ARG_CHECK(lda % 8 == 0 && ldb % 8 == 0, "bf16 leading dims must be multiples of 8");
  GPP_ARG_CHECK(lda >= (a_mn ? M : K) && ldb >= (b_mn ? N : K), "leading dim too small");
  return GPP_OK;
}

template <bool A_MN, bool B_MN, int EPI>
static int batched_bn(const void* a, int64_t lda, int64_t a_rows, const void* b, int64_t ldb,
                      int64_t b_rows, const EpiParams& ep, const BatchSpec& bs, int64_t M, int64_t N,
                      int64_t K, cudaStream_t stream) {
  // full operand extents: K-major -> (inner = ld, outer = rows); MN-major -> (inner = ld, outer = rows)
  const int64_t ai = lda, ao = a_rows, bi = ldb, bo = b_rows;
  if (K <= 2 * BK) {
    // attention scores / dP (K = head dim): one or two k-blocks, so a deep ring buys
    // nothing; 2 stages (97 KB smem, BN TMEM columns) let two CTAs share an SM and
    // overlap one tile's fp32 epilogue with the next tile's loads and MMA
    if (N > 128)
      return launch_tc<256, 2, A_MN, B_MN, EPI>(a, lda, b, ldb, ep, M, N, K, 1, stream, bs, ai, ao, bi, bo);
    return launch_tc<128, 2, A_MN, B_MN, EPI>(a, lda, b, ldb, ep, M, N, K, 1, stream, bs, ai, ao, bi, bo);
  }
  if (N > 128)
    return launch_tc<256, 4, A_MN, B_MN, EPI>(a, lda, b, ldb, ep, M, N, K, 1, stream, bs, ai, ao, bi, bo);
  if (N <= 64)  // head-dim outputs (P.V, dQ, dK, dV): 64-wide tiles, 96 KB smem -> 2 CTAs / SM
    return launch_tc<64, 4, A_MN, B_MN, EPI>(a, lda, b, ldb, ep, M, N, K, 1, stream, bs, ai, ao, bi, bo);
  return launch_tc<128, 6, A_MN, B_MN, EPI>(a, lda, b, ldb, ep, M, N, K, 1, stream, bs, ai, ao, bi, bo);
}

template <int EPI>
static int batched_layout(const void* a, int64_t lda, int64_t a_rows, int a_mn, const void* b,
                          int64_t ldb, int64_t b_rows, int b_mn, const EpiParams& ep,
                          const BatchSpec& bs, int64_t M, int64_t N, int64_t K, cudaStream_t s) {
  if (!a_mn && !b_mn) return batched_bn<false, false, EPI>(a, lda, a_rows, b, ldb, b_rows, ep, bs, M, N, K, s);
  if (!a_mn && b_mn) return batched_bn<false, true, EPI>(a, lda, a_rows, b, ldb, b_rows, ep, bs, M, N, K, s);
  if (a_mn && !b_mn) return batched_bn<true, false, EPI>(a, lda, a_rows, b, ldb, b_rows, ep, bs, M, N, K, s);
  return batched_bn<true, true, EPI>(a, lda, a_rows, b, ldb, b_rows, ep, bs, M, N, K, s);
}


// ------------------------------------------------------------------------
// Attention scores with the softmax fused into the epilogue (MMT, S <= 512 keys).
//
// One CTA per (batch = sample x head, 128 query rows): the whole 128 x S score block
// lives in TMEM (512 fp32 columns, two N=256 UMMAs per k-step), so the epilogue thread
// that owns a query row sees every key of it and writes the probabilities directly:
//   fw : P  = softmax(alpha * Q K^T)                 (3 TMEM passes: max, sum, write)
//   bw : dS = alpha * P o (dP - rowsum(P o dP)),  dP = dO V^T   (2 passes, P from HBM)
// The fp32 score / dP matrices never reach HBM (the unfused path wrote and re-read
// 2 x Z S^2 x 4 bytes per layer and direction).
// ------------------------------------------------------------------------
constexpr int ATT_N = 512;
constexpr int ATT_STAGES = 1;  // ~82 KB smem: two CTAs per SM (one computing, one loading)
constexpr int ATT_EPI_WARPS = 8;                        // two per TMEM lane quarter
constexpr int ATT_THREADS = 64 + 32 * ATT_EPI_WARPS;    // + TMA warp + MMA warp

template <bool BWD>
__global__ void __launch_bounds__(ATT_THREADS, 1)
    attn_softmax_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                        bf16* __restrict__ out, int64_t ldc, const bf16* __restrict__ P, int64_t ldp,
                        float alpha, int M, int N, int K, BatchSpec bs) {
  constexpr int A_BYTES = BM * BK * 2;
  constexpr int B_HALF = 256 * BK * 2;
  constexpr int STAGE_BYTES = A_BYTES + 2 * B_HALF;
  constexpr uint32_t IDESC = idesc_bf16<256, false, false>();

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + ATT_STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + ATT_STAGES;
  uint64_t* accum_bar = empty_bar + ATT_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum_bar + 1);
  float* red = reinterpret_cast<float*>(smem + ATT_STAGES * STAGE_BYTES + 256);  // [2 halves][128 rows]
  // per epilogue warp: a 32-row x 32-key bf16 chunk staged for coalesced row stores
  constexpr int ATT_STG_LD = 80;  // bytes per staged row (64 + pad)
  uint8_t* stg_all = smem + ATT_STAGES * STAGE_BYTES + 256 + 2 * BM * 4;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m_blocks = (M + BM - 1) / BM;
  const int z = static_cast<int>(blockIdx.x) / m_blocks;
  const int m_blk = static_cast<int>(blockIdx.x) % m_blocks;
  const int z_hi = z / bs.nlo, z_lo = z % bs.nlo;
  const int am_off = bs.a_m0 + z_hi * bs.a_m_hi + z_lo * bs.a_m_lo;
  const int ak_off = bs.a_k0 + z_hi * bs.a_k_hi + z_lo * bs.a_k_lo;
  const int bn_off = bs.b_n0 + z_hi * bs.b_n_hi + z_lo * bs.b_n_lo;
  const int bk_off = bs.b_k0 + z_hi * bs.b_k_hi + z_lo * bs.b_k_lo;
  const int64_t c_off = bs.c0 + z_hi * bs.c_hi + z_lo * bs.c_lo;
  const int num_kb = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
    for (int s = 0; s < ATT_STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(accum_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();  // barriers initialised

  // The whole TMEM (512 columns) is one CTA's score block, so a second resident CTA
  // blocks in tcgen05.alloc until this one frees it -- its TMA loads are issued BEFORE
  // the allocation and overlap this CTA's epilogue.
  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % ATT_STAGES;
        mbar_wait(&empty_bar[s], ((kb / ATT_STAGES) & 1) ^ 1);
        uint8_t* a_dst = smem + s * STAGE_BYTES;
        mbar_expect_tx(&full_bar[s], STAGE_BYTES);
        tma_load_2d(a_dst, &tma_a, &full_bar[s], kb * BK + ak_off, m_blk * BM + am_off);
        tma_load_2d(a_dst + A_BYTES, &tma_b, &full_bar[s], kb * BK + bk_off, bn_off);
        tma_load_2d(a_dst + A_BYTES + B_HALF, &tma_b, &full_bar[s], kb * BK + bk_off, bn_off + 256);
      }
    }
  } else {
    if (warp == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(ATT_N)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    asm volatile("bar.sync 2, %0;" ::"n"(32 + 32 * ATT_EPI_WARPS) : "memory");  // warps 1..9
    tc_fence_after();
  }
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
  } else if (warp == 1) {
    if (lane == 0) {
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % ATT_STAGES;
        mbar_wait(&full_bar[s], (kb / ATT_STAGES) & 1);
        tc_fence_after();
        const uint32_t a_base = smem_u32(smem + s * STAGE_BYTES);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          const uint64_t adesc = sdesc_sw128(a_base + k * 32, 16, 1024);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint64_t bdesc = sdesc_sw128(a_base + A_BYTES + h * B_HALF + k * 32, 16, 1024);
            umma_bf16(tmem_base + h * 256, adesc, bdesc, IDESC, (kb | k) != 0 ? 1u : 0u);
          }
        }
        umma_commit(&empty_bar[s]);
      }
      umma_commit(accum_bar);
    }
  } else {
    // epilogue: warp w handles TMEM lane quarter w % 4 (its 32 query rows) and key half
    // hf = (w - 2) / 4; the two halves of a row combine max / sums through smem
    mbar_wait(accum_bar, 0);
    tc_fence_after();
    const int q = warp & 3;
    const int hf = (warp - 2) / 4;
    const int lr = q * 32 + lane;
    const int row = m_blk * BM + lr;
    const bool live = row < M;
    const int c_lo = hf * 8, c_hi = min(N / 32, hf * 8 + 8);  // this half's 32-key chunks
    const uint32_t trow = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
    uint8_t* stg = stg_all + (warp - 2) * 32 * ATT_STG_LD;
    const int row_base = m_blk * BM + q * 32;
    // this thread's 32 outputs (64 B of its row) -> smem -> 4 lanes per row, 16 B each
    auto store_chunk = [&](int c, const uint4 (&pk)[4]) {
#pragma unroll
      for (int i = 0; i < 4; ++i) *reinterpret_cast<uint4*>(stg + lane * ATT_STG_LD + i * 16) = pk[i];
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = (lane >> 2) + 8 * i, seg = lane & 3;
        const uint4 val = *reinterpret_cast<const uint4*>(stg + r * ATT_STG_LD + seg * 16);
        if (row_base + r < M)
          *reinterpret_cast<uint4*>(out + c_off + static_cast<int64_t>(row_base + r) * ldc + c * 32 + seg * 8) = val;
      }
      __syncwarp();
    };
    auto combine = [&](float v, bool is_max) {
      red[hf * BM + lr] = v;
      asm volatile("bar.sync 1, %0;" ::"n"(32 * ATT_EPI_WARPS) : "memory");
      const float o = red[(1 - hf) * BM + lr];
      asm volatile("bar.sync 1, %0;" ::"n"(32 * ATT_EPI_WARPS) : "memory");  // red reusable
      return is_max ? fmaxf(v, o) : v + o;
    };
    if constexpr (!BWD) {
      float mx = -INFINITY;
      for (int c = c_lo; c < c_hi; ++c) {
        uint32_t v[32];
        tmem_ld32(trow + c * 32, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) mx = fmaxf(mx, __uint_as_float(v[j]));
      }
      mx = combine(mx, true);
      const float sl2 = alpha * 1.4426950408889634f;  // alpha * log2(e); alpha > 0
      const float mb = mx * sl2;
      float sum = 0.f;
      for (int c = c_lo; c < c_hi; ++c) {  // one exp per score, parked back in TMEM
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
      const float inv = 1.f / combine(sum, false);
      for (int c = c_lo; c < c_hi; ++c) {
        uint32_t v[32];
        tmem_ld32(trow + c * 32, v);
        uint4 pk[4];
        uint32_t* w = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(v[j]) * inv, __uint_as_float(v[j + 1]) * inv);
          w[j / 2] = *reinterpret_cast<const uint32_t*>(&h2);
        }
        store_chunk(c, pk);
      }
    } else {
      const bf16* prow = P + c_off + static_cast<int64_t>(live ? row : 0) * ldp;
      auto load_p = [&](int c, float (&pf)[32]) {
        uint4 r[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) r[i] = __ldg(reinterpret_cast<const uint4*>(prow + c * 32) + i);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r[i]);
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            pf[i * 8 + 2 * t] = __low2float(h[t]);
            pf[i * 8 + 2 * t + 1] = __high2float(h[t]);
          }
        }
      };
      float D = 0.f;
      for (int c = c_lo; c < c_hi; ++c) {
        uint32_t v[32];
        float pf[32];
        load_p(c, pf);
        tmem_ld32(trow + c * 32, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) D = fmaf(pf[j], __uint_as_float(v[j]), D);
      }
      D = combine(D, false);
      for (int c = c_lo; c < c_hi; ++c) {
        uint32_t v[32];
        float pf[32];
        load_p(c, pf);
        tmem_ld32(trow + c * 32, v);
        uint4 pk[4];
        uint32_t* w = reinterpret_cast<uint32_t*>(pk);
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const __nv_bfloat162 h2 = __floats2bfloat162_rn(alpha * pf[j] * (__uint_as_float(v[j]) - D),
                                                          alpha * pf[j + 1] * (__uint_as_float(v[j + 1]) - D));
          w[j / 2] = *reinterpret_cast<const uint32_t*>(&h2);
        }
        store_chunk(c, pk);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(ATT_N) : "memory");
  }
}

template <bool BWD>
static int launch_attn_softmax(bf16* out, int64_t ldc, const bf16* P, int64_t ldp, const void* a, int64_t lda,
                               int64_t a_rows, const void* b, int64_t ldb, int64_t b_rows, const BatchSpec& bs,
                               int64_t M, int64_t N, int64_t K, float alpha, cudaStream_t stream) {
  CUtensorMap ma, mb;
  int rc = make_map(&ma, a, lda, a_rows, lda, BK, BM);
  if (rc) return rc;
  rc = make_map(&mb, b, ldb, b_rows, ldb, BK, 256);
  if (rc) return rc;
  constexpr int SMEM = ATT_STAGES * (BM * BK * 2 + 2 * 256 * BK * 2) + 1024 + 256 + 2 * BM * 4 +
                       ATT_EPI_WARPS * 32 * 80;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(attn_softmax_kernel<BWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    attr_set = true;
  }
  const int64_t grid = static_cast<int64_t>(bs.nbatch) * ((M + BM - 1) / BM);
  attn_softmax_kernel<BWD><<<static_cast<unsigned>(grid), ATT_THREADS, SMEM, stream>>>(
      ma, mb, out, ldc, P, ldp, alpha, static_cast<int>(M), static_cast<int>(N), static_cast<int>(K), bs);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("attn_softmax launch: ") + cudaGetErrorString(e));
    return GPP_ERR_CUDA;
  }
  count_launch();
  return GPP_OK;
}

}  // namespace tc

int tc_gemm_batched(int epi, const void* a, int64_t lda, int64_t a_rows, int a_mn, const void* b,
                    int64_t ldb, int64_t b_rows, int b_mn, const EpiParams& ep, const BatchSpec& bs,
                    int64_t M, int64_t N, int64_t K, cudaStream_t stream) {
  GPP_ARG_CHECK(M > 0 && N > 0 && K > 0 && bs.nbatch >= 1 && bs.nlo >= 1, "bad shape");
  GPP_ARG_CHECK(K % 64 == 0, "batched GEMM needs K % 64 == 0 (no K-tile may straddle batches)");
  GPP_ARG_CHECK((reinterpret_cast<uintptr_t>(a) & 15) == 0 && (reinterpret_cast<uintptr_t>(b) & 15) == 0 &&
                    lda % 8 == 0 && ldb % 8 == 0, "TMA alignment");
  switch (epi) {
    case EPI_FWD: return tc::batched_layout<EPI_FWD>(a, lda, a_rows, a_mn, b, ldb, b_rows, b_mn, ep, bs, M, N, K, stream);
    case EPI_F32: return tc::batched_layout<EPI_F32>(a, lda, a_rows, a_mn, b, ldb, b_rows, b_mn, ep, bs, M, N, K, stream);
    default: return tc::batched_layout<EPI_BF16>(a, lda, a_rows, a_mn, b, ldb, b_rows, b_mn, ep, bs, M, N, K, stream);
  }
}

// Entry points used by capi.cu.
int tc_gemm(int epi, const void* a, int64_t lda, int a_mn, const void* b, int64_t ldb, int b_mn,
            const EpiParams& ep_in, int64_t M, int64_t N, int64_t K, cudaStream_t stream) {
  int rc = tc::check_operands(a, lda, a_mn, b, ldb, b_mn, M, N, K);
  if (rc) return rc;
  EpiParams ep = ep_in;
  take_prefetch_hint(ep);
  switch (epi) {
    case EPI_FWD:
      return tc::dispatch_layout<EPI_FWD>(a, lda, a_mn, b, ldb, b_mn, ep, M, N, K, stream);
    case EPI_DGRAD:
      return tc::dispatch_layout<EPI_DGRAD>(a, lda, a_mn, b, ldb, b_mn, ep, M, N, K, stream);
    case EPI_F32:
      return tc::dispatch_layout<EPI_F32>(a, lda, a_mn, b, ldb, b_mn, ep, M, N, K, stream);
    case EPI_SGD:
      return tc::dispatch_layout<EPI_SGD>(a, lda, a_mn, b, ldb, b_mn, ep, M, N, K, stream);
    default:
      return tc::dispatch_layout<EPI_BF16>(a, lda, a_mn, b, ldb, b_mn, ep, M, N, K, stream);
  }
}

int tc_attn_softmax(int bwd, void* out, int64_t ldc, const void* P, int64_t ldp, const void* a, int64_t lda,
                    int64_t a_rows, const void* b, int64_t ldb, int64_t b_rows, const BatchSpec& bs, int64_t M,
                    int64_t N, int64_t K, float alpha, cudaStream_t stream) {
  GPP_ARG_CHECK(M > 0 && N > 0 && K > 0 && bs.nbatch >= 1 && bs.nlo >= 1, "bad shape");
  GPP_ARG_CHECK(N <= tc::ATT_N && N % 32 == 0, "fused attention softmax needs 32 | keys <= 512");
  GPP_ARG_CHECK(K % tc::BK == 0 && K <= 4 * tc::BK, "head dim must be a multiple of 64, <= 256 (no k-tile may straddle heads)");
  GPP_ARG_CHECK(alpha > 0.f, "softmax scale must be positive");
  GPP_ARG_CHECK((reinterpret_cast<uintptr_t>(a) & 15) == 0 && (reinterpret_cast<uintptr_t>(b) & 15) == 0 &&
                    lda % 8 == 0 && ldb % 8 == 0, "TMA alignment");
  GPP_ARG_CHECK((reinterpret_cast<uintptr_t>(out) & 15) == 0 && ldc % 8 == 0 && bs.c0 % 8 == 0 &&
                    bs.c_hi % 8 == 0 && bs.c_lo % 8 == 0, "16-byte aligned output rows");
  if (bwd) {
    GPP_ARG_CHECK(P && (reinterpret_cast<uintptr_t>(P) & 15) == 0 && ldp % 8 == 0, "16-byte aligned P rows");
    return tc::launch_attn_softmax<true>(static_cast<bf16*>(out), ldc, static_cast<const bf16*>(P), ldp, a, lda,
                                         a_rows, b, ldb, b_rows, bs, M, N, K, alpha, stream);
  }
  return tc::launch_attn_softmax<false>(static_cast<bf16*>(out), ldc, nullptr, 0, a, lda, a_rows, b, ldb, b_rows,
                                        bs, M, N, K, alpha, stream);
}

}  // namespace gpp
