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
#include <mutex>
#include <unordered_map>

#include "gemm.cuh"

namespace gpp {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one swizzle row
constexpr int NUM_THREADS = 192;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// tcgen05.commit: mbarrier arrive once all previously issued MMAs of this thread completed.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// Shared-memory matrix descriptor (SM100 "version 1"), SWIZZLE_128B.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version for sm_100
  d |= static_cast<uint64_t>(2) << 61;  // layout: SWIZZLE_128B
  return d;
}

// Instruction descriptor for kind::f16: bf16 x bf16 -> f32, M=128, N=BN.
template <int BN, bool A_MN, bool B_MN>
__host__ __device__ constexpr uint32_t idesc_bf16() {
  return (1u << 4)                          // D format f32
         | (1u << 7)                        // A format bf16
         | (1u << 10)                       // B format bf16
         | ((A_MN ? 1u : 0u) << 15)         // A major
         | ((B_MN ? 1u : 0u) << 16)         // B major
         | (static_cast<uint32_t>(BN >> 3) << 17) |
         (static_cast<uint32_t>(BM >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
        "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
        "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Epilogue of one thread: 32 consecutive columns [col0, col0+32) of one row.
template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const EpiParams& ep, const uint32_t (&v)[32],
                                               int row, int col0, int M, int N) {
  if (row >= M || col0 >= N) return;
  const bool full = (col0 + 32 <= N);
  float f[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]) * ep.alpha;

  if constexpr (EPI == EPI_F32) {
    float* out = reinterpret_cast<float*>(ep.out) + static_cast<int64_t>(row) * ep.ldo + col0;
    const bool vec = full && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
    if (vec) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 o = make_float4(f[j], f[j + 1], f[j + 2], f[j + 3]);
        if (ep.beta != 0.f) {
          float4 c = *reinterpret_cast<const float4*>(out + j);
          o.x += ep.beta * c.x; o.y += ep.beta * c.y; o.z += ep.beta * c.z; o.w += ep.beta * c.w;
        }
        *reinterpret_cast<float4*>(out + j) = o;
      }
    } else {
      for (int j = 0; j < 32 && col0 + j < N; ++j) {
        float o = f[j];
        if (ep.beta != 0.f) o += ep.beta * out[j];
        out[j] = o;
      }
    }
    return;
  } else {
    if constexpr (EPI == EPI_FWD) {
      if (ep.bias != nullptr) {
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] += (full || col0 + j < N) ? __ldg(ep.bias + col0 + j) : 0.f;
      }
      if (ep.pre != nullptr) {
        bf16* pre = static_cast<bf16*>(ep.pre) + static_cast<int64_t>(row) * ep.ldpre + col0;
        for (int j = 0; j < 32 && col0 + j < N; ++j) pre[j] = __float2bfloat16_rn(f[j]);
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) f[j] = act_fwd(f[j], ep.act);
      if (ep.aux != nullptr) {
        const bf16* res = static_cast<const bf16*>(ep.aux) + static_cast<int64_t>(row) * ep.ldaux + col0;
        for (int j = 0; j < 32 && col0 + j < N; ++j) f[j] += __bfloat162float(res[j]);
      }
    } else if constexpr (EPI == EPI_DGRAD) {
      if (ep.act != GPP_ACT_NONE) {
        const bf16* sv = static_cast<const bf16*>(ep.aux) + static_cast<int64_t>(row) * ep.ldaux + col0;
        for (int j = 0; j < 32 && col0 + j < N; ++j) f[j] *= act_bwd(__bfloat162float(sv[j]), ep.act);
      }
    }
    bf16* out = reinterpret_cast<bf16*>(ep.out) + static_cast<int64_t>(row) * ep.ldo + col0;
    if constexpr (EPI == EPI_BF16) {
      if (ep.beta != 0.f) {
        for (int j = 0; j < 32 && col0 + j < N; ++j) f[j] += ep.beta * __bfloat162float(out[j]);
      }
    }
    const bool vec = full && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
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
        *reinterpret_cast<uint4*>(out + j) = pk;
      }
    } else {
      for (int j = 0; j < 32 && col0 + j < N; ++j) out[j] = __float2bfloat16_rn(f[j]);
    }
  }
}

template <int BN, int STAGES, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tma_a,
                   const __grid_constant__ CUtensorMap tma_b, EpiParams ep, int M, int N, int K) {
  constexpr int A_BYTES = BM * BK * 2;
  constexpr int B_BYTES = BN * BK * 2;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t TMEM_COLS = BN;  // power of two >= 32
  constexpr uint32_t IDESC = idesc_bf16<BN, A_MN, B_MN>();

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* accum_bar = empty_bar + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum_bar + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_blocks = (N + BN - 1) / BN;
  const int m_blk = blockIdx.x / n_blocks;
  const int n_blk = blockIdx.x % n_blocks;
  const int num_kb = (K + BK - 1) / BK;

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
          tma_load_2d(a_dst, &tma_a, &full_bar[s], kb * BK, m_blk * BM);
        } else {
#pragma unroll
          for (int c = 0; c < BM / 64; ++c)
            tma_load_2d(a_dst + c * 8192, &tma_a, &full_bar[s], m_blk * BM + c * 64, kb * BK);
        }
        if constexpr (!B_MN) {
          tma_load_2d(b_dst, &tma_b, &full_bar[s], kb * BK, n_blk * BN);
        } else {
#pragma unroll
          for (int c = 0; c < BN / 64; ++c)
            tma_load_2d(b_dst + c * 8192, &tma_b, &full_bar[s], n_blk * BN + c * 64, kb * BK);
        }
      }
    }
  } else if (warp == 1) {
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
      tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + c * 32, v);
      epilogue_chunk<EPI>(ep, v, row, n_blk * BN + c * 32, M, N);
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
  int box_inner, box_outer;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && inner == o.inner && outer == o.outer && ld == o.ld &&
           box_inner == o.box_inner && box_outer == o.box_outer;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = std::hash<const void*>()(k.ptr);
    h ^= std::hash<int64_t>()(k.inner * 1315423911LL + k.outer) + 0x9e3779b9 + (h << 6) + (h >> 2);
    h ^= std::hash<int64_t>()(k.ld * 31 + k.box_inner * 7 + k.box_outer) + (h << 6) + (h >> 2);
    return h;
  }
};

// 2-D bf16 tensor map over a row-major buffer: `outer` rows of `inner` elements, row pitch ld.
static int make_map(CUtensorMap* out, const void* ptr, int64_t inner, int64_t outer, int64_t ld,
                    int box_inner, int box_outer) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  MapKey key{ptr, inner, outer, ld, box_inner, box_outer};
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
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
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

template <int BN, int STAGES, bool A_MN, bool B_MN, int EPI>
static int launch_tc(const void* a, int64_t lda, const void* b, int64_t ldb, const EpiParams& ep,
                     int64_t M, int64_t N, int64_t K, cudaStream_t stream) {
  CUtensorMap ma, mb;
  int rc;
  // K-major operand: inner = K, outer = rows;  MN-major: inner = rows, outer = K.
  if (!A_MN) rc = make_map(&ma, a, K, M, lda, BK, BM);
  else rc = make_map(&ma, a, M, K, lda, 64, BK);
  if (rc) return rc;
  if (!B_MN) rc = make_map(&mb, b, K, N, ldb, BK, BN);
  else rc = make_map(&mb, b, N, K, ldb, 64, BK);
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
  gemm_tc_kernel<BN, STAGES, A_MN, B_MN, EPI><<<static_cast<unsigned>(tiles), NUM_THREADS, SMEM,
                                                stream>>>(ma, mb, ep, static_cast<int>(M),
                                                          static_cast<int>(N),
                                                          static_cast<int>(K));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string("gemm_tc launch: ") + cudaGetErrorString(e));
    return GPP_ERR_CUDA;
  }
  count_launch();
  return GPP_OK;
}

template <bool A_MN, bool B_MN, int EPI>
static int dispatch_bn(const void* a, int64_t lda, const void* b, int64_t ldb,
                       const EpiParams& ep, int64_t M, int64_t N, int64_t K,
                       cudaStream_t stream) {
  const int64_t mb = (M + BM - 1) / BM;
  // Prefer the 128x256 tile (full-rate single-CTA UMMA) unless it leaves most SMs idle.
  const int64_t tiles256 = mb * ((N + 255) / 256);
  if (N > 128 && tiles256 >= 96)
    return launch_tc<256, 4, A_MN, B_MN, EPI>(a, lda, b, ldb, ep, M, N, K, stream);
  return launch_tc<128, 6, A_MN, B_MN, EPI>(a, lda, b, ldb, ep, M, N, K, stream);
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

}  // namespace tc

// Entry points used by capi.cu.
int tc_gemm(int epi, const void* a, int64_t lda, int a_mn, const void* b, int64_t ldb, int b_mn,
            const EpiParams& ep, int64_t M, int64_t N, int64_t K, cudaStream_t stream) {
  int rc = tc::check_operands(a, lda, a_mn, b, ldb, b_mn, M, N, K);
  if (rc) return rc;
  switch (epi) {
    case EPI_FWD:
      return tc::dispatch_layout<EPI_FWD>(a, lda, a_mn, b, ldb, b_mn, ep, M, N, K, stream);
    case EPI_DGRAD:
      return tc::dispatch_layout<EPI_DGRAD>(a, lda, a_mn, b, ldb, b_mn, ep, M, N, K, stream);
    case EPI_F32:
      return tc::dispatch_layout<EPI_F32>(a, lda, a_mn, b, ldb, b_mn, ep, M, N, K, stream);
    default:
      return tc::dispatch_layout<EPI_BF16>(a, lda, a_mn, b, ldb, b_mn, ep, M, N, K, stream);
  }
}

}  // namespace gpp
