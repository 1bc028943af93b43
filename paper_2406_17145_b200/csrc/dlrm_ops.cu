// DLRM operators (Appendix B): embedding-bag
// gather-sum, its sparse SGD scatter, and the pairwise dot interaction.
// All HBM / latency bound: warp-per-bag with 8-byte vector row loads, ILP over the
// bag, warp-per-sample interaction staged through padded shared memory.
#include <algorithm>
#include <cstdlib>

#define GPP_PDL_CLASS 16  // programmatic-dependent-launch families: 16 embedding bags, 32 interaction, 64 sparse SGD
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
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
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
  pdl_wait();
  pdl_trigger();
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

// ---- deterministic sparse SGD over several tables (counting sort by row) ----------------
// table_t[r] -= lr * sum over the bag elements (m, b) with idx_t[m, b] == r of dpooled_t[m],
// the sum taken in increasing (m, b) order whatever the thread timing:
//   count  : cnt[t, r] += 1 per element (integer atomics: order-free)
//   scan   : start = exclusive prefix sum of cnt over all (t, r)   (3 kernels)
//   scatter: perm[start[t, r]++] = element id  (bucket order still arbitrary)
//   apply  : one warp per bucket (a run of equal (t, r) keys in perm, its end = the bumped
//            start): ranks its element ids, adds the pooled gradients in rank order, updates
//            the row once (256 B, coalesced).  Buckets > 32 by repeated min-extraction.
// Out-of-range indices are skipped and counted (g_bad_indices), as in the atomic kernel.
constexpr int kSgdTables = 32;
struct SgdTables {
  float* table[kSgdTables];
  const bf16* dpool[kSgdTables];
  const int64_t* idx[kSgdTables];
  int64_t rows[kSgdTables];
  int64_t row_base[kSgdTables];  // prefix of rows: key = row_base[t] + r
  int n, bag;
  int64_t M, ldd, ldi;
  float lr;
};

__device__ __forceinline__ int64_t sgd_key(const SgdTables& tb, int64_t e, int& t, int64_t& m) {
  const int64_t E = tb.M * tb.bag;
  t = static_cast<int>(e / E);
  const int64_t local = e - static_cast<int64_t>(t) * E;
  m = local / tb.bag;
  const int64_t r = __ldg(tb.idx[t] + m * tb.ldi + (local % tb.bag));
  if (r < 0 || r >= tb.rows[t]) return -1;
  return tb.row_base[t] + r;
}

__global__ void __launch_bounds__(256) sgd_count_kernel(unsigned* cnt, const __grid_constant__ SgdTables tb) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = static_cast<int64_t>(tb.n) * tb.M * tb.bag;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int t;
    int64_t m;
    const int64_t k = sgd_key(tb, e, t, m);
    if (k < 0) {
      atomicAdd(&g_bad_indices, 1ull);
      continue;
    }
    atomicAdd(cnt + k, 1u);
  }
}

// exclusive scan of cnt [n] in place: per-block sums, a one-block scan of those, then the
// per-block scans with their offsets.  Block = 1024 threads x 8 items.
constexpr int kScanItems = 8, kScanThreads = 1024, kScanBlock = kScanItems * kScanThreads;

__device__ __forceinline__ unsigned block_scan_excl(unsigned v, unsigned* sh, unsigned& total) {
  // warp inclusive scan
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    unsigned s = lane < (blockDim.x >> 5) ? sh[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    sh[lane] = s;  // inclusive warp-sum prefix
  }
  __syncthreads();
  total = sh[(blockDim.x >> 5) - 1];
  const unsigned before = w > 0 ? sh[w - 1] : 0u;
  __syncthreads();
  return before + x - v;
}

__global__ void __launch_bounds__(kScanThreads) scan_sums_kernel(const unsigned* cnt, unsigned* sums, int64_t n) {
  pdl_wait();
  pdl_trigger();
  __shared__ unsigned sh[32];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanBlock + threadIdx.x * kScanItems;
  unsigned v = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) v += base + i < n ? cnt[base + i] : 0u;
  unsigned total;
  block_scan_excl(v, sh, total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads) scan_top_kernel(unsigned* sums, int nb) {
  pdl_wait();
  pdl_trigger();
  __shared__ unsigned sh[32];
  unsigned carry = 0;
  for (int base = 0; base < nb; base += kScanThreads) {
    const int i = base + threadIdx.x;
    const unsigned v = i < nb ? sums[i] : 0u;
    unsigned total;
    const unsigned ex = block_scan_excl(v, sh, total);
    if (i < nb) sums[i] = carry + ex;
    carry += total;
  }
}

__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(unsigned* cnt, const unsigned* sums, int64_t n) {
  pdl_wait();
  pdl_trigger();
  __shared__ unsigned sh[32];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanBlock + threadIdx.x * kScanItems;
  unsigned v[kScanItems], tot = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = base + i < n ? cnt[base + i] : 0u;
    tot += v[i];
  }
  unsigned total;
  unsigned run = sums[blockIdx.x] + block_scan_excl(tot, sh, total);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) cnt[base + i] = run;
    run += v[i];
  }
}

__global__ void __launch_bounds__(256) sgd_scatter_kernel(unsigned* start, unsigned* perm,
                                                         const __grid_constant__ SgdTables tb) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = static_cast<int64_t>(tb.n) * tb.M * tb.bag;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int t;
    int64_t m;
    const int64_t k = sgd_key(tb, e, t, m);
    if (k < 0) continue;
    perm[atomicAdd(start + k, 1u)] = static_cast<unsigned>(e);
  }
}

// one thread per (table, row) key: its bucket is perm[end[k-1], end[k]) (the exclusive scan
// made start[k] = end[k-1]); the element ids are put in increasing order (insertion sort in
// registers for <= 8, repeated min-extraction beyond) and their bags' pooled gradients summed
// in that order into 64 fp32 registers, then the table row is updated once (256 B).
__global__ void __launch_bounds__(256) sgd_apply_kernel(const unsigned* end, const unsigned* perm, int64_t keys,
                                                       const __grid_constant__ SgdTables tb) {
  pdl_wait();
  pdl_trigger();
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= keys) return;
  const unsigned e1 = end[k], e0 = k > 0 ? end[k - 1] : 0u;
  const unsigned n = e1 - e0;
  if (n == 0) return;
  int t = 0;
  while (t + 1 < tb.n && k >= tb.row_base[t + 1]) ++t;
  const int64_t E = tb.M * tb.bag, tbase = static_cast<int64_t>(t) * E;
  const bf16* dp = tb.dpool[t];
  float acc[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) acc[i] = 0.f;
  auto add_bag = [&](unsigned e) {
    const int64_t m = (static_cast<int64_t>(e) - tbase) / tb.bag;
    const uint4* g = reinterpret_cast<const uint4*>(dp + m * tb.ldd);
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const uint4 u = __ldg(g + v);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(h[q]);
        acc[8 * v + 2 * q] += f.x;
        acc[8 * v + 2 * q + 1] += f.y;
      }
    }
  };
  if (n <= 8) {
    unsigned ids[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) ids[i] = i < static_cast<int>(n) ? perm[e0 + i] : 0xffffffffu;
#pragma unroll
    for (int i = 1; i < 8; ++i) {  // insertion sort (unused slots hold the max id: stay last)
#pragma unroll
      for (int j = i; j > 0; --j) {
        const unsigned a = ids[j - 1], b = ids[j];
        ids[j - 1] = min(a, b);
        ids[j] = max(a, b);
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < static_cast<int>(n)) add_bag(ids[i]);
  } else {
    unsigned last = 0;
    for (unsigned r = 0; r < n; ++r) {  // next smallest id > last (ids are unique)
      unsigned best = 0xffffffffu;
      for (unsigned i = e0; i < e1; ++i) {
        const unsigned e = perm[i];
        if ((r == 0 || e > last) && e < best) best = e;
      }
      last = best;
      add_bag(best);
    }
  }
  float4* row = reinterpret_cast<float4*>(tb.table[t] + (k - tb.row_base[t]) * 64);
#pragma unroll
  for (int v = 0; v < 16; ++v) {
    float4 w = row[v];
    w.x -= tb.lr * acc[4 * v];
    w.y -= tb.lr * acc[4 * v + 1];
    w.z -= tb.lr * acc[4 * v + 2];
    w.w -= tb.lr * acc[4 * v + 3];
    row[v] = w;
  }
}

// grow-only scratch (never freed: graphs captured earlier may reference it)
unsigned* sgd_scratch(size_t words, cudaStream_t stream) {
  static unsigned* bufs[64] = {nullptr};
  static size_t caps[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (caps[dev] >= words) return bufs[dev];
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(stream, &st);
  if (st != cudaStreamCaptureStatusNone) {
    set_error("embedding SGD scratch must be sized before CUDA-graph capture (run one eager step first)");
    return nullptr;
  }
  unsigned* p = nullptr;
  if (cudaMalloc(&p, words * sizeof(unsigned)) != cudaSuccess) {
    set_error("embedding SGD scratch allocation failed");
    return nullptr;
  }
  bufs[dev] = p;
  caps[dev] = words;
  return p;
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
  launch_pdl(embbag_fwd_kernel, dim3(static_cast<unsigned>((M + 7) / 8)), dim3(256), 0, static_cast<cudaStream_t>(stream), static_cast<bf16*>(out), ldo, table, idx, ldi, M, static_cast<int>(bag), rows);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_embbag_sgd(float* table, const void* dpooled, int64_t ldd, const int64_t* idx, int64_t ldi,
                   int64_t M, int64_t bag, int64_t D, int64_t rows, float lr, void* stream) {
  GPP_ARG_CHECK(table && dpooled && idx && M > 0 && bag > 0, "bad argument");
  GPP_ARG_CHECK(D == 64, "embedding dim must be 64");
  launch_pdl(embbag_sgd_kernel, dim3(static_cast<unsigned>((M + 7) / 8)), dim3(256), 0, static_cast<cudaStream_t>(stream), table, static_cast<const bf16*>(dpooled), ldd, idx, ldi, M, static_cast<int>(bag), lr, rows);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_embbag_sgd_multi(int n, float* const* tables, const int64_t* rows, const void* const* dpooled, int64_t ldd,
                         const int64_t* const* idx, int64_t ldi, int64_t M, int64_t bag, int64_t D, float lr,
                         void* stream) {
  GPP_ARG_CHECK(n >= 1 && n <= kSgdTables && tables && rows && dpooled && idx && M > 0 && bag > 0, "bad argument");
  GPP_ARG_CHECK(D == 64, "embedding dim must be 64");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  SgdTables tb{};
  int64_t keys = 0;
  for (int t = 0; t < n; ++t) {
    GPP_ARG_CHECK(tables[t] && dpooled[t] && idx[t] && rows[t] > 0, "bad table");
    tb.table[t] = tables[t];
    tb.dpool[t] = static_cast<const bf16*>(dpooled[t]);
    tb.idx[t] = idx[t];
    tb.rows[t] = rows[t];
    tb.row_base[t] = keys;
    keys += rows[t];
  }
  tb.n = n;
  tb.bag = static_cast<int>(bag);
  tb.M = M;
  tb.ldd = ldd;
  tb.ldi = ldi;
  tb.lr = lr;
  const int64_t total = static_cast<int64_t>(n) * M * bag;
  GPP_ARG_CHECK(total < (1ll << 32) && keys < (1ll << 31), "too many elements for 32-bit ids");
  const int64_t nsum = (keys + kScanBlock - 1) / kScanBlock;
  unsigned* scratch = sgd_scratch(static_cast<size_t>(keys + total + nsum), s);
  if (!scratch) return GPP_ERR_CUDA;
  unsigned* cnt = scratch;            // counts, then bucket starts, then bucket ends
  unsigned* perm = scratch + keys;    // element ids in bucket order
  unsigned* sums = perm + total;
  if (cudaMemsetAsync(cnt, 0, static_cast<size_t>(keys) * sizeof(unsigned), s) != cudaSuccess) {
    set_error("embedding SGD: memset failed");
    return GPP_ERR_CUDA;
  }
  const unsigned eg = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  launch_pdl_impl(64, sgd_count_kernel, dim3(eg), dim3(256), 0, s, cnt, tb);
  GPP_LAUNCH_CHECK();
  launch_pdl_impl(64, scan_sums_kernel, dim3(static_cast<unsigned>(nsum)), dim3(kScanThreads), 0, s, cnt, sums, keys);
  GPP_LAUNCH_CHECK();
  launch_pdl_impl(64, scan_top_kernel, dim3(1), dim3(kScanThreads), 0, s, sums, static_cast<int>(nsum));
  GPP_LAUNCH_CHECK();
  launch_pdl_impl(64, scan_apply_kernel, dim3(static_cast<unsigned>(nsum)), dim3(kScanThreads), 0, s, cnt, sums, keys);
  GPP_LAUNCH_CHECK();
  launch_pdl_impl(64, sgd_scatter_kernel, dim3(eg), dim3(256), 0, s, cnt, perm, tb);
  GPP_LAUNCH_CHECK();
  // after the scatter cnt[k] is bucket k's end; its start is cnt[k - 1]
  launch_pdl_impl(64, sgd_apply_kernel, dim3(static_cast<unsigned>((keys + 255) / 256)), dim3(256), 0, s, cnt, perm, keys, tb);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_interaction_fwd(void* out, int64_t ldo, int64_t out_cols, const void* z, int64_t ldz,
                        int64_t M, int64_t F, int64_t D, void* stream) {
  GPP_ARG_CHECK(out && z && M > 0 && F >= 2 && D == 64, "bad argument");
  GPP_ARG_CHECK(out_cols >= 64 + F * (F - 1) / 2 && out_cols <= ldo, "output too narrow");
  const size_t smem = 4 * F * ZLD * sizeof(float);
  launch_pdl_impl(32, interaction_fwd_kernel, dim3(static_cast<unsigned>((M + 3) / 4)), dim3(128), smem, static_cast<cudaStream_t>(stream), static_cast<bf16*>(out), ldo, out_cols, static_cast<const bf16*>(z), ldz, M, static_cast<int>(F));
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

int gpp_interaction_bwd(void* dz, int64_t lddz, const void* dout, int64_t lddo, const void* z,
                        int64_t ldz, int64_t M, int64_t F, int64_t D, int mask_first, void* stream) {
  GPP_ARG_CHECK(dz && dout && z && M > 0 && F >= 2 && D == 64, "bad argument");
  // GPP_INTERACTION_GENERIC=1 forces the generic kernel (tests assert both are bit-identical)
  const char* gen = getenv("GPP_INTERACTION_GENERIC");
  if (F == 27 && !(gen && gen[0] == '1')) {  // DLRM: 26 tables + the bottom MLP
    launch_pdl_impl(32, interaction_bwd_reg_kernel<27>, dim3(static_cast<unsigned>((M + 3) / 4)), dim3(128), 0, static_cast<cudaStream_t>(stream), static_cast<bf16*>(dz), lddz, static_cast<const bf16*>(dout), lddo, static_cast<const bf16*>(z), ldz, M,
        mask_first);
    GPP_LAUNCH_CHECK();
    return GPP_OK;
  }
  const size_t smem = 4 * (F * ZLD + F * (F - 1) / 2 + 1) * sizeof(float);
  launch_pdl_impl(32, interaction_bwd_kernel, dim3(static_cast<unsigned>((M + 3) / 4)), dim3(128), smem, static_cast<cudaStream_t>(stream), static_cast<bf16*>(dz), lddz, static_cast<const bf16*>(dout), lddo, static_cast<const bf16*>(z), ldz, M,
      static_cast<int>(F), mask_first);
  GPP_LAUNCH_CHECK();
  return GPP_OK;
}

}  // extern "C"
