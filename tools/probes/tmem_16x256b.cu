// Probe: the register <-> (TMEM lane, column) mapping of tcgen05.ld.16x256b.x4 (sm_100a).
// TMEM is filled with value = lane * 1000 + column through 32x32b stores (lane = row per
// thread), then warp 0 reads lanes 0..15 with 16x256b.x4; each thread's 16 registers are
// printed.   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/p tools/probes/tmem_16x256b.cu
#include <cstdio>
#include <cstdint>

__global__ void probe(uint32_t* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
        static_cast<uint32_t>(__cvta_generic_to_shared(&slot))));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const int row = warp * 32 + lane;
  uint32_t v[8];
  for (int c0 = 0; c0 < 32; c0 += 8) {
    for (int i = 0; i < 8; ++i) v[i] = row * 1000 + c0 + i;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                     tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 16; ++i) out[lane * 16 + i] = r[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 32 * 16 * 4);
  probe<<<1, 128>>>(d);
  uint32_t h[512];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  for (int t = 0; t < 32; ++t) {
    printf("t%02d:", t);
    for (int i = 0; i < 16; ++i) printf(" %u.%u", h[t * 16 + i] / 1000, h[t * 16 + i] % 1000);
    printf("\n");
  }
  return 0;
}
