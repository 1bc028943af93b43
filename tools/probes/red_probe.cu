// Probe: L2 fp32 reduction throughput for an FA-style dQ accumulation (each of the T x d
// fp32 dQ elements receives `adds` contributions from different CTAs), red.global.add
// with 4-, 8- and 16-byte vectors vs plain 16-byte stores of the same bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/r tools/probes/red_probe.cu && /tmp/r
#include <cstdio>
#include <cstdint>

template <int V>
__global__ void red_kernel(float* __restrict__ dq, int64_t n, int adds) {
  // CTA c handles elements [(c % nchunk) * 8192, +8192) for contribution c / nchunk
  const int64_t nchunk = n / 8192;
  const int64_t chunk = blockIdx.x % nchunk;
  float* base = dq + chunk * 8192;
  for (int i = threadIdx.x * V; i < 8192; i += 256 * V) {
    if constexpr (V == 1) atomicAdd(base + i, 1.f);
    if constexpr (V == 2) atomicAdd(reinterpret_cast<float2*>(base + i), make_float2(1.f, 1.f));
    if constexpr (V == 4) atomicAdd(reinterpret_cast<float4*>(base + i), make_float4(1.f, 1.f, 1.f, 1.f));
  }
}
__global__ void store_kernel(float* __restrict__ dq, int64_t n) {
  const int64_t nchunk = n / 8192;
  float* base = dq + (blockIdx.x % nchunk) * 8192;
  for (int i = threadIdx.x * 4; i < 8192; i += 1024)
    *reinterpret_cast<float4*>(base + i) = make_float4(1.f, 1.f, 1.f, 1.f);
}

int main() {
  const int64_t n = 8192LL * 1024;  // T x d of one MMT layer's dQ
  const int adds = 4;                // S / 128 key blocks per query row
  float* dq;
  cudaMalloc(&dq, n * 4);
  cudaMemset(dq, 0, n * 4);
  const int grid = static_cast<int>(n / 8192) * adds;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1e3 / 10;
    printf("%-12s %8.1f us  %7.1f GB/s payload  %.2f G ops/s\n", name, us, n * adds * 4.0 / (us * 1e3),
           0.0);
  };
  run("red.f32", [&] { red_kernel<1><<<grid, 256>>>(dq, n, adds); });
  run("red.v2.f32", [&] { red_kernel<2><<<grid, 256>>>(dq, n, adds); });
  run("red.v4.f32", [&] { red_kernel<4><<<grid, 256>>>(dq, n, adds); });
  run("st.v4 (ref)", [&] { store_kernel<<<grid, 256>>>(dq, n); });
  printf("err=%s (payload = %lld floats x %d adds = %.1f MB)\n", cudaGetErrorString(cudaGetLastError()),
         (long long)n, adds, n * adds * 4.0 / 1e6);
  return 0;
}
