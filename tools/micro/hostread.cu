// Zero-copy read bandwidth from page-locked host memory vs the DMA copy engine.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hostread hostread.cu
#include <cstdio>
#include <cuda_runtime.h>

// each warp streams a contiguous region, `ahead` tiles of 32 x VEC words in flight
template <int VEC, int AHEAD>
__global__ void k_read(const unsigned long long* __restrict__ src, size_t n_words, unsigned long long* sink) {
  const unsigned lane = threadIdx.x & 31;
  const size_t warps = size_t(gridDim.x) * (blockDim.x >> 5);
  const size_t w = size_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const size_t per = (n_words / warps) & ~size_t(127);
  const unsigned long long* p = src + w * per;
  constexpr int T = 32 * VEC;
  unsigned long long acc = 0;
  unsigned long long q[AHEAD][VEC];
  for (int a = 0; a < AHEAD; ++a)
    for (int v = 0; v < VEC; ++v) q[a][v] = 0;
  size_t i = 0;
#pragma unroll
  for (int a = 0; a < AHEAD; ++a)
    if (size_t(a + 1) * T <= per) {
      if (VEC == 2) { ulonglong2 x = __ldcg(reinterpret_cast<const ulonglong2*>(p + a * T) + lane); q[a][0] = x.x; q[a][VEC - 1] = x.y; }
      else q[a][0] = __ldcg(p + a * T + lane);
    }
  for (i = 0; i + T <= per; i += T) {
    for (int v = 0; v < VEC; ++v) acc += q[0][v];
#pragma unroll
    for (int a = 0; a + 1 < AHEAD; ++a)
      for (int v = 0; v < VEC; ++v) q[a][v] = q[a + 1][v];
    const size_t nx = i + size_t(AHEAD) * T;
    if (nx + T <= per) {
      if (VEC == 2) { ulonglong2 x = __ldcg(reinterpret_cast<const ulonglong2*>(p + nx) + lane); q[AHEAD - 1][0] = x.x; q[AHEAD - 1][VEC - 1] = x.y; }
      else q[AHEAD - 1][0] = __ldcg(p + nx + lane);
    }
    // emulate compute between tiles
    __nanosleep(DELAY_NS);
  }
  if (acc == 0x12345) *sink = acc;
}

template <int VEC, int AHEAD>
void run(const unsigned long long* h, size_t n, unsigned long long* sink, int warps_per_cta) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  k_read<VEC, AHEAD><<<148, 32 * warps_per_cta>>>(h, n, sink);
  cudaEventRecord(a);
  for (int r = 0; r < 3; ++r) k_read<VEC, AHEAD><<<148, 32 * warps_per_cta>>>(h, n, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("zero-copy VEC=%d AHEAD=%d warps/SM=%2d delay=%dns: %.1f GB/s (%s)\n", VEC, AHEAD, warps_per_cta, DELAY_NS,
         3.0 * n * 8 / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const size_t n = size_t(233) << 20 >> 3;   // 233 MB of words
  unsigned long long *h, *d, *sink;
  cudaHostAlloc(&h, n * 8, cudaHostAllocMapped);
  for (size_t i = 0; i < n; ++i) h[i] = i;
  cudaMalloc(&d, n * 8);
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaMemcpy(d, h, n * 8, cudaMemcpyHostToDevice);
  cudaEventRecord(a);
  for (int r = 0; r < 3; ++r) cudaMemcpyAsync(d, h, n * 8, cudaMemcpyHostToDevice);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("DMA H2D: %.1f GB/s\n", 3.0 * n * 8 / (ms * 1e-3) / 1e9);
  for (int wpc : {4, 14, 32}) {
    run<1, 1>(h, n, sink, wpc);
    run<1, 2>(h, n, sink, wpc);
    run<2, 1>(h, n, sink, wpc);
    run<1, 4>(h, n, sink, wpc);
  }
  return 0;
}
