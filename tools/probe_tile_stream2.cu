// DRAM access-pattern probe (development tool): the fused update's HBM stream (read W, V;
// write W', V') over an 8192 × 8192 fp32 pair, (a) linearly (float4 grid-stride) and
// (b) in the fused dW kernel's pattern: 128 × 128 tiles (W row-major [in][out], a tile =
// 128 rows × 512 B), tile t = m_t · n_tiles + n_t, G persistent CTAs each walking a
// contiguous range of tiles — and (c) the same tiles walked n-major across CTAs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_tile_stream2 tools/probe_tile_stream2.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void linear(float4* W, float4* V, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 w = __ldcs(W + i), v = __ldcs(V + i);
    v.x = 0.9f * v.x + 0.1f; v.y = 0.9f * v.y + 0.1f; v.z = 0.9f * v.z + 0.1f; v.w = 0.9f * v.w + 0.1f;
    w.x -= 1e-3f * v.x; w.y -= 1e-3f * v.y; w.z -= 1e-3f * v.z; w.w -= 1e-3f * v.w;
    __stcs(W + i, w);
    __stcs(V + i, v);
  }
}

// one CTA (1024 threads) per "persistent slot"; tile: 128 rows (n) × 128 floats (m)
template <bool NMAJOR>
__global__ void tiled(float* W, float* V, int M, int mt, int nt, int G) {
  const int tiles = mt * nt;
  const int b = blockIdx.x;
  const int t0 = (int)((long long)b * tiles / G), t1 = (int)((long long)(b + 1) * tiles / G);
  for (int tt = t0; tt < t1; ++tt) {
    int m_t, n_t;
    if (NMAJOR) { n_t = tt / mt; m_t = tt % mt; } else { m_t = tt / nt; n_t = tt % nt; }
    // 1024 threads: 32 float4 per row → 32 rows per pass, 4 passes
#pragma unroll
    for (int pass = 0; pass < 4; ++pass) {
      const int r = pass * 32 + (threadIdx.x >> 5);
      const size_t o = (size_t)(n_t * 128 + r) * M + m_t * 128 + (threadIdx.x & 31) * 4;
      float4 w = __ldcs(reinterpret_cast<float4*>(W + o)), v = __ldcs(reinterpret_cast<float4*>(V + o));
      v.x = 0.9f * v.x + 0.1f; v.y = 0.9f * v.y + 0.1f; v.z = 0.9f * v.z + 0.1f; v.w = 0.9f * v.w + 0.1f;
      w.x -= 1e-3f * v.x; w.y -= 1e-3f * v.y; w.z -= 1e-3f * v.z; w.w -= 1e-3f * v.w;
      __stcs(reinterpret_cast<float4*>(W + o), w);
      __stcs(reinterpret_cast<float4*>(V + o), v);
    }
  }
}

int main() {
  const int M = 8192, N = 8192;
  const size_t n = (size_t)M * N;
  float *W, *V;
  cudaMalloc(&W, n * 4);
  cudaMalloc(&V, n * 4);
  cudaMemset(W, 0, n * 4);
  cudaMemset(V, 0, n * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / 10;
    printf("%-34s %8.1f us  %7.1f GB/s (16 B/param)\n", name, us, 16.0 * n / us / 1e3);
  };
  timeit("linear float4, 148x8 CTAs", [&] { linear<<<148 * 8, 256>>>((float4*)W, (float4*)V, n / 4); });
  for (int G : {148, 296, 592}) {
    char buf[64];
    snprintf(buf, 64, "tiled m-major contiguous, G=%d", G);
    timeit(buf, [&] { tiled<false><<<G, 1024>>>(W, V, M, M / 128, N / 128, G); });
    snprintf(buf, 64, "tiled n-major contiguous, G=%d", G);
    timeit(buf, [&] { tiled<true><<<G, 1024>>>(W, V, M, M / 128, N / 128, G); });
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
