// HBM streaming patterns of the fused dW+update epilogue (development tool):
// read W, V and write W, V (16 B/param) over an 8192 x 8192 fp32 matrix, as
//  (a) a linear float4 grid-stride stream (K-B kernel pattern),
//  (b) 128x128 tiles, lane = row-contiguous m, 4 B per lane, 32 columns per batch
//      (the tc_dw_kernel epilogue pattern), tiles traversed n-major or m-major.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void linear(float4* W, float4* V, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 w = __ldcs(W + i), v = __ldcs(V + i);
    v.x = 0.9f * v.x + 0.1f; v.y = 0.9f * v.y + 0.1f; v.z = 0.9f * v.z + 0.1f; v.w = 0.9f * v.w + 0.1f;
    w.x -= 0.01f * v.x; w.y -= 0.01f * v.y; w.z -= 0.01f * v.z; w.w -= 0.01f * v.w;
    __stcs(W + i, w); __stcs(V + i, v);
  }
}
template <int J>
__global__ void __launch_bounds__(256) tiles(float* W, float* V, int M, int N, int order) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quad = warp & 3, half = warp >> 2;
  const int mt = M / 128, nt = N / 128, T = mt * nt;
  const int t0 = (long long)blockIdx.x * T / gridDim.x, t1 = (long long)(blockIdx.x + 1) * T / gridDim.x;
  for (int t = t0; t < t1; ++t) {
    const int m_t = order ? t % mt : t / nt, n_t = order ? t / mt : t % nt;
    const int m = m_t * 128 + quad * 32 + lane;
    for (int c = half * 64; c < half * 64 + 64; c += J) {
      const size_t o0 = (size_t)(n_t * 128 + c) * M + m;
      float w[J], v[J];
#pragma unroll
      for (int j = 0; j < J; ++j) { w[j] = __ldcs(W + o0 + (size_t)j * M); v[j] = __ldcs(V + o0 + (size_t)j * M); }
#pragma unroll
      for (int j = 0; j < J; ++j) {
        v[j] = 0.9f * v[j] + 0.1f; w[j] -= 0.01f * v[j];
        __stcs(W + o0 + (size_t)j * M, w[j]); __stcs(V + o0 + (size_t)j * M, v[j]);
      }
    }
  }
}
__global__ void fill(float* W, float* V, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned h = (unsigned)(i * 2654435761u);
    W[i] = (h & 0xffff) * 1e-5f - 0.3f;
    V[i] = ((h >> 16) & 0xffff) * 1e-6f;
  }
}
// 16 warps per CTA: 4 per lane quadrant, 32 columns each, J = 16 (the kernel's epilogue)
__global__ void __launch_bounds__(512) tiles16(float* W, float* V, int M, int N) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quad = warp & 3, part = warp >> 2;
  const int mt = M / 128, nt = N / 128, T = mt * nt;
  const int t0 = (long long)blockIdx.x * T / gridDim.x, t1 = (long long)(blockIdx.x + 1) * T / gridDim.x;
  for (int t = t0; t < t1; ++t) {
    const int m_t = t / nt, n_t = t % nt;
    const int m = m_t * 128 + quad * 32 + lane;
    for (int c = part * 32; c < part * 32 + 32; c += 16) {
      const size_t o0 = (size_t)(n_t * 128 + c) * M + m;
      float w[16], v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) { w[j] = __ldcs(W + o0 + (size_t)j * M); v[j] = __ldcs(V + o0 + (size_t)j * M); }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        v[j] = 0.9f * v[j] + 0.1f; w[j] -= 0.01f * v[j];
        __stcs(W + o0 + (size_t)j * M, w[j]); __stcs(V + o0 + (size_t)j * M, v[j]);
      }
    }
  }
}
__device__ __forceinline__ float ld_na(const float* p) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__global__ void __launch_bounds__(512) tiles16na(float* W, float* V, int M, int N) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quad = warp & 3, part = warp >> 2;
  const int mt = M / 128, nt = N / 128, T = mt * nt;
  const int t0 = (long long)blockIdx.x * T / gridDim.x, t1 = (long long)(blockIdx.x + 1) * T / gridDim.x;
  for (int t = t0; t < t1; ++t) {
    const int m_t = t / nt, n_t = t % nt;
    const int m = m_t * 128 + quad * 32 + lane;
    for (int c = part * 32; c < part * 32 + 32; c += 16) {
      const size_t o0 = (size_t)(n_t * 128 + c) * M + m;
      float w[16], v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) { w[j] = ld_na(W + o0 + (size_t)j * M); v[j] = ld_na(V + o0 + (size_t)j * M); }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        v[j] = 0.9f * v[j] + 0.1f; w[j] -= 0.01f * v[j];
        __stcs(W + o0 + (size_t)j * M, w[j]); __stcs(V + o0 + (size_t)j * M, v[j]);
      }
    }
  }
}
int main() {
  const int M = 8192, N = 8192;
  const size_t n = (size_t)M * N;
  float *W, *V;
  cudaMalloc(&W, n * 4); cudaMalloc(&V, n * 4);
  cudaMemset(W, 0, n * 4); cudaMemset(V, 0, n * 4);
  fill<<<1184, 256>>>(W, V, n);
  cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](const char* name, auto f) {
    f(); cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) f();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-40s %8.1f us  %7.1f GB/s\n", name, ms * 1e3 / 5, 16.0 * n / (ms / 5 * 1e-3) / 1e9);
  };
  run("linear float4 (1184 x 256)", [&] { linear<<<1184, 256>>>((float4*)W, (float4*)V, n / 4); });
  run("tiles J=32 m-major, 148 CTA x 8 warps", [&] { tiles<32><<<148, 256>>>(W, V, M, N, 0); });
  run("tiles J=32 n-major, 148 CTA x 8 warps", [&] { tiles<32><<<148, 256>>>(W, V, M, N, 1); });
  run("tiles J=16 n-major, 296 CTA", [&] { tiles<16><<<296, 256>>>(W, V, M, N, 1); });
  run("tiles J=16 m-major, 148 CTA x 16 warps", [&] { tiles16<<<148, 512>>>(W, V, M, N); });
  cudaFuncSetAttribute(tiles16, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(tiles16na, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  run("tiles16 + 100 KB smem", [&] { tiles16<<<148, 512, 100 * 1024>>>(W, V, M, N); });
  run("tiles16 + 160 KB smem", [&] { tiles16<<<148, 512, 160 * 1024>>>(W, V, M, N); });
  run("tiles16 + 220 KB smem", [&] { tiles16<<<148, 512, 220 * 1024>>>(W, V, M, N); });
  run("tiles16 no_allocate + 220 KB smem", [&] { tiles16na<<<148, 512, 220 * 1024>>>(W, V, M, N); });
  run("tiles J=32 m-major, 592 CTA", [&] { tiles<32><<<592, 256>>>(W, V, M, N, 0); });
  run("tiles J=32 n-major, 592 CTA", [&] { tiles<32><<<592, 256>>>(W, V, M, N, 1); });
  return 0;
}
