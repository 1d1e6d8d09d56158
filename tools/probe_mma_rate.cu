// MMA issue-rate probe (development tool): cycles per tcgen05.mma kind::tf32 for
// SS / TS modes and N = 128 / 256, alone and with 4 warps hammering shared memory.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t kdesc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint32_t idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__global__ void rate(int N, int ts, int noise, int iters, long long* out, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  char* s = (char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) ((float*)s)[i] = 0.001f * (i % 97);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tslot;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc(128, N);
    const uint32_t sa = smem_u32(s), sb = smem_u32(s + 16384);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
      for (int kk = 0; kk < 4; ++kk) {
        uint32_t acc = (it | kk) ? 1u : 0u;
        if (ts)
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}"
                       ::"r"(tm), "r"(tm + 256 + kk * 8), "l"(kdesc(sb + kk * 32)), "r"(id), "r"(acc) : "memory");
        else
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                       ::"r"(tm), "l"(kdesc(sa + kk * 32)), "l"(kdesc(sb + kk * 32)), "r"(id), "r"(acc) : "memory");
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    uint32_t ok = 0;
    do {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0) : "memory");
    } while (!ok);
    out[0] = clock64() - t0;
    stop = 1;
  } else if (warp >= 2 && noise) {
    // 4 warps: LDS.128 + STS.128 over a 64 KB region (96 KB offset), until the MMAs finish
    const int t = threadIdx.x - 64;
    float4 acc = make_float4(0, 0, 0, 0);
    char* base = s + 96 * 1024;
    long long n = 0;
    while (!stop) {
      for (int r = 0; r < 32; ++r) {
        int c = (t + r * 128) & 4095;
        float4 v = *(float4*)(base + c * 16);
        acc.x += v.x; acc.y += v.y;
        *(float4*)(base + ((c + 2048) & 4095) * 16) = v;
        ++n;
      }
    }
    if (acc.x == 12345.f) sink[0] = acc.y;
    if (t == 0) out[1] = n;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}
int main() {
  const int smem = 1024 + 160 * 1024;
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long* out; float* sink;
  cudaMallocManaged(&out, 16); cudaMallocManaged(&sink, 4);
  for (int N : {32, 64, 128, 256})
    for (int ts = 0; ts < 2; ++ts)
      for (int noise = 0; noise < 2; ++noise) {
        for (int rep = 0; rep < 2; ++rep) {
          out[1] = 0;
          rate<<<1, 192, smem>>>(N, ts, noise, 2000, out, sink);
          cudaError_t e = cudaDeviceSynchronize();
          if (rep) printf("N=%d %s noise=%d: %.1f cycles/MMA  (noise iters %lld) %s\n", N, ts ? "TS" : "SS", noise,
                          out[0] / 8000.0, out[1], cudaGetErrorString(e));
        }
      }
  // many CTAs at once (one per SM): is the rate per SM the same?
  return 0;
}
