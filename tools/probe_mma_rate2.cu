// MMA rate probe, warp-converged issue (development tool): cycles per tcgen05.mma kind::tf32
// with A in TMEM (TS) and B from shared memory, for M = 64 / 128 and N = 64 / 128 / 256,
// issued the way the product kernels issue them (the whole warp runs the loop with the
// descriptors in uniform registers, one elected lane issues), on 1 CTA and on one CTA per SM.
// Values are garbage; only the rate is measured.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe2 tools/probe_mma_rate2.cu && /tmp/probe2
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t kdesc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}" : "=r"(pred)::"memory");
  return pred != 0;
}

__global__ void rate(int M, int N, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  char* s = (char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((float*)s)[i] = 0.001f * (i % 97);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
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
  if (warp == 0) {
    const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t sb = smem_u32(s);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t acc = (it | kk) ? 1u : 0u;
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(tm),
              "r"(tm + 256 + kk * 8), "l"(kdesc(sb + kk * 32)), "r"(id), "r"(acc)
              : "memory");
        }
      }
      __syncwarp();
    }
    if (elect_one())
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                   : "memory");
    __syncwarp();
    uint32_t ok = 0;
    do {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
          : "=r"(ok)
          : "r"(smem_u32(&bar)), "r"(0)
          : "memory");
    } while (!ok);
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  const int smem = 1024 + 64 * 1024;
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* out;
  cudaMallocManaged(&out, sizeof(long long) * 256);
  const int iters = 4000;
  for (int M : {64, 128})
    for (int N : {64, 128, 256})
      for (int grid : {1, sms}) {
        for (int rep = 0; rep < 2; ++rep) {
          rate<<<grid, 128, smem>>>(M, N, iters, out);
          cudaError_t e = cudaDeviceSynchronize();
          if (!rep) continue;
          long long mx = 0;
          for (int b = 0; b < grid; ++b) mx = out[b] > mx ? out[b] : mx;
          const double cyc = (double)mx / (iters * 4);
          printf("M=%3d N=%3d CTAs=%3d: %6.1f cycles/MMA  %7.0f flop/cycle/SM  %s\n", M, N, grid, cyc,
                 2.0 * M * N * 8 / cyc, cudaGetErrorString(e));
        }
      }
  return 0;
}
