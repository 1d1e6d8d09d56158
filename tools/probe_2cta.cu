// cta_group::2 tcgen05 MMA rate probe (development tool): a 2-CTA cluster issues
// M=256 (128 rows per CTA), N=128 (64 B rows per CTA), K=8 kind::tf32 MMAs (SS mode)
// and reports cycles per MMA and the correctness of the accumulator.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t kdesc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
template <int ts, int ALLOC>
__global__ void __cluster_dims__(2, 1, 1) probe2(const float* A, const float* B, float* D, int iters, int N,
                                                 long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  char* s = (char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  char* sa = s;            // 128 rows x 128 B (this CTA's half of A)
  char* sb = s + 16384;    // N/2 rows x 128 B (this CTA's half of B)
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cta_rank();
  for (int e = tid; e < 128 * 32; e += blockDim.x) {
    int r = e / 32, k = e % 32;
    *(float*)(sa + r * 128 + (((k / 4) ^ (r & 7)) << 4) + (k % 4) * 4) = A[(rank * 128 + r) * 32 + k];
  }
  for (int e = tid; e < (N / 2) * 32; e += blockDim.x) {
    int r = e / 32, k = e % 32;
    *(float*)(sb + r * 128 + (((k / 4) ^ (r & 7)) << 4) + (k % 4) * 4) = B[(rank * (N / 2) + r) * 32 + k];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "n"(ALLOC));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tslot;
  if (ts && warp < 4) {  // A row (rank*128 + warp*32 + lane) -> TMEM lane, columns 256..287
    uint32_t v[32];
    for (int k = 0; k < 32; ++k) v[k] = __float_as_uint(A[(rank * 128 + warp * 32 + lane) * 32 + k]);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
        ::"r"(tm + ((uint32_t)(warp * 32) << 16) + 256 % ALLOC), "r"(v[0]),"r"(v[1]),"r"(v[2]),"r"(v[3]),"r"(v[4]),"r"(v[5]),"r"(v[6]),"r"(v[7]),"r"(v[8]),"r"(v[9]),"r"(v[10]),"r"(v[11]),"r"(v[12]),"r"(v[13]),"r"(v[14]),"r"(v[15]),"r"(v[16]),"r"(v[17]),"r"(v[18]),"r"(v[19]),"r"(v[20]),"r"(v[21]),"r"(v[22]),"r"(v[23]),"r"(v[24]),"r"(v[25]),"r"(v[26]),"r"(v[27]),"r"(v[28]),"r"(v[29]),"r"(v[30]),"r"(v[31]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (rank == 0 && tid == 0) {
    const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
    long long t0 = clock64();
    cyc[1] = t0;
    for (int it = 0; it < iters; ++it)
      for (int kk = 0; kk < 4; ++kk) {
        uint32_t acc = (it | kk) ? 1u : 0u;
        if (ts) asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}"
                     ::"r"(tm), "r"(tm + 256 % ALLOC + kk * 8), "l"(kdesc(smem_u32(sb) + kk * 32)), "r"(id), "r"(acc) : "memory");
        else asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}"
                     ::"r"(tm), "l"(kdesc(smem_u32(sa) + kk * 32)), "l"(kdesc(smem_u32(sb) + kk * 32)), "r"(id), "r"(acc)
                     : "memory");
      }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");

  }
  // both CTAs wait for the MMAs
  {
    uint32_t ok = 0;
    do {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(ok) : "r"(smem_u32(&bar)), "r"(0) : "memory");
    } while (!ok);
  }
  if (rank == 0 && tid == 0) cyc[0] = clock64() - cyc[1];
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    for (int c = 0; c < N; c += 16) {
      uint32_t r[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                   : "r"(tm + ((uint32_t)(warp * 32) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 16; ++j) D[(rank * 128 + warp * 32 + lane) * N + c + j] = __uint_as_float(r[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(ALLOC));
}

int main() {
  const int smem = 1024 + 16384 + 16384;
  float *A, *B, *D;
  long long* cyc;
  cudaMallocManaged(&A, 256 * 32 * 4);
  cudaMallocManaged(&B, 256 * 32 * 4);
  cudaMallocManaged(&D, 256 * 256 * 4);
  cudaMallocManaged(&cyc, 16);
  srand(3);
  for (int i = 0; i < 256 * 32; ++i) A[i] = (rand() % 2001 - 1000) / 1000.0f;
  for (int i = 0; i < 256 * 32; ++i) B[i] = (rand() % 2001 - 1000) / 1000.0f;
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int N : {64, 128, 256}) {
      kern<<<2, 128, smem>>>(A, B, D, 1, N, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      double maxerr = 0;
      for (int m = 0; m < 256; ++m)
        for (int n = 0; n < N; ++n) {
          double ref = 0;
          for (int k = 0; k < 32; ++k) ref += (double)A[m * 32 + k] * B[n * 32 + k];
          maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
        }
      double best = 1e30;
      for (int rep = 0; rep < 5; ++rep) {
        kern<<<2, 128, smem>>>(A, B, D, 2000, N, cyc);
        cudaDeviceSynchronize();
        best = fmin(best, cyc[0] / 8000.0);
      }
      printf("cta_group::2 %s M=256 N=%d: maxerr %.3e (%s/%s); best-of-5 %.1f cycles per MMA\n", name, N, maxerr,
             cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()), best);
    }
  };
  run(probe2<0, 256>, "SS alloc256");
  run(probe2<0, 512>, "SS alloc512");
  run(probe2<1, 512>, "TS alloc512");
  return 0;
}
