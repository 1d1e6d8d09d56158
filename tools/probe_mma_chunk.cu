// MMA rate probe, chunked (development tool): cycles per tcgen05.mma kind::tf32 when the
// MMAs come in chunks of `per` with one tcgen05.commit per chunk, the B operand rotating
// over a smem ring and (TS) the A operand over TMEM slots — the shape of the fwd / dX
// main loop — on 1 CTA or on every SM at once.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_mma_chunk tools/probe_mma_chunk.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t kdesc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint32_t idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t par) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  } while (!ok);
}

// mode bit0: TS (A from TMEM); bit1: rotate B over 4 smem stages / A over 4 TMEM slots;
// bit2: wait for the commit of chunk c-3 before issuing chunk c (a 3-deep ring)
// ncommit: commits per chunk (0: one commit every 4 chunks)
template <int PER, bool ELECT>
__global__ void rate(int per_rt, int mode, int chunks, int ncommit, long long* out) {
  constexpr int per = PER;
  extern __shared__ __align__(1024) uint8_t sm[];
  char* s = (char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) ((float*)s)[i] = 0.001f * (i % 97);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
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
  if (ELECT ? (warp == 0) : (threadIdx.x == 0)) {
    const uint32_t id = idesc(128, 128);
    long long t0 = clock64();
    for (int c = 0; c < chunks; ++c) {
      const int st = (mode & 2) ? (c & 3) : 0;
      if ((mode & 4) && c >= 3) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        wait(smem_u32(&bar[(c - 3) & 3]), ((c - 3) >> 2) & 1);
      }
      const uint32_t sa = smem_u32(s + st * 16384), sb = smem_u32(s + 65536 + st * 16384);
      const uint32_t ta = tm + 128 + st * 64;
#pragma unroll
      for (int j = 0; j < per; ++j) {
        const int kk = j & 3;
        uint32_t acc = (c | j) ? 1u : 0u;
        if (ELECT) {
          if (mode & 1)
            asm volatile("{\n .reg .pred p, e;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 p, %4, 0;\n @e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}"
                         ::"r"(tm), "r"(ta + kk * 8), "l"(kdesc(sb + kk * 32)), "r"(id), "r"(acc) : "memory");
          else
            asm volatile("{\n .reg .pred p, e;\n elect.sync _|e, 0xffffffff;\n setp.ne.b32 p, %4, 0;\n @e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                         ::"r"(tm), "l"(kdesc(sa + kk * 32)), "l"(kdesc(sb + kk * 32)), "r"(id), "r"(acc) : "memory");
        } else if (mode & 1)
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}"
                       ::"r"(tm), "r"(ta + kk * 8), "l"(kdesc(sb + kk * 32)), "r"(id), "r"(acc) : "memory");
        else
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
                       ::"r"(tm), "l"(kdesc(sa + kk * 32)), "l"(kdesc(sb + kk * 32)), "r"(id), "r"(acc) : "memory");
      }
      if (ELECT) {
        asm volatile("{\n .reg .pred e;\n elect.sync _|e, 0xffffffff;\n @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(&bar[c & 3])) : "memory");
      } else if (ncommit == 0) {
        if ((c & 3) == 3 || c == chunks - 1) commit(smem_u32(&bar[c & 3]));
      } else {
        commit(smem_u32(&bar[c & 3]));
        for (int q = 1; q < ncommit; ++q) commit(smem_u32(&bar[3 - (c & 3)]) + 0);
      }
    }
    // drain: wait for the last chunk's commit
    wait(smem_u32(&bar[(chunks - 1) & 3]), ((chunks - 1) >> 2) & 1);
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int PER, bool ELECT>
void run1(int mode, int nc, long long* out, int smem) {
  const int chunks = 2048, grid = 148;
  cudaFuncSetAttribute(rate<PER, ELECT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) {
    rate<PER, ELECT><<<grid, 128, smem>>>(PER, mode, chunks, nc, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
  }
  long long mx = 0;
  for (int i = 0; i < grid; ++i) mx = out[i] > mx ? out[i] : mx;
  printf("elect=%d commits=%d %s per=%2d (unrolled): %6.1f cycles/MMA  %7.1f cycles/chunk\n", (int)ELECT, nc,
         (mode & 1) ? "TS" : "SS", PER, mx / (double)(chunks * PER), mx / (double)chunks);
}

int main() {
  const int smem = 1024 + 160 * 1024;
  long long* out;
  cudaMallocManaged(&out, 148 * 8);
  for (int mode : {0, 1}) {
    run1<4, false>(mode, 1, out, smem);
    run1<12, false>(mode, 1, out, smem);
    run1<16, false>(mode, 1, out, smem);
    run1<4, true>(mode, 1, out, smem);
    run1<12, true>(mode, 1, out, smem);
    run1<16, true>(mode, 1, out, smem);
    run1<12, false>(mode, 0, out, smem);
  }
  return 0;
}
