// Microbenchmark / semantics probe for tcgen05 kind::tf32 on sm_100a (development tool,
// not part of the product path). Prints:
//   1. how raw fp32 inputs are reduced to tf32 (truncate vs round-to-nearest)
//   2. SS-mode MMA issue throughput (cycles per M=128,N=bn,K=8 MMA)
//   3. TS-mode (A from TMEM) correctness and throughput
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>
#include <cmath>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t kdesc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint32_t idesc(int M, int N, int amn = 0, int bmn = 0) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)amn << 15) | ((uint32_t)bmn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// MN-major SW128: 32-element MN chunks (128 B rows, one per k) of 32 k-rows (4 KB) per chunk;
// LBO = MN-chunk stride (4096 B), SBO = 8-k-row group stride (1024 B)
__device__ int g_lbo = 4096, g_sbo = 1024;
__device__ __forceinline__ uint64_t mdesc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(g_lbo >> 4) << 16) | ((uint64_t)(g_sbo >> 4) << 32) | (1ull << 46) |
         (1ull << 61);  // SWIZZLE_128B_BASE32B
}
__global__ void set_lbo(int l, int s) { g_lbo = l; g_sbo = s; }
__device__ __forceinline__ int mn_off(int r, int k) { return (r >> 5) * 4096 + k * 128 + ((((r & 31) >> 3) ^ (k & 3)) << 5) + (r & 7) * 4; }
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}"
               ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}"
               ::"r"(d), "r"(a_tmem), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
  } while (!ok);
}

// smem: A tile 128 rows x 128 B (K-major SW128), B tile 256 rows x 128 B
__global__ void probe(const float* A, const float* B, float* D, int bn, int iters, int mode, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  char* s = (char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  char* sa = s;
  char* sb = s + 128 * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // fill A (128 x 32 fp32 K-major swizzled) and B (bn x 32)
  for (int e = tid; e < 128 * 32; e += blockDim.x) {
    int r = e / 32, k = e % 32;
    int off = (mode >= 2) ? mn_off(r, k) : r * 128 + ((((k / 4) ^ (r & 7))) << 4) + (k % 4) * 4;
    *(float*)(sa + off) = A[r * 32 + k];
  }
  for (int e = tid; e < bn * 32; e += blockDim.x) {
    int r = e / 32, k = e % 32;
    int off = (mode == 3) ? mn_off(r, k) : r * 128 + ((((k / 4) ^ (r & 7))) << 4) + (k % 4) * 4;
    *(float*)(sb + off) = B[r * 32 + k];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
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
  const uint32_t acc_col = 0, a_col = 256;  // A operand in TMEM at columns 256..287
  if (mode == 1) {
    // A into TMEM: lane m, columns k (32 fp32 columns)
    if (warp < 4) {
      uint32_t v[32];
      for (int k = 0; k < 32; ++k) v[k] = __float_as_uint(A[(warp * 32 + lane) * 32 + k]);
      uint32_t taddr = tm + ((uint32_t)(warp * 32) << 16) + a_col;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                   ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                   "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
                   "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]),
                   "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  if (tid == 0) {
    const uint32_t id = idesc(128, bn, mode >= 2 ? 1 : 0, mode == 3 ? 1 : 0);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t acc = (it > 0 || kk > 0) ? 1u : 0u;
        if (mode == 0) mma_ss(tm + acc_col, kdesc(smem_u32(sa) + kk * 32), kdesc(smem_u32(sb) + kk * 32), id, acc);
        else if (mode == 2) mma_ss(tm + acc_col, mdesc(smem_u32(sa) + kk * 1024), kdesc(smem_u32(sb) + kk * 32), id, acc);
        else if (mode == 3) mma_ss(tm + acc_col, mdesc(smem_u32(sa) + kk * 1024), mdesc(smem_u32(sb) + kk * 1024), id, acc);
        else mma_ts(tm + acc_col, tm + a_col + kk * 8, kdesc(smem_u32(sb) + kk * 32), id, acc);
      }
    }
    commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    long long t1 = clock64();
    cyc[0] = t1 - t0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    for (int c = 0; c < bn; c += 16) {
      uint32_t r[16];
      uint32_t taddr = tm + ((uint32_t)(warp * 32) << 16) + acc_col + c;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                   : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 16; ++j) D[(warp * 32 + lane) * bn + c + j] = __uint_as_float(r[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  const int smem = 1024 + 128 * 128 + 256 * 128 + 8192;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  float *A, *B, *D;
  long long* cyc;
  cudaMallocManaged(&A, 128 * 32 * 4);
  cudaMallocManaged(&B, 256 * 32 * 4);
  cudaMallocManaged(&D, 128 * 256 * 4);
  cudaMallocManaged(&cyc, 8);
  // 1. rounding semantics: A = 1 + 3*2^-12 (between tf32 neighbours 1 and 1+2^-10), B = 1
  const float x = 1.0f + 3.0f * powf(2.f, -12);
  for (int i = 0; i < 128 * 32; ++i) A[i] = x;
  for (int i = 0; i < 256 * 32; ++i) B[i] = 1.0f;
  for (int mode = 0; mode < 2; ++mode) {
    probe<<<1, 128, smem>>>(A, B, D, 16, 1, mode, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %s: err=%s  D/32=%.10f  (trunc -> 1.0, rna -> %.10f, exact -> %.10f)\n", mode ? "TS" : "SS",
           cudaGetErrorString(e), D[0] / 32.0, 1.0 + 1.0 / 1024, (double)x);
  }
  // 2/3. correctness with random values vs fp64 (tf32-level tolerance), and throughput
  srand(1);
  for (int i = 0; i < 128 * 32; ++i) A[i] = (rand() % 2001 - 1000) / 1000.0f;
  for (int i = 0; i < 256 * 32; ++i) B[i] = (rand() % 2001 - 1000) / 1000.0f;
  int combos[4][2] = {{4096, 512}, {512, 4096}, {4096, 1024}, {1024, 4096}};
  for (int ci = 0; ci < 4; ++ci) {
    set_lbo<<<1, 1>>>(combos[ci][0], combos[ci][1]);
    cudaDeviceSynchronize();
    for (int mode = 2; mode < 4; ++mode) {
      int bn = 64;
      probe<<<1, 128, smem>>>(A, B, D, bn, 1, mode, cyc);
      cudaDeviceSynchronize();
      double maxerr = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < bn; ++n) {
          double ref = 0;
          for (int k = 0; k < 32; ++k) ref += (double)A[m * 32 + k] * B[n * 32 + k];
          maxerr = fmax(maxerr, fabs(ref - D[m * bn + n]));
        }
      printf("LBO=%d SBO=%d mode %d: maxerr %.3e\n", combos[ci][0], combos[ci][1], mode, maxerr);
    }
  }
  for (int bn : {128}) {
    for (int mode = 0; mode < 2; ++mode) {
      probe<<<1, 128, smem>>>(A, B, D, bn, 1, mode, cyc);
      cudaDeviceSynchronize();
      double maxerr = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < bn; ++n) {
          double ref = 0;
          for (int k = 0; k < 32; ++k) ref += (double)A[m * 32 + k] * B[n * 32 + k];
          maxerr = fmax(maxerr, fabs(ref - D[m * bn + n]));
        }
      probe<<<1, 128, smem>>>(A, B, D, bn, 1000, mode, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      printf("bn=%3d %s: max|err| (K=32) = %.3e ; %.1f cycles per MMA (M=128,N=%d,K=8) err=%s\n", bn, mode == 1 ? "TS" : (mode == 0 ? "SS" : (mode == 2 ? "SS-Amn" : "SS-ABmn")),
             maxerr, cyc[0] / 4000.0, bn, cudaGetErrorString(e));
    }
  }
  return 0;
}
