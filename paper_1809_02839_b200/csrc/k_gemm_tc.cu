// K-A: tcgen05 tensor-core GEMMs of the dense stage path.
//
// Every stage GEMM is written as D[M×N] = Σ_k A(m,k)·B(n,k) with the WEIGHT-side
// dimension on M (TMEM lanes) so that the epilogue stores are coalesced along m:
//   fwd : M = out, N = B,  K = in ;  A(o,i) = W[i·out+o] (MN-major), B(b,i) = X[b·in+i]   (K-major)
//   dX  : M = in,  N = B,  K = out;  A(i,o) = W[i·out+o] (K-major),  B(b,o) = dZ[b·out+o] (K-major)
//   dW  : M = out, N = in, K = B  ;  A(o,b) = dZ[b·out+o] (MN-major), B(i,b) = X[b·in+i]  (MN-major)
// and the output element (m, n) always lives at out[n·M + m].
//
// Pipeline per CTA (one 128 × bn output tile, one K range), 6 warps, STAGES-deep ring:
//   warp 0      TMA producer: raw fp32 tiles → stage (K-major operands SWIZZLE_128B,
//               MN-major operands SWIZZLE_128B_ATOM_32B — the tf32 MN-major UMMA layout)
//   warps 2..5  converter (FP32X3 only): lo = x − trunc_tf32(x) in the same layout.
//               The tensor core truncates fp32 inputs to tf32 (tools/probe_tcgen05.cu),
//               so the raw tile itself is the "hi" operand: no rewrite, no transpose.
//   warp 1      MMA issuer: tcgen05.mma.cta_group::1.kind::tf32 (A, B from smem),
//               fp32 accumulator in TMEM (128 lanes × bn columns);
//               FP32X3 issues hi·hi + lo·hi + hi·lo
//   warps 2..5  epilogue: tcgen05.ld → fused bias/ReLU (fwd), ReLU mask (dX) → global;
//               split-K partials are reduced in fixed split order by the last CTA.
#include <cuda.h>

#include <mutex>

#include "kernels.hpp"

namespace st {

int64_t tc_workspace_bytes(int, int, int);
st_status launch_bias_grad(const float* dZ, int B, int n_out, float* gb, cudaStream_t s);

namespace {

constexpr int BM = 128;            // TMEM lanes per tile
constexpr int BNMAX = 128;         // accumulator columns per tile
constexpr int BK = 32;             // fp32 elements per 128-byte swizzle row
constexpr int kThreads = 192;
constexpr int TILE_BYTES = BM * BK * 4;   // 16 KB: one 128 × 32 fp32 operand tile
constexpr int STAGE_BYTES = 4 * TILE_BYTES;  // A raw (= hi), B raw (= hi), A lo, B lo
constexpr int smem_bytes(int stages) { return stages * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/; }

enum { EPI_FWD = 0, EPI_DX = 1, EPI_DW = 2 };

struct TcParams {
  int M, N, K;
  int kb_total, kb_per_split, splits;
  int bn;            // MMA N (multiple of 16, ≤ 128)
  float* out;        // out[n·M + m]
  const float* aux;  // fwd: bias[M]; dX: mask (same indexing as out)
  int relu;
  float* ws;         // split-K partials [splits][tiles][BNMAX][BM]
  int* counters;     // [tiles]
  uint32_t idesc;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accum) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(
          tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptors (sm_100 version 1).
// K-major operand: rows of 128 B (32 fp32 along K), SWIZZLE_128B, 8-row atoms of
// 1024 B (SBO); a K step of 8 tf32 advances the start address by 32 B.
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// MN-major operand (32-bit elements need SWIZZLE_128B_BASE32B): 32-element MN
// chunks of 128 B per k row, 32 k rows per chunk (4 KB → LBO), 4-row k groups
// of 512 B (SBO); a K step of 8 advances the start address by 1024 B.
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(4096 >> 4) << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)1 << 61);
}
template <bool MN>
__device__ __forceinline__ uint64_t op_desc(uint32_t base, int kk) {
  return MN ? desc_mnmajor(base + kk * 1024) : desc_kmajor(base + kk * 32);
}

// The tensor core truncates fp32 operands to tf32 (measured: tools/probe_tcgen05.cu),
// so the raw tile IS the "hi" operand and lo = x − trunc_tf32(x) is exact in fp32.
__device__ __forceinline__ float lo_part(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// lo = x − hi over `chunks` 16-byte chunks: elementwise, so it is layout-agnostic
// (raw and lo buffers share the same swizzled arrangement).
__device__ __forceinline__ void make_lo(const char* raw, char* lo, int chunks, int tid) {
  int c = tid;
  for (; c + 3 * 128 < chunks; c += 4 * 128) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = *reinterpret_cast<const float4*>(raw + (c + u * 128) * 16);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float4 l = make_float4(lo_part(v[u].x), lo_part(v[u].y), lo_part(v[u].z), lo_part(v[u].w));
      *reinterpret_cast<float4*>(lo + (c + u * 128) * 16) = l;
    }
  }
  for (; c < chunks; c += 128) {
    const float4 v = *reinterpret_cast<const float4*>(raw + c * 16);
    *reinterpret_cast<float4*>(lo + c * 16) = make_float4(lo_part(v.x), lo_part(v.y), lo_part(v.z), lo_part(v.w));
  }
}

template <int EPI, bool A_MN, bool B_MN, bool kX3, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  const uint32_t b_full = smem_u32(bars);            // TMA landed        (1 arrive + tx)
  const uint32_t b_conv = b_full + 8 * STAGES;       // lo tiles written  (4 converter warps)
  const uint32_t b_empty = b_conv + 8 * STAGES;      // MMAs done reading (tcgen05.commit)
  const uint32_t b_acc_full = b_empty + 8 * STAGES;  // accumulator complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * STAGES + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m_tile = blockIdx.x, n_tile = blockIdx.y, split = blockIdx.z;
  const int m0 = m_tile * BM, n0 = n_tile * BNMAX;
  const int kb0 = split * p.kb_per_split;
  const int kb1 = min(p.kb_total, kb0 + p.kb_per_split);
  const int nkb = kb1 - kb0;
  const int bn = p.bn;
  const int nbox_b = (bn + 31) / 32;
  const int b_chunks = B_MN ? nbox_b * 256 : bn * 8;  // 16-byte chunks of the B tile

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(b_full + 8 * s, 1);
      mbar_init(b_conv + 8 * s, 4);
      mbar_init(b_empty + 8 * s, 1);
    }
    mbar_init(b_acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(BNMAX));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)(TILE_BYTES + (B_MN ? nbox_b * 4096 : bn * BK * 4));
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        mbar_wait(b_empty + 8 * s, ((i / STAGES) & 1) ^ 1);
        const uint32_t full = b_full + 8 * s;
        mbar_expect_tx(full, bytes);
        const int k0 = (kb0 + i) * BK;
        const uint32_t dA = smem_u32(smem + s * STAGE_BYTES);
        const uint32_t dB = dA + TILE_BYTES;
        if (A_MN) {
#pragma unroll
          for (int c = 0; c < BM / 32; ++c) tma_load_2d(dA + c * 4096, &mapA, m0 + 32 * c, k0, full);
        } else {
          tma_load_2d(dA, &mapA, k0, m0, full);
        }
        if (B_MN) {
          for (int c = 0; c < nbox_b; ++c) tma_load_2d(dB + c * 4096, &mapB, n0 + 32 * c, k0, full);
        } else {
          tma_load_2d(dB, &mapB, k0, n0, full);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread)
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait((kX3 ? b_conv : b_full) + 8 * s, ph);
        tc_fence_after();
        const uint32_t a_hi = smem_u32(smem + s * STAGE_BYTES), b_hi = a_hi + TILE_BYTES;
        const uint32_t a_lo = a_hi + 2 * TILE_BYTES, b_lo = a_hi + 3 * TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
          tc_mma(tmem, op_desc<A_MN>(a_hi, kk), op_desc<B_MN>(b_hi, kk), p.idesc, acc);
          if (kX3) {
            tc_mma(tmem, op_desc<A_MN>(a_lo, kk), op_desc<B_MN>(b_hi, kk), p.idesc, 1u);
            tc_mma(tmem, op_desc<A_MN>(a_hi, kk), op_desc<B_MN>(b_lo, kk), p.idesc, 1u);
          }
        }
        tc_commit(b_empty + 8 * s);
      }
      tc_commit(b_acc_full);
    }
  } else {
    // ---------------- converter (warps 2..5): lo tiles for the 3xTF32 split
    const int ctid = threadIdx.x - 64;  // 0..127
    if (kX3) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        mbar_wait(b_full + 8 * s, (i / STAGES) & 1);
        char* st = smem + s * STAGE_BYTES;
        make_lo(st, st + 2 * TILE_BYTES, TILE_BYTES / 16, ctid);
        make_lo(st + TILE_BYTES, st + 3 * TILE_BYTES, b_chunks, ctid);
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(b_conv + 8 * s);
      }
    }

    // ---------------- epilogue: TMEM lane = m (this warp's quadrant), columns = n
    mbar_wait(b_acc_full, 0);
    tc_fence_after();
    const int quad = warp & 3;
    const int m = m0 + quad * 32 + lane;
    const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16);
    const int tiles = gridDim.x * gridDim.y;
    const int tile = n_tile * gridDim.x + m_tile;
    if (p.splits > 1) {
      float* wsp = p.ws + ((size_t)split * tiles + tile) * (BNMAX * BM);
      for (int c = 0; c < bn; c += 16) {
        float v[16];
        tc_ld16(trow + c, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) wsp[(size_t)(c + j) * BM + quad * 32 + lane] = v[j];
      }
      __threadfence();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (ctid == 0) {
        const int prev = atomicAdd(p.counters + tile, 1);
        *last_flag = (prev == p.splits - 1);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (*last_flag) {
        __threadfence();
        const float bias = (EPI == EPI_FWD && p.aux && m < p.M) ? p.aux[m] : 0.f;
        for (int c = 0; c < bn; ++c) {
          const int n = n0 + c;
          float acc = 0.f;
          for (int s = 0; s < p.splits; ++s)
            acc += __ldcg(p.ws + ((size_t)s * tiles + tile) * (BNMAX * BM) + (size_t)c * BM + quad * 32 + lane);
          if (m < p.M && n < p.N) {
            const size_t o = (size_t)n * p.M + m;
            float v = acc;
            if (EPI == EPI_FWD) {
              v += bias;
              if (p.relu) v = fmaxf(v, 0.f);
            } else if (EPI == EPI_DX) {
              if (p.aux && !(p.aux[o] > 0.f)) v = 0.f;
            }
            p.out[o] = v;
          }
        }
        if (ctid == 0) p.counters[tile] = 0;  // self-reset for the next launch
      }
    } else {
      const float bias = (EPI == EPI_FWD && p.aux && m < p.M) ? p.aux[m] : 0.f;
      for (int c = 0; c < bn; c += 16) {
        float v[16];
        tc_ld16(trow + c, v);
        if (m < p.M) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int n = n0 + c + j;
            if (n < p.N) {
              const size_t o = (size_t)n * p.M + m;
              float x = v[j];
              if (EPI == EPI_FWD) {
                x += bias;
                if (p.relu) x = fmaxf(x, 0.f);
              } else if (EPI == EPI_DX) {
                if (p.aux && !(p.aux[o] > 0.f)) x = 0.f;
              }
              p.out[o] = x;
            }
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BNMAX));
  }
}

// ------------------------------------------------------------------ host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 2D fp32 tensor [outer][inner] with row pitch `pitch` elements; box {32, box_outer}.
// K-major operands (inner = K) use SWIZZLE_128B; MN-major ones (inner = M or N) the
// 32-byte-atom variant the tf32 MN-major UMMA layout requires.
bool make_map(CUtensorMap* m, const float* base, int inner, int outer, int pitch, int box_outer, bool mn_major) {
  EncodeFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)pitch * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

uint32_t make_idesc(int bn, bool a_mn, bool b_mn) {
  uint32_t d = 0;
  d |= 1u << 4;                       // D format F32
  d |= 2u << 7;                       // A format TF32
  d |= 2u << 10;                      // B format TF32
  d |= (a_mn ? 1u : 0u) << 15;        // A major (0 = K, 1 = MN)
  d |= (b_mn ? 1u : 0u) << 16;        // B major
  d |= (uint32_t)(bn >> 3) << 17;     // N >> 3
  d |= (uint32_t)(BM >> 4) << 24;     // M >> 4
  return d;
}

// MMA N of a tile: the tile's columns rounded up to a multiple of 16 (≤ 128); the
// B box of K-major operands has exactly bn rows (OOB rows are zero-filled by TMA).
int bn_for(int N) { return std::max(16, (std::min(N, BNMAX) + 15) / 16 * 16); }

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

static thread_local int g_launches = 0;
constexpr size_t kCounterBytes = 64 * 1024;

template <int EPI, bool A_MN, bool B_MN>
st_status launch(const GemmArgs& g, int M, int N, int K, const CUtensorMap& ma, const CUtensorMap& mb, float* out,
                 const float* aux, int relu) {
  TcParams p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.kb_total = (K + BK - 1) / BK;
  const int mt = (M + BM - 1) / BM, nt = (N + BNMAX - 1) / BNMAX;
  int splits = 1;
  const int tiles = mt * nt;
  if (tiles < num_sms()) splits = std::min(num_sms() / tiles, p.kb_total);
  if (splits < 1) splits = 1;
  const size_t part_bytes = (size_t)BNMAX * BM * 4;
  const size_t ws_cap = (size_t)tc_workspace_bytes(0, 0, 0) - kCounterBytes;
  while (splits > 1 && ((size_t)splits * tiles * part_bytes > ws_cap || tiles > (int)(kCounterBytes / 4))) --splits;
  p.kb_per_split = (p.kb_total + splits - 1) / splits;
  p.splits = (p.kb_total + p.kb_per_split - 1) / p.kb_per_split;
  p.bn = bn_for(N);
  p.out = out;
  p.aux = aux;
  p.relu = relu;
  p.counters = reinterpret_cast<int*>(g.work);
  p.ws = reinterpret_cast<float*>(static_cast<char*>(g.work) + kCounterBytes);
  p.idesc = make_idesc(p.bn, A_MN, B_MN);
  dim3 grid(mt, nt, p.splits);
  constexpr int S = 3;
  auto kern = (g.mode == ST_GEMM_FP32X3) ? tc_gemm_kernel<EPI, A_MN, B_MN, true, S>
                                         : tc_gemm_kernel<EPI, A_MN, B_MN, false, S>;
  static bool attr_set[2] = {false, false};
  const int ai = g.mode == ST_GEMM_FP32X3 ? 1 : 0;
  if (!attr_set[ai]) {
    ST_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes(S)));
    attr_set[ai] = true;
  }
  kern<<<grid, kThreads, smem_bytes(S), g.stream>>>(ma, mb, p);
  ST_CUDA_TRY(cudaGetLastError());
  g_launches = 1;
  return ST_OK;
}

bool tma_ok(const void* p, int pitch) { return aligned16(p) && (pitch % 4) == 0; }

}  // namespace

int tc_last_launches() { return g_launches; }
// counters (64 KB, zero-initialised by the owner, self-resetting) + split-K partials
// for up to 2 × #SMs output tiles of 128 × 128 fp32.
int64_t tc_workspace_bytes(int, int, int) { return (int64_t)kCounterBytes + (int64_t)2 * 148 * BNMAX * BM * 4; }

st_status simt_fwd(const GemmArgs& g, const float* X, const float* W, const float* bias, float* Z, int relu);
st_status simt_dx(const GemmArgs& g, const float* dZ, const float* W, const float* mask, float* D);
st_status simt_dw(const GemmArgs& g, const float* X, const float* dZ, float* G, float* gb);
int simt_last_launches();

// fwd: M = out, N = B, K = in
st_status tc_fwd(const GemmArgs& g, const float* X, const float* W, const float* bias, float* Z, int relu) {
  if (!tma_ok(W, g.n_out) || !tma_ok(X, g.n_in) || !get_encode()) {
    // TMA needs 16-byte pitches (e.g. the 10-wide output layer): CUDA-core split-K path
    st_status s = simt_fwd(g, X, W, bias, Z, relu);
    g_launches = simt_last_launches();
    return s;
  }
  CUtensorMap ma, mb;
  if (!make_map(&ma, W, g.n_out, g.n_in, g.n_out, 32, true) || !make_map(&mb, X, g.n_in, g.B, g.n_in, bn_for(g.B), false))
    return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (fwd)");
  return launch<EPI_FWD, true, false>(g, g.n_out, g.B, g.n_in, ma, mb, Z, bias, relu);
}

// dX: M = in, N = B, K = out
st_status tc_dx(const GemmArgs& g, const float* dZ, const float* W, const float* mask, float* D) {
  if (!tma_ok(W, g.n_out) || !tma_ok(dZ, g.n_out) || !get_encode()) {
    st_status s = simt_dx(g, dZ, W, mask, D);
    g_launches = simt_last_launches();
    return s;
  }
  CUtensorMap ma, mb;
  if (!make_map(&ma, W, g.n_out, g.n_in, g.n_out, BM, false) || !make_map(&mb, dZ, g.n_out, g.B, g.n_out, bn_for(g.B), false))
    return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (dX)");
  return launch<EPI_DX, false, false>(g, g.n_in, g.B, g.n_out, ma, mb, D, mask, 0);
}

// dW: M = out, N = in, K = B
st_status tc_dw(const GemmArgs& g, const float* X, const float* dZ, float* G, float* gb) {
  if (!tma_ok(dZ, g.n_out) || !tma_ok(X, g.n_in) || !get_encode()) {
    st_status s = simt_dw(g, X, dZ, G, gb);
    g_launches = simt_last_launches();
    return s;
  }
  CUtensorMap ma, mb;
  if (!make_map(&ma, dZ, g.n_out, g.B, g.n_out, 32, true) || !make_map(&mb, X, g.n_in, g.B, g.n_in, 32, true))
    return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (dW)");
  ST_TRY((launch<EPI_DW, true, true>(g, g.n_out, g.n_in, g.B, ma, mb, G, nullptr, 0)));
  if (gb) {
    ST_TRY(launch_bias_grad(dZ, g.B, g.n_out, gb, g.stream));
    g_launches = 2;
  }
  return ST_OK;
}

}  // namespace st
