// K-A: tcgen05 tensor-core GEMMs of the dense stage path.
//
// Every stage GEMM is written as D[M×N] = Σ_k A(m,k)·B(n,k) with the WEIGHT-side
// dimension on M (TMEM lanes) so that the epilogue stores are coalesced along m:
//   fwd : M = out, N = B,  K = in ;  A(o,i) = W[i·out+o] (MN-major), B(b,i) = X[b·in+i]   (K-major)
//   dX  : M = in,  N = B,  K = out;  A(i,o) = W[i·out+o] (K-major),  B(b,o) = dZ[b·out+o] (K-major)
//   dW  : M = out, N = in, K = B  ;  A(o,b) = dZ[b·out+o] (MN-major), B(i,b) = X[b·in+i]  (MN-major)
// and the output element (m, n) always lives at out[n·M + m].
//
// Pipeline per CTA (one 128 × bn output tile, one K range), 6 warps:
//   warp 0      TMA producer: raw fp32 tiles (128B-swizzled boxes) → raw ring
//   warps 2..5  converter: raw tile → K-major SW128 "hi" (and "lo" for FP32X3) tiles
//               (hi = cvt.rna.tf32(x), lo = x − hi; the 3xTF32 split),
//               transposing MN-major operands on the way → conv ring
//   warp 1      MMA issuer: tcgen05.mma.cta_group::1.kind::tf32, fp32 accumulator in
//               TMEM (128 lanes × bn columns); FP32X3 issues hi·hi + lo·hi + hi·lo
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
constexpr int RS = 3;              // raw (TMA) stages
constexpr int CS = 2;              // converted stages
constexpr int kThreads = 192;
constexpr int TILE_BYTES = BM * BK * 4;  // 16 KB for 128 rows
constexpr int RAW_STAGE = 2 * TILE_BYTES;
constexpr int CONV_STAGE = 4 * TILE_BYTES;  // A_hi, A_lo, B_hi, B_lo
constexpr int SMEM_BYTES = RS * RAW_STAGE + CS * CONV_STAGE + 1024 /*align*/ + 256 /*barriers*/;

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

// K-major, 128B-swizzled UMMA shared-memory descriptor (rows of 128 B, 8-row atoms of 1024 B).
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;               // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;     // SBO: 8-row group stride
  d |= (uint64_t)1 << 46;               // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;               // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// 16-byte chunk position inside a K-major SW128 tile: row r, chunk j (0..7)
__device__ __forceinline__ uint32_t kmaj_off(int r, int j) { return (uint32_t)(r * 128 + ((j ^ (r & 7)) << 4)); }

template <bool kX3>
__device__ __forceinline__ void split4(float4 v, float4& hi, float4& lo) {
  hi.x = tf32_hi(v.x);
  hi.y = tf32_hi(v.y);
  hi.z = tf32_hi(v.z);
  hi.w = tf32_hi(v.w);
  if (kX3) {
    lo.x = v.x - hi.x;
    lo.y = v.y - hi.y;
    lo.z = v.z - hi.z;
    lo.w = v.w - hi.w;
  }
}

// raw K-major tile (TMA SW128 box {32, rows}) → hi/lo K-major tiles: same physical chunk layout.
template <bool kX3>
__device__ __forceinline__ void convert_kmajor(const char* raw, char* hi, char* lo, int rows, int tid) {
  for (int c = tid; c < rows * 8; c += 128) {
    const float4 v = *reinterpret_cast<const float4*>(raw + c * 16);
    float4 h, l;
    split4<kX3>(v, h, l);
    *reinterpret_cast<float4*>(hi + c * 16) = h;
    if (kX3) *reinterpret_cast<float4*>(lo + c * 16) = l;
  }
}

// raw MN-major tile (rows/32 boxes {32 mn, 32 k}, each 4 KB, SW128) → K-major hi/lo tiles.
template <bool kX3>
__device__ __forceinline__ void convert_mnmajor(const char* raw, char* hi, char* lo, int rows, int tid) {
  for (int r = tid; r < rows; r += 128) {
    const char* box = raw + (r >> 5) * 4096;
    const int mm = r & 31;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float4 v;
      float* pv = reinterpret_cast<float*>(&v);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = 4 * j + q;
        pv[q] = *reinterpret_cast<const float*>(box + k * 128 + ((((mm >> 2) ^ (k & 7))) << 4) + (mm & 3) * 4);
      }
      float4 h, l;
      split4<kX3>(v, h, l);
      *reinterpret_cast<float4*>(hi + kmaj_off(r, j)) = h;
      if (kX3) *reinterpret_cast<float4*>(lo + kmaj_off(r, j)) = l;
    }
  }
}

template <int EPI, bool A_MN, bool B_MN, bool kX3>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  char* raw_base = smem;
  char* conv_base = smem + RS * RAW_STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(conv_base + CS * CONV_STAGE);
  // barrier layout
  const uint32_t b_raw_full = smem_u32(bars);
  const uint32_t b_raw_empty = b_raw_full + 8 * RS;
  const uint32_t b_conv_full = b_raw_empty + 8 * RS;
  const uint32_t b_conv_empty = b_conv_full + 8 * CS;
  const uint32_t b_acc_full = b_conv_empty + 8 * CS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * RS + 2 * CS + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m_tile = blockIdx.x, n_tile = blockIdx.y, split = blockIdx.z;
  const int m0 = m_tile * BM, n0 = n_tile * BNMAX;
  const int kb0 = split * p.kb_per_split;
  const int kb1 = min(p.kb_total, kb0 + p.kb_per_split);
  const int nkb = kb1 - kb0;
  const int bn = p.bn;

  if (threadIdx.x == 0) {
    for (int s = 0; s < RS; ++s) {
      mbar_init(b_raw_full + 8 * s, 1);
      mbar_init(b_raw_empty + 8 * s, 4);
    }
    for (int s = 0; s < CS; ++s) {
      mbar_init(b_conv_full + 8 * s, 4);
      mbar_init(b_conv_empty + 8 * s, 1);
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
      const int nbox_b = (bn + 31) / 32;
      const uint32_t bytes = (uint32_t)(BM * BK * 4 + (B_MN ? nbox_b * 4096 : bn * BK * 4));
      for (int i = 0; i < nkb; ++i) {
        const int s = i % RS;
        const uint32_t ph = (i / RS) & 1;
        mbar_wait(b_raw_empty + 8 * s, ph ^ 1);
        const uint32_t full = b_raw_full + 8 * s;
        mbar_expect_tx(full, bytes);
        const int k0 = (kb0 + i) * BK;
        const uint32_t dA = smem_u32(raw_base + s * RAW_STAGE);
        const uint32_t dB = dA + TILE_BYTES;
        if (A_MN) {
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
    // ---------------- MMA issuer
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % CS;
        const uint32_t ph = (i / CS) & 1;
        mbar_wait(b_conv_full + 8 * s, ph);
        tc_fence_after();
        const uint32_t base = smem_u32(conv_base + s * CONV_STAGE);
        const uint32_t a_hi = base, a_lo = base + TILE_BYTES, b_hi = base + 2 * TILE_BYTES,
                       b_lo = base + 3 * TILE_BYTES;
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          const uint32_t off = kk * 32;  // 8 tf32 = 32 bytes along the swizzled row
          const uint32_t acc = (i > 0 || kk > 0) ? 1u : 0u;
          tc_mma(tmem, kmajor_desc(a_hi + off), kmajor_desc(b_hi + off), p.idesc, acc);
          if (kX3) {
            tc_mma(tmem, kmajor_desc(a_lo + off), kmajor_desc(b_hi + off), p.idesc, 1u);
            tc_mma(tmem, kmajor_desc(a_hi + off), kmajor_desc(b_lo + off), p.idesc, 1u);
          }
        }
        tc_commit(b_conv_empty + 8 * s);
      }
      tc_commit(b_acc_full);
    }
  } else {
    // ---------------- converter (warps 2..5), then epilogue
    const int ctid = threadIdx.x - 64;  // 0..127
    for (int i = 0; i < nkb; ++i) {
      const int rs = i % RS, cs = i % CS;
      mbar_wait(b_raw_full + 8 * rs, (i / RS) & 1);
      mbar_wait(b_conv_empty + 8 * cs, ((i / CS) & 1) ^ 1);
      const char* rA = raw_base + rs * RAW_STAGE;
      const char* rB = rA + TILE_BYTES;
      char* cbase = conv_base + cs * CONV_STAGE;
      if (A_MN)
        convert_mnmajor<kX3>(rA, cbase, cbase + TILE_BYTES, BM, ctid);
      else
        convert_kmajor<kX3>(rA, cbase, cbase + TILE_BYTES, BM, ctid);
      if (B_MN)
        convert_mnmajor<kX3>(rB, cbase + 2 * TILE_BYTES, cbase + 3 * TILE_BYTES, bn, ctid);
      else
        convert_kmajor<kX3>(rB, cbase + 2 * TILE_BYTES, cbase + 3 * TILE_BYTES, bn, ctid);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(b_raw_empty + 8 * rs);
        mbar_arrive(b_conv_full + 8 * cs);
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
        for (int c = 0; c < bn; ++c) {
          const int n = n0 + c;
          float acc = 0.f;
          for (int s = 0; s < p.splits; ++s)
            acc += __ldcg(p.ws + ((size_t)s * tiles + tile) * (BNMAX * BM) + (size_t)c * BM + quad * 32 + lane);
          if (m < p.M && n < p.N) {
            const size_t o = (size_t)n * p.M + m;
            float v = acc;
            if (EPI == EPI_FWD) {
              if (p.aux) v += p.aux[m];
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
bool make_map(CUtensorMap* m, const float* base, int inner, int outer, int pitch, int box_outer) {
  EncodeFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)pitch * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
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

uint32_t make_idesc(int bn) {
  uint32_t d = 0;
  d |= 1u << 4;                       // D format F32
  d |= 2u << 7;                       // A format TF32
  d |= 2u << 10;                      // B format TF32
  d |= 0u << 15;                      // A K-major
  d |= 0u << 16;                      // B K-major
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
  p.idesc = make_idesc(p.bn);
  dim3 grid(mt, nt, p.splits);
  auto kern = (g.mode == ST_GEMM_FP32X3) ? tc_gemm_kernel<EPI, A_MN, B_MN, true> : tc_gemm_kernel<EPI, A_MN, B_MN, false>;
  static bool attr_set[2] = {false, false};
  const int ai = g.mode == ST_GEMM_FP32X3 ? 1 : 0;
  if (!attr_set[ai]) {
    ST_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    attr_set[ai] = true;
  }
  kern<<<grid, kThreads, SMEM_BYTES, g.stream>>>(ma, mb, p);
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

// fwd: M = out, N = B, K = in
st_status tc_fwd(const GemmArgs& g, const float* X, const float* W, const float* bias, float* Z, int relu) {
  if (!tma_ok(W, g.n_out) || !tma_ok(X, g.n_in) || !get_encode()) {
    g_launches = 1;
    return simt_fwd(g, X, W, bias, Z, relu);  // TMA needs 16-byte pitches (e.g. the 10-wide output layer)
  }
  CUtensorMap ma, mb;
  if (!make_map(&ma, W, g.n_out, g.n_in, g.n_out, 32) || !make_map(&mb, X, g.n_in, g.B, g.n_in, bn_for(g.B)))
    return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (fwd)");
  return launch<EPI_FWD, true, false>(g, g.n_out, g.B, g.n_in, ma, mb, Z, bias, relu);
}

// dX: M = in, N = B, K = out
st_status tc_dx(const GemmArgs& g, const float* dZ, const float* W, const float* mask, float* D) {
  if (!tma_ok(W, g.n_out) || !tma_ok(dZ, g.n_out) || !get_encode()) {
    g_launches = 1;
    return simt_dx(g, dZ, W, mask, D);
  }
  CUtensorMap ma, mb;
  if (!make_map(&ma, W, g.n_out, g.n_in, g.n_out, BM) || !make_map(&mb, dZ, g.n_out, g.B, g.n_out, bn_for(g.B)))
    return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (dX)");
  return launch<EPI_DX, false, false>(g, g.n_in, g.B, g.n_out, ma, mb, D, mask, 0);
}

// dW: M = out, N = in, K = B
st_status tc_dw(const GemmArgs& g, const float* X, const float* dZ, float* G, float* gb) {
  if (!tma_ok(dZ, g.n_out) || !tma_ok(X, g.n_in) || !get_encode()) {
    g_launches = gb ? 2 : 1;
    return simt_dw(g, X, dZ, G, gb);
  }
  CUtensorMap ma, mb;
  if (!make_map(&ma, dZ, g.n_out, g.B, g.n_out, 32) || !make_map(&mb, X, g.n_in, g.B, g.n_in, 32))
    return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (dW)");
  ST_TRY((launch<EPI_DW, true, true>(g, g.n_out, g.n_in, g.B, ma, mb, G, nullptr, 0)));
  if (gb) {
    ST_TRY(launch_bias_grad(dZ, g.B, g.n_out, gb, g.stream));
    g_launches = 2;
  }
  return ST_OK;
}

}  // namespace st
