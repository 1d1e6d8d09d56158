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
#include <atomic>
#include <mutex>
#include <set>
#include <tuple>
#include <cuda.h>

#include <cstdlib>
#include <mutex>

#include "knobs.hpp"
#include "kernels.hpp"
#include "tc_ptx.cuh"

namespace st {

int64_t tc_workspace_bytes(int, int, int);
int launch_bias_grad(const float* dZ, int rows, int n_out, float* gb, void* work, int64_t work_bytes,
                     cudaStream_t s);

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
  int dev_flags;     // development only (ST_GEMM_DEV_FLAGS): bit0 skip MMAs, bit1 skip converter math,
                     // bit2 / bit3 skip B / A loads, bit4 skip TMEM stores, bit5 skip tcgen05.wait::st
  UpdateArgs upd;    // dW fused with K-B: weight-block targets (index n·M + m, like out)
  int wv_stream;     // fused K-B: W / V chunks staged in smem by TMA (mapW / mapV valid)
  int wv_direct;     // with wv_stream: w', v' stored from registers (the slot is refilled as soon
                     // as the epilogue has read it) instead of TMA-stored out of the slot
  int lockstep;      // dW: CTA b owns m-tile b % m_tiles and the (b / m_tiles)-th part of its n-tiles, so
                     // concurrent CTAs stream adjacent 512-B segments of the same W / V rows
  int ext_reduce;    // split-K: every CTA only writes its partial; splitk_epilogue_kernel reduces
  int sk;            // stream-K (fwd / dX TS kernel): CTA b takes chunks [b·U/G, (b+1)·U/G) of
                     // the tile-major (tile, K-block) space, U = tiles · kb_total, G = gridDim.x
  int mt, tiles;     // stream-K: m tiles, total tiles (tile = n_tile · mt + m_tile)
  int row;           // output element (m, n) at out[m·N + n] (implicit-GEMM conv fwd / dX), else out[n·M + m]
  int split_acc;     // TMEM-A kernel: the two small 3xTF32 terms (lo·hi, hi·lo) in their own accumulator,
                     // added to the hi·hi one in fp32 by the epilogue (long-K dW chains: ~3× less error)
  int seg;           // TMEM-A kernel: > 0 — each accumulator sums at most `seg` K-blocks; the epilogue
                     // adds the segments in fp32 registers (round-to-nearest) while the MMAs fill the
                     // other accumulator. The tensor core's accumulation loses precision systematically
                     // with every step (the error of one accumulator grows linearly with its K length,
                     // profiles/r2_gemm_error_vs_splits.txt); short segments bound it.
  int cv_H, cv_W, cv_C;  // implicit-GEMM conv: NHWC image height, width, channels of the implicit operand
};

using namespace ptx;



// Development timeline (ST_GEMM_DEV_FLAGS bit 7): %globaltimer at fixed points of each
// CTA, written into the unused upper half of the split-K counter block.
__device__ __forceinline__ void dbg_mark(const TcParams& p, int slot) {
  if (p.dev_flags & 128) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    if (cta < 240) reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(p.counters) + 32768)[cta * 16 + slot] = t;
  }
}

__device__ __forceinline__ void dbg_put(const TcParams& p, int slot, uint64_t v) {
  if (p.dev_flags & 128) {
    const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    if (cta < 240) reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(p.counters) + 32768)[cta * 16 + slot] = v;
  }
}

// 16 output columns n0c .. n0c + 15 of row m: fused bias + ReLU (fwd) or ReLU mask (dX).
// All mask loads are issued before any store (out and aux may not alias, but the
// compiler cannot know that): one memory latency per 16 columns, not per column.
template <int EPI>
__device__ __forceinline__ void epilogue_store16(const TcParams& p, int m, int n0c, const float* acc, float bias) {
  const int nv = min(16, p.N - n0c);
  if (p.row) {
    // row-major output (implicit conv): this thread's 16 columns are contiguous; bias by
    // column; the dX mask has the output's indexing. float4 when the row pitch allows it.
    float v[16];
    float* dst = p.out + (size_t)m * p.N + n0c;
    const float* mk = (EPI == EPI_DX && p.aux) ? p.aux + (size_t)m * p.N + n0c : nullptr;
    if (nv == 16 && (p.N & 3) == 0) {
      float mv[16];
      if (mk) {
#pragma unroll
        for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(mv + j) = __ldg(reinterpret_cast<const float4*>(mk + j));
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float x = acc[j];
        if (EPI == EPI_FWD) {
          if (p.aux) x += __ldg(p.aux + n0c + j);
          if (p.relu) x = fmaxf(x, 0.f);
        } else if (EPI == EPI_DX && mk) {
          x = (mv[j] > 0.f) ? x : 0.f;
        }
        v[j] = x;
      }
#pragma unroll
      for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(dst + j) = *reinterpret_cast<const float4*>(v + j);
    } else {
      for (int j = 0; j < nv; ++j) {
        float x = acc[j];
        if (EPI == EPI_FWD) {
          if (p.aux) x += p.aux[n0c + j];
          if (p.relu) x = fmaxf(x, 0.f);
        } else if (EPI == EPI_DX && mk) {
          x = (mk[j] > 0.f) ? x : 0.f;
        }
        dst[j] = x;
      }
    }
    return;
  }
  if (EPI == EPI_DX && p.aux) {
    float mk[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) mk[j] = (j < nv) ? __ldg(p.aux + (size_t)(n0c + j) * p.M + m) : 0.f;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < nv) p.out[(size_t)(n0c + j) * p.M + m] = (mk[j] > 0.f) ? acc[j] : 0.f;
    return;
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (j < nv) {
      float v = acc[j];
      if (EPI == EPI_FWD) {
        v += bias;
        if (p.relu) v = fmaxf(v, 0.f);
      }
      p.out[(size_t)(n0c + j) * p.M + m] = v;
    }
  }
}

// Epilogue (4 warps, 128 threads): TMEM lane = m (the warp's quadrant), columns = n.
// Fused: fwd bias + ReLU, dX ReLU mask; split-K partials reduced in fixed split order
// by the last CTA of the tile (deterministic), counters self-reset.
template <int EPI>
__device__ __forceinline__ void epilogue(const TcParams& p, uint32_t tmem, int warp, int lane, int m0, int n0,
                                         int split, int tile, int tiles, int* last_flag, uint32_t b_acc_full,
                                         uint32_t tmem2 = 0) {
  mbar_wait(b_acc_full, 0);
  tc_fence_after();
  const int bn = p.bn;
  const int ctid = (warp - 2) * 32 + lane;
  if (ctid == 0) dbg_mark(p, 3);
  const int quad = warp & 3;
  const int m = m0 + quad * 32 + lane;
  const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16);
  const uint32_t trow2 = tmem2 + ((uint32_t)(quad * 32) << 16);  // second accumulator (tmem2 ≠ 0)
  if (p.splits > 1) {
    float* wsp = p.ws + ((size_t)split * tiles + tile) * (BNMAX * BM);
    for (int c = 0; c < bn; c += 16) {
      float v[16];
      tc_ld16(trow + c, v);
      if (tmem2) {
        float w2[16];
        tc_ld16(trow2 + c, w2);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] += w2[j];
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) wsp[(size_t)(c + j) * BM + quad * 32 + lane] = v[j];
    }
    if (p.ext_reduce) return;  // many splits: the parallel reduce kernel sums them
    __threadfence();
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (ctid == 0) {
      dbg_mark(p, 4);
      const int prev = atomicAdd(p.counters + tile, 1);
      *last_flag = (prev == p.splits - 1);
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (ctid == 0) dbg_mark(p, 5);
    if (*last_flag) {
      __threadfence();
      const float bias = (EPI == EPI_FWD && p.aux && m < p.M && !p.row) ? p.aux[m] : 0.f;
      // Fixed split order 0..S−1 (deterministic); this CTA's own partial comes from
      // TMEM, the others from the workspace. 32 columns per chunk with every global load
      // of the chunk (partials, dX mask) issued before the first use: the fix-up is
      // latency-bound, so the chunk count is what costs.
      for (int c = 0; c < bn; c += 32) {
        float acc[32], mk[32];
        const int nv = min(32, p.N - (n0 + c));
        if (EPI == EPI_DX && p.aux && m < p.M) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            mk[j] = (j < nv) ? __ldg(p.aux + (p.row ? (size_t)m * p.N + (n0 + c + j) : (size_t)(n0 + c + j) * p.M + m))
                             : 0.f;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = 0.f;
        for (int s = 0; s < p.splits; ++s) {
          float v[32];
          if (s == split) {
            tc_ld16_nowait(trow + c, reinterpret_cast<uint32_t*>(v));
            tc_ld16_nowait(trow + c + 16, reinterpret_cast<uint32_t*>(v + 16));
            tc_wait_ld();
            if (tmem2) {
              float w2[32];
              tc_ld16_nowait(trow2 + c, reinterpret_cast<uint32_t*>(w2));
              tc_ld16_nowait(trow2 + c + 16, reinterpret_cast<uint32_t*>(w2 + 16));
              tc_wait_ld();
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] += w2[j];
            }
          } else {
            const float* src = p.ws + ((size_t)s * tiles + tile) * (BNMAX * BM) + (size_t)c * BM + quad * 32 + lane;
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = (c + j < BNMAX) ? __ldcg(src + (size_t)j * BM) : 0.f;
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[j] += v[j];
        }
        if (m < p.M) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (j < nv) {
              float v = acc[j];
              if (EPI == EPI_FWD) {
                v += p.row ? (p.aux ? p.aux[n0 + c + j] : 0.f) : bias;
                if (p.relu) v = fmaxf(v, 0.f);
              } else if (EPI == EPI_DX) {
                if (p.aux && !(mk[j] > 0.f)) v = 0.f;
              }
              p.out[p.row ? (size_t)m * p.N + (n0 + c + j) : (size_t)(n0 + c + j) * p.M + m] = v;
            }
          }
        }
      }
      if (ctid == 0) p.counters[tile] = 0;  // self-reset for the next launch
      if (ctid == 0) dbg_mark(p, 6);
    }
  } else {
    const float bias = (EPI == EPI_FWD && p.aux && m < p.M && !p.row) ? p.aux[m] : 0.f;
    for (int c = 0; c < bn; c += 16) {
      float v[16];
      tc_ld16(trow + c, v);
      if (tmem2) {
        float w2[16];
        tc_ld16(trow2 + c, w2);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] += w2[j];
      }
      if (m < p.M) epilogue_store16<EPI>(p, m, n0 + c, v, bias);
    }
  }
}

// Implicit-GEMM 3×3 / pad-1 convolution (a10) on the same kernel: CV selects how the
// producer addresses the operands (NHWC activations through 4-D TMA boxes whose
// out-of-image part TMA zero-fills = the padding; no im2col buffer):
//   CV_FWD: M = P pixels, N = Cout, K = 9·Cin in (kh, kw, ci) order.  A = X shifted by
//           (kh−1, kw−1) [128 pixel rows × 32 ci, K-major]; B = W [K × Cout] MN-major.
//   CV_DX : M = P, N = Cin, K = 9·Cout in (kh, kw, co) order.  A = dZ shifted by
//           (1−kh, 1−kw) (the flipped kernel); B = W viewed as [9][Cin][Cout] (3-D map),
//           box {32 co, bn ci, 1}: K-major.
//   CV_DW : M = Cout, N = 9·Cin, K = P.  A = dZ [P × Cout] MN-major (2-D, as EPI_DW);
//           B = X shifted by (kh−1, kw−1) [32 pixels × 32 ci boxes, MN-major].
// CV_FWD / CV_DX write row-major (p.row): out[p·N + n] is NHWC.
//   CV_ROWS: plain 2-D operands (A K-major [M × K], B as B_MN says), row-major output —
//           the padded-im2col first conv (Cin = 3: 27 taps·channels padded to 32).
//   CV_DWT: dW with M = 9·Cin, N = Cout, K = P (for Cout < 128: no half-empty M tile).
//           A = X window boxes (MN-major, 32 ci × 32 pixels), B = dZ [P × Cout]
//           MN-major; row-major output = G[(tap, ci)·Cout + co].
enum { CV_NONE = 0, CV_FWD = 1, CV_DX = 2, CV_DW = 3, CV_ROWS = 4, CV_DWT = 5 };

// One ring stage of operand tiles: K-block k0 of the (m0, n0) tile, TMA into dA / dB,
// completing on `full` (plain 2-D operands, or the implicit-conv windows of CV).
template <bool A_MN, bool B_MN, int CV>
__device__ __forceinline__ void load_stage(const TcParams& p, const CUtensorMap* mA, const CUtensorMap* mB,
                                           uint32_t dA, uint32_t dB, uint32_t full, int m0, int n0, int k0,
                                           int nbox_b) {
  if (CV == CV_FWD || CV == CV_DX) {
    // K-block (kh, kw, c0): the 128-pixel tile [b0.., h0.., w0..] shifted by the tap
    const int HW = p.cv_H * p.cv_W;
    const int b0 = m0 / HW, r0 = m0 - b0 * HW, h0 = r0 / p.cv_W, w0 = r0 - h0 * p.cv_W;
    const int q = k0 / p.cv_C, c0 = k0 - q * p.cv_C, kh = q / 3, kw = q - 3 * kh;
    const int dh = (CV == CV_FWD) ? kh - 1 : 1 - kh, dw = (CV == CV_FWD) ? kw - 1 : 1 - kw;
    tma_load_4d(dA, mA, c0, w0 + dw, h0 + dh, b0, full);
    if (CV == CV_FWD) {
      for (int c = 0; c < nbox_b; ++c) tma_load_2d(dB + c * 4096, mB, n0 + 32 * c, k0, full);
    } else {
      tma_load_3d(dB, mB, c0, n0, q, full);
    }
    return;
  }
  if (CV == CV_DWT) {
    const int HW = p.cv_H * p.cv_W;
    const int b0 = k0 / HW, r0 = k0 - b0 * HW, h0 = r0 / p.cv_W, w0 = r0 - h0 * p.cv_W;
#pragma unroll
    for (int c = 0; c < BM / 32; ++c) {
      const int m = m0 + 32 * c, q = m / p.cv_C, ci0 = m - q * p.cv_C, kh = q / 3, kw = q - 3 * kh;
      tma_load_4d(dA + c * 4096, mA, ci0, w0 + kw - 1, h0 + kh - 1, b0, full);
    }
    for (int c = 0; c < nbox_b; ++c) tma_load_2d(dB + c * 4096, mB, n0 + 32 * c, k0, full);
    return;
  }
  if (CV == CV_DW) {
#pragma unroll
    for (int c = 0; c < BM / 32; ++c) tma_load_2d(dA + c * 4096, mA, m0 + 32 * c, k0, full);
    const int HW = p.cv_H * p.cv_W;
    const int b0 = k0 / HW, r0 = k0 - b0 * HW, h0 = r0 / p.cv_W, w0 = r0 - h0 * p.cv_W;
    for (int c = 0; c < nbox_b; ++c) {
      const int n = n0 + 32 * c, q = n / p.cv_C, ci0 = n - q * p.cv_C, kh = q / 3, kw = q - 3 * kh;
      tma_load_4d(dB + c * 4096, mB, ci0, w0 + kw - 1, h0 + kh - 1, b0, full);
    }
    return;
  }
  if (A_MN) {
#pragma unroll
    for (int c = 0; c < BM / 32; ++c) tma_load_2d(dA + c * 4096, mA, m0 + 32 * c, k0, full);
  } else {
    tma_load_2d(dA, mA, k0, m0, full);
  }
  if (B_MN) {
    for (int c = 0; c < nbox_b; ++c) tma_load_2d(dB + c * 4096, mB, n0 + 32 * c, k0, full);
  } else {
    tma_load_2d(dB, mB, k0, n0, full);
  }
}

template <int EPI, bool A_MN, bool B_MN, bool kX3, int STAGES, int CV = CV_NONE>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  char* smem = align_smem_1k(smem_raw);
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
        load_stage<A_MN, B_MN, CV>(p, &mapA, &mapB, dA, dB, full, m0, n0, k0, nbox_b);
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

    epilogue<EPI>(p, tmem, warp, lane, m0, n0, split, n_tile * gridDim.x + m_tile, gridDim.x * gridDim.y,
                  last_flag, b_acc_full);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BNMAX));
  }
}


// Persistent variant for the implicit-conv fwd / dX GEMMs (M = pixels: hundreds of
// small tiles, no K split). One CTA per SM walks tiles t = blockIdx.x + j·gridDim.x
// (m fastest: concurrent CTAs share the weight tile in L2); the operand ring runs on
// across tiles, and two TMEM accumulators let the epilogue of tile j (warps 6..9)
// overlap the MMAs of tile j+1. Warp 0 TMA, warp 1 MMA (warp-converged, elected
// issuing lane), warps 2..5 lo converters (3xTF32), warps 6..9 epilogue.
constexpr int kPThreads = 320;

template <int EPI, bool A_MN, bool B_MN, bool kX3, int STAGES, int CV>
__global__ void __launch_bounds__(kPThreads, 1)
    tc_gemm_persistent_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                              TcParams p, int mt, int tiles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  char* smem = align_smem_1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  const uint32_t b_full = smem_u32(bars);
  const uint32_t b_conv = b_full + 8 * STAGES;
  const uint32_t b_empty = b_conv + 8 * STAGES;
  const uint32_t acc_full = b_empty + 8 * STAGES;  // [2]
  const uint32_t acc_empty = acc_full + 16;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * STAGES + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nkb = p.kb_total;
  const int bn = p.bn;
  const int nbox_b = (bn + 31) / 32;
  const int b_chunks = B_MN ? nbox_b * 256 : bn * 8;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(b_full + 8 * s, 1);
      mbar_init(b_conv + 8 * s, 4);
      mbar_init(b_empty + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(acc_full + 8 * a, 1);
      mbar_init(acc_empty + 8 * a, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2 * BNMAX));
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
    // ---------------- TMA producer (ring continues across tiles)
    const uint32_t bytes = (uint32_t)(TILE_BYTES + (B_MN ? nbox_b * 4096 : bn * BK * 4));
    int it = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int m0 = (t % mt) * BM, n0 = (t / mt) * BNMAX;
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int s = it % STAGES;
        mbar_wait(b_empty + 8 * s, ((it / STAGES) & 1) ^ 1);
        const uint32_t full = b_full + 8 * s;
        const uint32_t dA = smem_u32(smem + s * STAGE_BYTES);
        if (elect_one()) {
          mbar_expect_tx(full, bytes);
          load_stage<A_MN, B_MN, CV>(p, &mapA, &mapB, dA, dA + TILE_BYTES, full, m0, n0, kb * BK, nbox_b);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    int it = 0, j = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++j) {
      const int buf = j & 1;
      const uint32_t d = tmem + (uint32_t)(buf * BNMAX);
      mbar_wait(acc_empty + 8 * buf, ((j >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int s = it % STAGES;
        mbar_wait((kX3 ? b_conv : b_full) + 8 * s, (it / STAGES) & 1);
        tc_fence_after();
        const uint32_t a_hi = smem_u32(smem + s * STAGE_BYTES), b_hi = a_hi + TILE_BYTES;
        const uint32_t a_lo = a_hi + 2 * TILE_BYTES, b_lo = a_hi + 3 * TILE_BYTES;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
            tc_mma(d, op_desc<A_MN>(a_hi, kk), op_desc<B_MN>(b_hi, kk), p.idesc, acc);
            if (kX3) {
              tc_mma(d, op_desc<A_MN>(a_lo, kk), op_desc<B_MN>(b_hi, kk), p.idesc, 1u);
              tc_mma(d, op_desc<A_MN>(a_hi, kk), op_desc<B_MN>(b_lo, kk), p.idesc, 1u);
            }
          }
          tc_commit(b_empty + 8 * s);
          if (kb == nkb - 1) tc_commit(acc_full + 8 * buf);
        }
        __syncwarp();
      }
    }
  } else if (warp < 6) {
    // ---------------- converters (warps 2..5): lo tiles for the 3xTF32 split
    if (kX3) {
      const int ctid = threadIdx.x - 64;
      int it = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(b_full + 8 * s, (it / STAGES) & 1);
          char* st = smem + s * STAGE_BYTES;
          make_lo(st, st + 2 * TILE_BYTES, TILE_BYTES / 16, ctid);
          make_lo(st + TILE_BYTES, st + 3 * TILE_BYTES, b_chunks, ctid);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(b_conv + 8 * s);
        }
      }
    }
  } else {
    // ---------------- epilogue (warps 6..9 → TMEM quadrants 2, 3, 0, 1)
    const int quad = warp & 3;
    int j = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++j) {
      const int buf = j & 1;
      const int m0 = (t % mt) * BM, n0 = (t / mt) * BNMAX;
      mbar_wait(acc_full + 8 * buf, (j >> 1) & 1);
      tc_fence_after();
      const int m = m0 + quad * 32 + lane;
      const uint32_t trow = tmem + (uint32_t)(buf * BNMAX) + ((uint32_t)(quad * 32) << 16);
      const float bias = (EPI == EPI_FWD && p.aux && m < p.M && !p.row) ? p.aux[m] : 0.f;
      for (int c = 0; c < bn; c += 16) {
        float v[16];
        tc_ld16(trow + c, v);
        if (m < p.M) epilogue_store16<EPI>(p, m, n0 + c, v, bias);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty + 8 * buf);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BNMAX));
  }
}


// FP32X3 persistent GEMM with the A operand in TMEM (A-from-TMEM MMAs): the implicit-conv
// fwd / dX / dW and the tall dense dW (LSTM / LM softmax: K = T·B rows).
// With A and B both read from smem by three MMAs per K step (plus the converter's
// passes), the persistent kernel above is bound by shared-memory bandwidth (~144 KB of
// smem traffic per 128 × 64 × 32 K-block vs ~576 MMA cycles). Here the converter warps
// read each raw window tile once and write hi / lo into a TMEM slot (tcgen05.st), and
// compute the weight lo tile in smem; the MMAs then read only the weight tiles from smem.
// Ring: CS stages × (A raw 16 KB + B raw 16 KB + B lo 16 KB), TMEM slot s ↔ stage s
// (64 columns: 32 hi + 32 lo), 2 accumulators × 128 columns: 256 + CS·64 ≤ 512.
// Work units u = split·tiles + tile (tile m-fastest); with p.splits > 1 every unit covers
// kb_per_split K-blocks and writes its partial tile to the workspace (the split-K layout
// of epilogue()), reduced in fixed split order by splitk_epilogue_kernel.
constexpr int CS = 4;
constexpr int CS_STAGE = 3 * TILE_BYTES;
constexpr int cs_smem_bytes() { return CS * CS_STAGE + 1024 + 256; }

// NARROW (MMA N ≤ 64, e.g. the 64-channel conv layers): B tiles are half size, so the ring
// is 6 stages of 32 KB and the accumulators 64 columns wide (TMEM 2·64 + 6·64 = 512).
template <bool NARROW>
constexpr int tsg_stage_bytes() { return TILE_BYTES + 2 * (NARROW ? TILE_BYTES / 2 : TILE_BYTES); }
template <bool NARROW>
constexpr int tsg_smem_bytes() { return (NARROW ? 6 : CS) * tsg_stage_bytes<NARROW>() + 1024 + 256; }

template <int EPI, bool A_MN, bool B_MN, int CV, bool NARROW = false>
__global__ void __launch_bounds__(kPThreads, 1)
    tc_tsg_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                      TcParams p, int mt, int tiles) {
  constexpr int NS = NARROW ? 6 : CS;                     // ring stages = TMEM A slots
  constexpr int BT = NARROW ? TILE_BYTES / 2 : TILE_BYTES;  // B raw / B lo tile bytes
  constexpr int STG = TILE_BYTES + 2 * BT;
  constexpr uint32_t AW = NARROW ? 64 : BNMAX;             // accumulator columns
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  char* smem = align_smem_1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NS * STG);
  const uint32_t b_full = smem_u32(bars);          // TMA landed (A + B)           [NS]
  const uint32_t b_ready = b_full + 8 * NS;        // TMEM hi/lo + B lo written    [NS] (4 warps)
  const uint32_t b_empty = b_ready + 8 * NS;       // MMAs done with stage + slot  [NS]
  const uint32_t acc_full = b_empty + 8 * NS;      // [2]
  const uint32_t acc_empty = acc_full + 16;        // [2] (4 epilogue warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * NS + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int units = tiles * p.splits;
  // K-block range of unit u
  auto kb_range = [&](int u, int& k0, int& k1) {
    const int sp = u / tiles;
    k0 = sp * p.kb_per_split;
    k1 = min(p.kb_total, k0 + p.kb_per_split);
  };
  const int bn = p.bn;
  const int nbox_b = (bn + 31) / 32;
  const int b_chunks = B_MN ? nbox_b * 256 : bn * 8;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(b_full + 8 * s, 1);
      mbar_init(b_ready + 8 * s, 4);
      mbar_init(b_empty + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(acc_full + 8 * a, 1);
      mbar_init(acc_empty + 8 * a, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
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
  const uint32_t tmemA = tmem + 2 * AW;  // NS slots of 64 columns

  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (warp == 0) {
    // ---------------- TMA producer (programmatic dependent launch: operands only after the
    // predecessor completed; a no-op without the launch attribute)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t bytes = (uint32_t)(TILE_BYTES + (B_MN ? nbox_b * 4096 : bn * BK * 4));
    int it = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int t = u % tiles, m0 = (t % mt) * BM, n0 = (t / mt) * BNMAX;
      int kb0, kb1;
      kb_range(u, kb0, kb1);
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const int s = it % NS;
        mbar_wait(b_empty + 8 * s, ((it / NS) & 1) ^ 1);
        const uint32_t full = b_full + 8 * s;
        const uint32_t dA = smem_u32(smem + s * STG);
        if (elect_one()) {
          mbar_expect_tx(full, bytes);
          load_stage<A_MN, B_MN, CV>(p, &mapA, &mapB, dA, dA + TILE_BYTES, full, m0, n0, kb * BK, nbox_b);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (A hi / lo from TMEM slot s, B hi / lo from smem)
    // j counts accumulator hand-offs: one per unit, or one per K segment (p.seg)
    int it = 0, j = 0;
    const bool sa = p.split_acc != 0 && p.seg == 0;  // small terms in their own accumulator
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int kb0, kb1;
      kb_range(u, kb0, kb1);
      int buf = 0;
      uint32_t d = tmem, d2 = tmem;
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const bool seg_start = p.seg ? ((kb - kb0) % p.seg == 0) : (kb == kb0);
        const bool seg_end = (kb == kb1 - 1) || (p.seg && (kb - kb0) % p.seg == p.seg - 1);
        if (seg_start) {
          buf = sa ? 0 : (j & 1);
          const uint32_t par = sa ? (uint32_t)(j & 1) : (uint32_t)((j >> 1) & 1);
          d = tmem + (uint32_t)buf * AW;
          d2 = sa ? tmem + AW : d;
          mbar_wait(acc_empty + 8 * buf, par ^ 1);
          tc_fence_after();
        }
        const int s = it % NS;
        mbar_wait(b_ready + 8 * s, (it / NS) & 1);
        tc_fence_after();
        const uint32_t b_hi = smem_u32(smem + s * STG) + TILE_BYTES, b_lo = b_hi + BT;
        const uint32_t a_hi = tmemA + s * 64, a_lo = a_hi + 32;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint32_t acc = (!seg_start || kk > 0) ? 1u : 0u;
            tc_mma_ts(d, a_hi + kk * 8, op_desc<B_MN>(b_hi, kk), p.idesc, acc);
            tc_mma_ts(d2, a_lo + kk * 8, op_desc<B_MN>(b_hi, kk), p.idesc, sa ? acc : 1u);
            tc_mma_ts(d2, a_hi + kk * 8, op_desc<B_MN>(b_lo, kk), p.idesc, 1u);
          }
          tc_commit(b_empty + 8 * s);
          if (seg_end) tc_commit(acc_full + 8 * buf);
        }
        __syncwarp();
        if (seg_end) ++j;
      }
    }
  } else if (warp < 6) {
    // ---------------- converters (warps 2..5): A row r → TMEM lane r (hi, lo); B lo in smem
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const int ctid = threadIdx.x - 64;
    int it = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int kb0, kb1;
      kb_range(u, kb0, kb1);
      for (int kb = kb0; kb < kb1; ++kb, ++it) {
        const int s = it % NS;
        mbar_wait(b_full + 8 * s, (it / NS) & 1);
        char* st = smem + s * STG;
        uint32_t hi[32], lo[32];
        if (A_MN) {
          // element (k, r): box r/32, row k (128 B), 32-byte atoms swizzled by k % 4
          const char* box = st + (r >> 5) * 4096;
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const float x =
                *reinterpret_cast<const float*>(box + q * 128 + ((((r & 31) >> 3) ^ (q & 3)) << 5) + (r & 7) * 4);
            hi[q] = __float_as_uint(x);
            lo[q] = __float_as_uint(lo_part(x));
          }
        } else {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 v = *reinterpret_cast<const float4*>(st + r * 128 + ((c ^ (r & 7)) << 4));
            hi[4 * c + 0] = __float_as_uint(v.x);
            hi[4 * c + 1] = __float_as_uint(v.y);
            hi[4 * c + 2] = __float_as_uint(v.z);
            hi[4 * c + 3] = __float_as_uint(v.w);
            lo[4 * c + 0] = __float_as_uint(lo_part(v.x));
            lo[4 * c + 1] = __float_as_uint(lo_part(v.y));
            lo[4 * c + 2] = __float_as_uint(lo_part(v.z));
            lo[4 * c + 3] = __float_as_uint(lo_part(v.w));
          }
        }
        make_lo(st + TILE_BYTES, st + TILE_BYTES + BT, b_chunks, ctid);
        fence_proxy_async();
        // the slot's previous MMAs are done: the producer refilled this stage only after
        // b_empty[s], which commits after every MMA that read TMEM slot s
        tc_fence_after();
        const uint32_t taddr = tmemA + s * 64 + ((uint32_t)(quad * 32) << 16);
        tc_st32(taddr, hi);
        tc_st32(taddr + 32, lo);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(b_ready + 8 * s);
      }
    }
  } else {
    // ---------------- epilogue (warps 6..9 → TMEM quadrants 2, 3, 0, 1)
    const int quad = warp & 3;
    int j = 0;
    const bool sa = p.split_acc != 0 && p.seg == 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int t = u % tiles, m0 = (t % mt) * BM, n0 = (t / mt) * BNMAX;
      const int m = m0 + quad * 32 + lane;
      if (p.seg) {
        // segmented: sum the unit's segments in registers (fixed order, round-to-nearest)
        int kb0, kb1;
        kb_range(u, kb0, kb1);
        const int nseg = (kb1 - kb0 + p.seg - 1) / p.seg;
        float run[BNMAX];
        for (int i = 0; i < nseg; ++i, ++j) {
          const int buf = j & 1;
          mbar_wait(acc_full + 8 * buf, (uint32_t)((j >> 1) & 1));
          tc_fence_after();
          const uint32_t trow = tmem + (uint32_t)buf * AW + ((uint32_t)(quad * 32) << 16);
#pragma unroll
          for (int c = 0; c < (int)AW; c += 16) {
            if (c < bn) {
              float v[16];
              tc_ld16(trow + c, v);
#pragma unroll
              for (int q = 0; q < 16; ++q) run[c + q] = i ? __fadd_rn(run[c + q], v[q]) : v[q];
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(acc_empty + 8 * buf);
        }
        if (p.splits > 1) {
          float* wsp = p.ws + ((size_t)(u / tiles) * tiles + t) * (BNMAX * BM);
#pragma unroll
          for (int c = 0; c < (int)AW; c += 16)
            if (c < bn) {
#pragma unroll
              for (int q = 0; q < 16; ++q) wsp[(size_t)(c + q) * BM + quad * 32 + lane] = run[c + q];
            }
        } else {
          const float bias = (EPI == EPI_FWD && p.aux && m < p.M && !p.row) ? p.aux[m] : 0.f;
#pragma unroll
          for (int c = 0; c < (int)AW; c += 16)
            if (c < bn && m < p.M) {
              float v[16];
#pragma unroll
              for (int q = 0; q < 16; ++q) v[q] = run[c + q];
              epilogue_store16<EPI>(p, m, n0 + c, v, bias);
            }
        }
        continue;
      }
      const int buf = sa ? 0 : (j & 1);
      mbar_wait(acc_full + 8 * buf, sa ? (uint32_t)(j & 1) : (uint32_t)((j >> 1) & 1));
      ++j;
      tc_fence_after();
      const uint32_t trow = tmem + (uint32_t)buf * AW + ((uint32_t)(quad * 32) << 16);
      const uint32_t trow2 = tmem + AW + ((uint32_t)(quad * 32) << 16);
      if (p.splits > 1) {
        float* wsp = p.ws + ((size_t)(u / tiles) * tiles + t) * (BNMAX * BM);
        for (int c = 0; c < bn; c += 16) {
          float v[16];
          tc_ld16(trow + c, v);
          if (sa) {
            float w2[16];
            tc_ld16(trow2 + c, w2);
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] += w2[q];
          }
#pragma unroll
          for (int q = 0; q < 16; ++q) wsp[(size_t)(c + q) * BM + quad * 32 + lane] = v[q];
        }
      } else {
        const float bias = (EPI == EPI_FWD && p.aux && m < p.M && !p.row) ? p.aux[m] : 0.f;
        for (int c = 0; c < bn; c += 16) {
          float v[16];
          tc_ld16(trow + c, v);
          if (sa) {
            float w2[16];
            tc_ld16(trow2 + c, w2);
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] += w2[q];
          }
          if (m < p.M) epilogue_store16<EPI>(p, m, n0 + c, v, bias);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty + 8 * buf);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// ---------------------------------------------------------------- stream-K
// First chunk of CTA b's range (b = G gives U).
__device__ __forceinline__ long long sk_begin(int b, int G, long long U) { return (long long)b * U / G; }
// The CTA whose range holds chunk x.
__device__ __forceinline__ int sk_owner(long long x, int G, long long U) {
  int b = (int)(((x + 1) * G + U - 1) / U) - 1;
  while (b + 1 < G && sk_begin(b + 1, G, U) <= x) ++b;
  while (b > 0 && sk_begin(b, G, U) > x) --b;
  return b;
}
// Partial slot of the segment (tile, CTA b): a CTA holds at most two partial segments,
// the one its range starts in (2b) and the one it ends in (2b + 1).
__device__ __forceinline__ size_t sk_slot(int tile, int b, int G, long long U, int kbt) {
  return (size_t)(sk_begin(b, G, U) >= (long long)tile * kbt ? 2 * b : 2 * b + 1);
}

// Stream-K segment epilogue (the 4 converter warps). The tile's segments belong to the
// consecutive CTAs b_first .. b_first + nseg − 1; a whole-tile segment stores directly,
// otherwise every segment writes its partial and the last CTA to arrive sums them in
// segment order (deterministic) and applies the fused epilogue. acc parity = segment
// count of this CTA & 1.
template <int EPI>
__device__ __forceinline__ void epilogue_sk(const TcParams& p, uint32_t tmem, int warp, int lane, int tile,
                                            long long U, int* last_flag, uint32_t b_acc_full, uint32_t parity) {
  mbar_wait(b_acc_full, parity);
  tc_fence_after();
  const int G = gridDim.x, b = blockIdx.x, kbt = p.kb_total;
  const int m0 = (tile % p.mt) * BM, n0 = (tile / p.mt) * BNMAX;
  const int bn = p.bn;
  const int ctid = (warp - 2) * 32 + lane;
  const int quad = warp & 3;
  const int m = m0 + quad * 32 + lane;
  const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16);
  const int b_first = sk_owner((long long)tile * kbt, G, U);
  const int nseg = sk_owner((long long)tile * kbt + kbt - 1, G, U) - b_first + 1;
  const float bias = (EPI == EPI_FWD && p.aux && m < p.M && !p.row) ? p.aux[m] : 0.f;
  if (nseg == 1) {
    for (int c = 0; c < bn; c += 16) {
      float v[16];
      tc_ld16(trow + c, v);
      if (m < p.M) epilogue_store16<EPI>(p, m, n0 + c, v, bias);
    }
    return;
  }
  float* wsp = p.ws + sk_slot(tile, b, G, U, kbt) * (BNMAX * BM);
  for (int c = 0; c < bn; c += 16) {
    float v[16];
    tc_ld16(trow + c, v);
#pragma unroll
    for (int j = 0; j < 16; ++j) wsp[(size_t)(c + j) * BM + quad * 32 + lane] = v[j];
  }
  __threadfence();
  asm volatile("bar.sync 1, 128;" ::: "memory");
  if (ctid == 0) *last_flag = (atomicAdd(p.counters + tile, 1) == nseg - 1);
  asm volatile("bar.sync 1, 128;" ::: "memory");
  const bool last = *last_flag;
  asm volatile("bar.sync 1, 128;" ::: "memory");  // the flag is reused by the next segment
  if (!last) return;
  __threadfence();
  for (int c = 0; c < bn; c += 32) {
    float acc[32], mk[32];
    const int nv = min(32, p.N - (n0 + c));
    if (EPI == EPI_DX && p.aux && m < p.M) {
#pragma unroll
      for (int j = 0; j < 32; ++j) mk[j] = (j < nv) ? __ldg(p.aux + (size_t)(n0 + c + j) * p.M + m) : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.f;
    for (int sgi = 0; sgi < nseg; ++sgi) {
      const int bs = b_first + sgi;
      float v[32];
      if (bs == b) {
        tc_ld16_nowait(trow + c, reinterpret_cast<uint32_t*>(v));
        tc_ld16_nowait(trow + c + 16, reinterpret_cast<uint32_t*>(v + 16));
        tc_wait_ld();
      } else {
        const float* src = p.ws + sk_slot(tile, bs, G, U, kbt) * (BNMAX * BM) + (size_t)c * BM + quad * 32 + lane;
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = (c + j < BNMAX) ? __ldcg(src + (size_t)j * BM) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] += v[j];
    }
    if (m < p.M) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (j < nv) {
          float v = acc[j];
          if (EPI == EPI_FWD) {
            v += bias;
            if (p.relu) v = fmaxf(v, 0.f);
          } else if (EPI == EPI_DX) {
            if (p.aux && !(mk[j] > 0.f)) v = 0.f;
          }
          p.out[(size_t)(n0 + c + j) * p.M + m] = v;
        }
      }
    }
  }
  if (ctid == 0) p.counters[tile] = 0;  // self-reset for the next launch
}

// ============================================================================
// FP32X3 forward / dX kernel: weights through TMEM (tcgen05.mma A-from-TMEM).
//
// The weight operand (A, 128 rows of W per tile, K-major for dX, MN-major for fwd)
// streams from HBM through a deep smem ring (RA × 16 KB). Converter warps read
// each raw tile once, write hi (= raw, the tensor core truncates) and
// lo = x − trunc_tf32(x) straight into a TMEM ring with tcgen05.st and release the
// smem slot immediately. The activation operand (B, K-major) arrives as hi + lo
// tiles by TMA (lo precomputed once per GEMM by split_lo_kernel). The MMA thread
// issues A_hi·B_hi + A_lo·B_hi + A_hi·B_lo per K step of 8, reading only B from smem.
// ============================================================================
#ifndef ST_TS_RA
#define ST_TS_RA 6
#endif
#ifndef ST_TS_RB
#define ST_TS_RB 3
#endif
constexpr int TS_RA = ST_TS_RA;          // weight (A) raw ring stages, 16 KB each
constexpr int TS_RB = ST_TS_RB;          // activation (B) ring stages, hi + lo ≤ 32 KB
constexpr int TS_TA = 6;                 // TMEM A slots (64 columns: 32 hi + 32 lo): 128 + 6·64 = 512
constexpr int TS_THREADS = 224;          // 7 warps
constexpr int TS_B_STAGE = 2 * BNMAX * BK * 4;
constexpr int ts_smem_bytes() { return TS_RA * TILE_BYTES + TS_RB * TS_B_STAGE + 1024 + 512; }


template <int EPI, bool A_MN>
__global__ void __launch_bounds__(TS_THREADS, 1)
    tc_ts_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                 const __grid_constant__ CUtensorMap mapBlo, TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  char* smem = align_smem_1k(smem_raw);
  char* ringA = smem;
  char* ringB = smem + TS_RA * TILE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ringB + TS_RB * TS_B_STAGE);
  const uint32_t a_full = smem_u32(bars);          // TMA landed (A)          [RA]
  const uint32_t a_free = a_full + 8 * TS_RA;      // converter read it       [RA]
  const uint32_t b_full = a_free + 8 * TS_RA;      // TMA landed (B hi + lo)  [RB]
  const uint32_t b_empty = b_full + 8 * TS_RB;     // MMA done with B         [RB]
  const uint32_t t_full = b_empty + 8 * TS_RB;     // TMEM A slot written     [TA]
  const uint32_t t_empty = t_full + 8 * TS_TA;     // MMA done with TMEM slot [TA]
  const uint32_t acc_full = t_empty + 8 * TS_TA;
  const uint32_t acc_empty = acc_full + 8;         // stream-K: epilogue drained the accumulator
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * TS_RA + 2 * TS_RB + 2 * TS_TA + 2);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m_tile = blockIdx.x, n_tile = blockIdx.y, split = blockIdx.z;
  const int m0 = m_tile * BM, n0 = n_tile * BNMAX;
  const int kb0 = split * p.kb_per_split;
  const int bn = p.bn;
  // this CTA's chunks g0 .. g0 + nkb − 1 of the tile-major (tile, K-block) space
  const int kbt = p.kb_total;
  const long long U = (long long)p.tiles * kbt;
  const int g0 = p.sk ? (int)sk_begin(blockIdx.x, gridDim.x, U) : (n_tile * gridDim.x + m_tile) * kbt + kb0;
  const int nkb = p.sk ? (int)sk_begin(blockIdx.x + 1, gridDim.x, U) - g0 : min(kbt, kb0 + p.kb_per_split) - kb0;
  const int mt = p.sk ? p.mt : (int)gridDim.x;
  const int tile0 = g0 / kbt, kbs0 = g0 - tile0 * kbt;  // first chunk: tile, K-block (walked incrementally)
  if (threadIdx.x == 0) dbg_mark(p, 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < TS_RA; ++s) {
      mbar_init(a_full + 8 * s, 1);
      mbar_init(a_free + 8 * s, 4);
    }
    for (int s = 0; s < TS_RB; ++s) {
      mbar_init(b_full + 8 * s, 1);
      mbar_init(b_empty + 8 * s, 1);
    }
    for (int s = 0; s < TS_TA; ++s) {
      mbar_init(t_full + 8 * s, 4);
      mbar_init(t_empty + 8 * s, 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapBlo)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) dbg_mark(p, 1);
  const uint32_t tmem = *tmem_slot;      // accumulator: columns [0, 128)
  const uint32_t tmemA = tmem + BNMAX;   // A ring: columns [128, 128 + 64·TA)

  if (warp == 0) {
    // ---------------- TMA producer, weights (A)
    if (lane == 0) {
      for (int i = 0, tile = tile0, kb = kbs0; i < nkb; ++i, kb = (kb + 1 == kbt) ? (++tile, 0) : kb + 1) {
        const int s = i % TS_RA;
        mbar_wait(a_free + 8 * s, ((i / TS_RA) & 1) ^ 1);
        const uint32_t full = a_full + 8 * s;
        if (p.dev_flags & 8) {
          mbar_arrive(full);
          continue;
        }
        mbar_expect_tx(full, TILE_BYTES);
        const int k0 = kb * BK, am0 = (tile % mt) * BM;
        const uint32_t dA = smem_u32(ringA + s * TILE_BYTES);
        if (A_MN) {
#pragma unroll
          for (int c = 0; c < BM / 32; ++c) tma_load_2d(dA + c * 4096, &mapA, am0 + 32 * c, k0, full);
        } else {
          tma_load_2d(dA, &mapA, k0, am0, full);
        }
      }
    }
  } else if (warp == 6) {
    // ---------------- TMA producer, activations (B hi + lo)
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)(2 * bn * BK * 4);
      for (int i = 0, tile = tile0, kb = kbs0; i < nkb; ++i, kb = (kb + 1 == kbt) ? (++tile, 0) : kb + 1) {
        const int s = i % TS_RB;
        mbar_wait(b_empty + 8 * s, ((i / TS_RB) & 1) ^ 1);
        const uint32_t full = b_full + 8 * s;
        if (p.dev_flags & 4) {
          mbar_arrive(full);
          continue;
        }
        mbar_expect_tx(full, bytes);
        const int k0 = kb * BK, bn0 = (tile / mt) * BNMAX;
        const uint32_t dB = smem_u32(ringB + s * TS_B_STAGE);
        tma_load_2d(dB, &mapB, k0, bn0, full);
        tma_load_2d(dB + BNMAX * BK * 4, &mapBlo, k0, bn0, full);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: the whole warp walks the loop (warp-uniform operands
    // stay in uniform registers), one elected lane issues
    {
      int seg = 0;
      for (int i = 0, kb = kbs0; i < nkb; ++i, kb = (kb + 1 == kbt) ? 0 : kb + 1) {
        const int sb = i % TS_RB, ta = i % TS_TA;
        const bool seg_start = (i == 0) || (kb == 0);
        const bool seg_end = (i == nkb - 1) || (kb + 1 == kbt);
        if (seg_start && seg > 0) mbar_wait(acc_empty, (seg - 1) & 1);  // stream-K: accumulator drained
        mbar_wait(t_full + 8 * ta, (i / TS_TA) & 1);
        mbar_wait(b_full + 8 * sb, (i / TS_RB) & 1);
        tc_fence_after();
        const uint32_t b_hi = smem_u32(ringB + sb * TS_B_STAGE), b_lo = b_hi + BNMAX * BK * 4;
        const uint32_t a_hi = tmemA + ta * 64, a_lo = a_hi + 32;
        const uint32_t acc0 = seg_start ? 0u : 1u;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            if (p.dev_flags & 1) break;
            tc_mma_ts(tmem, a_hi + kk * 8, desc_kmajor(b_hi + kk * 32), p.idesc, kk > 0 ? 1u : acc0);
            tc_mma_ts(tmem, a_lo + kk * 8, desc_kmajor(b_hi + kk * 32), p.idesc, 1u);
            if (!(p.dev_flags & 256)) tc_mma_ts(tmem, a_hi + kk * 8, desc_kmajor(b_lo + kk * 32), p.idesc, 1u);
          }
          tc_commit(b_empty + 8 * sb);
          tc_commit(t_empty + 8 * ta);
          if (seg_end) tc_commit(acc_full);
        }
        __syncwarp();
        if (seg_end) ++seg;
      }
      if (lane == 0) dbg_mark(p, 2);
    }
  } else {
    // ---------------- converter (warps 2..5): raw weight tile → TMEM hi / lo
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // tile row = TMEM lane
    int sk_seg = 0;
    for (int i = 0, tile = tile0, kb = kbs0; i < nkb; ++i, kb = (kb + 1 == kbt) ? (++tile, 0) : kb + 1) {
      const int s = i % TS_RA, ta = i % TS_TA;
      mbar_wait(a_full + 8 * s, (i / TS_RA) & 1);
      const char* t = ringA + s * TILE_BYTES;
      uint32_t hi[32], lo[32];
      if (p.dev_flags & 2) {
#pragma unroll
        for (int k = 0; k < 32; ++k) hi[k] = lo[k] = 0;
      } else if (A_MN) {
        // element (k, r): box r/32, row k (128 B), 32-byte atoms swizzled by k % 4
        const char* box = t + (r >> 5) * 4096;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float x = *reinterpret_cast<const float*>(box + k * 128 + ((((r & 31) >> 3) ^ (k & 3)) << 5) +
                                                          (r & 7) * 4);
          hi[k] = __float_as_uint(x);
          lo[k] = __float_as_uint(lo_part(x));
        }
      } else {
        // row r: 8 chunks of 16 B, SWIZZLE_128B
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 v = *reinterpret_cast<const float4*>(t + r * 128 + ((j ^ (r & 7)) << 4));
          hi[4 * j + 0] = __float_as_uint(v.x);
          hi[4 * j + 1] = __float_as_uint(v.y);
          hi[4 * j + 2] = __float_as_uint(v.z);
          hi[4 * j + 3] = __float_as_uint(v.w);
          lo[4 * j + 0] = __float_as_uint(lo_part(v.x));
          lo[4 * j + 1] = __float_as_uint(lo_part(v.y));
          lo[4 * j + 2] = __float_as_uint(lo_part(v.z));
          lo[4 * j + 3] = __float_as_uint(lo_part(v.w));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(a_free + 8 * s);  // smem slot can be refilled
      mbar_wait(t_empty + 8 * ta, ((i / TS_TA) & 1) ^ 1);
      tc_fence_after();
      const uint32_t taddr = tmemA + ta * 64 + ((uint32_t)(quad * 32) << 16);
      if (!(p.dev_flags & 16)) {
        tc_st32(taddr, hi);
        tc_st32(taddr + 32, lo);
        if (!(p.dev_flags & 32)) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(t_full + 8 * ta);
      if (p.sk) {
        if (i == nkb - 1 || kb + 1 == kbt) {
          epilogue_sk<EPI>(p, tmem, warp, lane, tile, U, last_flag, acc_full, (uint32_t)(sk_seg & 1));
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(acc_empty);
          ++sk_seg;
        }
      }
    }
    if (!p.sk)
      epilogue<EPI>(p, tmem, warp, lane, m0, n0, split, n_tile * gridDim.x + m_tile, gridDim.x * gridDim.y,
                    last_flag, acc_full);
    if (threadIdx.x == 64) dbg_mark(p, 7);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    if (lane == 0) dbg_mark(p, 8);
  }
}

// ============================================================================
// FP32X3 forward / dX kernel, CTA-pair form (tcgen05.mma.cta_group::2).
//
// Same dataflow as tc_ts_kernel, but a 2-CTA cluster computes one 256 × bn tile:
// each CTA converts ITS 128 weight rows into ITS TMEM (A-from-TMEM) and stages bn/2
// activation rows (hi + lo) in its smem; the leader CTA (rank 0) issues M = 256 MMAs
// that read both CTAs' operands and write each CTA's 128 accumulator lanes. Measured
// (tools/probe_2cta.cu): 64 cycles per M=256, N=128, K=8 MMA — 128 × 128 × 8 per SM
// every 64 cycles, against 94 for the single-CTA TS MMA.
// Cross-CTA protocol: B TMA loads of both CTAs complete on the LEADER's b_full
// (.cta_group::2 TMA), converters of both CTAs arrive remotely on the leader's t_full,
// and the leader's commits multicast to the b_empty / t_empty / acc_full barriers of both.
// ============================================================================
constexpr int TS2_RB = 4;                         // activation ring stages (hi + lo of bn/2 rows ≤ 16 KB)
constexpr int TS2_B_STAGE = 2 * (BNMAX / 2) * BK * 4;
constexpr int ts2_smem_bytes() { return TS_RA * TILE_BYTES + TS2_RB * TS2_B_STAGE + 1024 + 512; }

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
// TMA into this CTA's smem, completion signalled on an mbarrier of either CTA of the pair
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                                 uint32_t cluster_bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(cluster_bar)
      : "memory");
}
// 4-D (NHWC window) variant: coordinates (c, w, h, b), zero fill outside the image
__device__ __forceinline__ void tma_load_4d_pair(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                                 uint32_t cluster_bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(cluster_bar)
      : "memory");
}
__device__ __forceinline__ void tc_mma_ts2(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accum) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(
          tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void tc_commit2(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// SA: the two small 3xTF32 terms go to a second TMEM accumulator (4 A slots instead of 6),
// added to the hi·hi accumulator in fp32 by the epilogue (reading D24)
// CONV: B is the implicit 3×3 window of an NHWC activation (CV_FWD addressing, 64-pixel
// 4-D boxes per CTA) and its precomputed lo — the conv forward with the weights on M
// (Cout ≥ 256: full 256-row pair tiles), pixels on N, output NHWC as out[p·Cout + co].
template <int EPI, bool A_MN, bool SA = false, bool CONV = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TS_THREADS, 1)
    tc_ts2_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                  const __grid_constant__ CUtensorMap mapBlo, TcParams p) {
  constexpr int TA = SA ? 4 : TS_TA;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  char* smem = align_smem_1k(smem_raw);
  char* ringA = smem;
  char* ringB = smem + TS_RA * TILE_BYTES;
  // programmatic dependent launch (GemmArgs::pdl): let the next kernel of the stream launch
  // now; this kernel's own dependency on its predecessor is waited for by the B producer
  // only (the weights — operand A — are not written by the preceding kernel). Both are
  // no-ops without the launch attribute.
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  uint64_t* bars = reinterpret_cast<uint64_t*>(ringB + TS2_RB * TS2_B_STAGE);
  const uint32_t a_full = smem_u32(bars);          // TMA landed (A, own)              [RA]
  const uint32_t a_free = a_full + 8 * TS_RA;      // converter read it (own)          [RA]
  const uint32_t b_full = a_free + 8 * TS_RA;      // B hi + lo of BOTH CTAs (leader)  [RB]
  const uint32_t b_empty = b_full + 8 * TS2_RB;    // MMA done with B (multicast)      [RB]
  const uint32_t t_full = b_empty + 8 * TS2_RB;    // TMEM A slots of both (leader)    [TA]
  const uint32_t t_empty = t_full + 8 * TS_TA;     // MMA done with TMEM (multicast)   [TA]
  const uint32_t acc_full = t_empty + 8 * TS_TA;   // accumulator complete (multicast)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * TS_RA + 2 * TS2_RB + 2 * TS_TA + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int m_tile = blockIdx.x, n_tile = blockIdx.y, split = blockIdx.z;
  const int m0 = m_tile * BM, n0 = n_tile * BNMAX;
  const int kb0 = split * p.kb_per_split;
  const int nkb = min(p.kb_total, kb0 + p.kb_per_split) - kb0;
  const int bn = p.bn;
  const int bh = bn / 2;  // activation rows staged by this CTA
  if (threadIdx.x == 0) dbg_mark(p, 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < TS_RA; ++s) {
      mbar_init(a_full + 8 * s, 1);
      mbar_init(a_free + 8 * s, 4);
    }
    for (int s = 0; s < TS2_RB; ++s) {
      mbar_init(b_full + 8 * s, 1);
      mbar_init(b_empty + 8 * s, 1);
    }
    for (int s = 0; s < TS_TA; ++s) {
      mbar_init(t_full + 8 * s, 8);
      mbar_init(t_empty + 8 * s, 1);
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapBlo)) : "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmemA = tmem + (SA ? 2 : 1) * BNMAX;
  if (threadIdx.x == 0) dbg_mark(p, 1);

  if (warp == 0) {
    // ---------------- TMA producer, weights (A): this CTA's 128 rows (warp-converged loop,
    // elected lane issues: the tensor-map coordinates stay in uniform registers)
    {
      const bool oob = m0 >= p.M;  // padding CTA of an odd tile count: rows masked at the end
      uint64_t w_f = 0;
      for (int i = 0; i < nkb; ++i) {
        const int s = i % TS_RA;
        const uint64_t c0 = clock64();
        mbar_wait(a_free + 8 * s, ((i / TS_RA) & 1) ^ 1);
        w_f += clock64() - c0;
        const uint32_t full = a_full + 8 * s;
        const int k0 = (kb0 + i) * BK;
        const uint32_t dA = smem_u32(ringA + s * TILE_BYTES);
        if (elect_one()) {
          if (oob || (p.dev_flags & 8)) {
            mbar_arrive(full);
          } else {
            mbar_expect_tx(full, TILE_BYTES);
            if (A_MN) {
#pragma unroll
              for (int c = 0; c < BM / 32; ++c) tma_load_2d(dA + c * 4096, &mapA, m0 + 32 * c, k0, full);
            } else {
              tma_load_2d(dA, &mapA, k0, m0, full);
            }
          }
        }
        __syncwarp();
      }
      if (lane == 0) dbg_put(p, 15, w_f);
    }
  } else if (warp == 6) {
    // ---------------- TMA producer, activations: rows n0 + rank·bn/2 .. +bn/2 (hi + lo)
    {
      asm volatile("griddepcontrol.wait;" ::: "memory");  // the activations come from the previous kernel
      const uint32_t bytes = (uint32_t)(2 * 2 * bh * BK * 4);  // both CTAs, hi + lo
      for (int i = 0; i < nkb; ++i) {
        const int s = i % TS2_RB;
        mbar_wait(b_empty + 8 * s, ((i / TS2_RB) & 1) ^ 1);
        const uint32_t full_leader = map_to_rank(b_full + 8 * s, 0);
        const int k0 = (kb0 + i) * BK;
        const uint32_t dB = smem_u32(ringB + s * TS2_B_STAGE);
        if (elect_one()) {
          if (rank == 0) mbar_expect_tx(b_full + 8 * s, bytes);
          if (CONV) {
            const int HW = p.cv_H * p.cv_W, p0 = n0 + (int)rank * bh;
            const int b0 = p0 / HW, r0 = p0 - b0 * HW, h0 = r0 / p.cv_W, w0 = r0 - h0 * p.cv_W;
            const int q = k0 / p.cv_C, c0 = k0 - q * p.cv_C, kh = q / 3, kw = q - 3 * kh;
            tma_load_4d_pair(dB, &mapB, c0, w0 + kw - 1, h0 + kh - 1, b0, full_leader);
            tma_load_4d_pair(dB + (BNMAX / 2) * BK * 4, &mapBlo, c0, w0 + kw - 1, h0 + kh - 1, b0, full_leader);
          } else {
            tma_load_2d_pair(dB, &mapB, k0, n0 + (int)rank * bh, full_leader);
            tma_load_2d_pair(dB + (BNMAX / 2) * BK * 4, &mapBlo, k0, n0 + (int)rank * bh, full_leader);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA only): warp-converged loop, elected lane issues
    if (rank == 0) {
      uint64_t w_t = 0, w_b = 0, w_i = 0;
      for (int i = 0; i < nkb; ++i) {
        const int sb = i % TS2_RB, ta = i % TA;
        const uint64_t c0 = clock64();
        mbar_wait(t_full + 8 * ta, (i / TA) & 1);
        const uint64_t c1 = clock64();
        mbar_wait(b_full + 8 * sb, (i / TS2_RB) & 1);
        const uint64_t c2 = clock64();
        w_t += c1 - c0;
        w_b += c2 - c1;
        tc_fence_after();
        const uint32_t b_hi = smem_u32(ringB + sb * TS2_B_STAGE), b_lo = b_hi + (BNMAX / 2) * BK * 4;
        const uint32_t a_hi = tmemA + ta * 64, a_lo = a_hi + 32;
        const uint32_t acc0 = i > 0 ? 1u : 0u;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            if (p.dev_flags & 1) break;
            const uint32_t d2 = SA ? tmem + (uint32_t)BNMAX : tmem;
            tc_mma_ts2(tmem, a_hi + kk * 8, desc_kmajor(b_hi + kk * 32), p.idesc, kk > 0 ? 1u : acc0);
            tc_mma_ts2(d2, a_lo + kk * 8, desc_kmajor(b_hi + kk * 32), p.idesc, SA ? (kk > 0 ? 1u : acc0) : 1u);
            if (!(p.dev_flags & 256)) tc_mma_ts2(d2, a_hi + kk * 8, desc_kmajor(b_lo + kk * 32), p.idesc, 1u);
          }
          tc_commit2(b_empty + 8 * sb);
          tc_commit2(t_empty + 8 * ta);
        }
        __syncwarp();
        w_i += clock64() - c2;
      }
      if (elect_one()) tc_commit2(acc_full);
      __syncwarp();
      if (lane == 0) {
        dbg_mark(p, 2);
        dbg_put(p, 9, w_t);
        dbg_put(p, 10, w_b);
        dbg_put(p, 11, w_i);
      }
    }
  } else {
    // ---------------- converter (warps 2..5): raw weight tile → this CTA's TMEM hi / lo
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    uint64_t w_a = 0, w_e = 0, w_s = 0;
    // dX with a ReLU mask and no K split: the epilogue (these warps, after the last K-block)
    // reads a 128 × bn mask tile written long ago (the stashed activation, in HBM); pull it
    // into L2 ~16 K-blocks before the end, late enough that the weight stream does not evict it
    const int pf_at = (EPI == EPI_DX && p.aux && p.splits == 1 && !p.row) ? max(0, nkb - 16) : -1;
    for (int i = 0; i < nkb; ++i) {
      const int s = i % TS_RA, ta = i % TA;
      if (i == pf_at && m0 + r < p.M) {
        const float* mrow = p.aux + m0 + r;
        for (int n = n0; n < min(p.N, n0 + p.bn); ++n)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(mrow + (size_t)n * p.M));
      }
      const uint64_t c0 = clock64();
      mbar_wait(a_full + 8 * s, (i / TS_RA) & 1);
      w_a += clock64() - c0;
      const char* t = ringA + s * TILE_BYTES;
      uint32_t hi[32], lo[32];
      if (p.dev_flags & 2) {
#pragma unroll
        for (int k = 0; k < 32; ++k) hi[k] = lo[k] = 0;
      } else if (A_MN) {
        const char* box = t + (r >> 5) * 4096;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float x = *reinterpret_cast<const float*>(box + k * 128 + ((((r & 31) >> 3) ^ (k & 3)) << 5) +
                                                          (r & 7) * 4);
          hi[k] = __float_as_uint(x);
          lo[k] = __float_as_uint(lo_part(x));
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 v = *reinterpret_cast<const float4*>(t + r * 128 + ((j ^ (r & 7)) << 4));
          hi[4 * j + 0] = __float_as_uint(v.x);
          hi[4 * j + 1] = __float_as_uint(v.y);
          hi[4 * j + 2] = __float_as_uint(v.z);
          hi[4 * j + 3] = __float_as_uint(v.w);
          lo[4 * j + 0] = __float_as_uint(lo_part(v.x));
          lo[4 * j + 1] = __float_as_uint(lo_part(v.y));
          lo[4 * j + 2] = __float_as_uint(lo_part(v.z));
          lo[4 * j + 3] = __float_as_uint(lo_part(v.w));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(a_free + 8 * s);
      const uint64_t c1 = clock64();
      mbar_wait(t_empty + 8 * ta, ((i / TA) & 1) ^ 1);
      const uint64_t c2 = clock64();
      w_e += c2 - c1;
      tc_fence_after();
      const uint32_t taddr = tmemA + ta * 64 + ((uint32_t)(quad * 32) << 16);
      if (!(p.dev_flags & 16)) {
        tc_st32(taddr, hi);
        tc_st32(taddr + 32, lo);
        if (!(p.dev_flags & 32)) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(map_to_rank(t_full + 8 * ta, 0));
      w_s += clock64() - c2;
    }
    if (threadIdx.x == 64) {
      dbg_put(p, 12, w_a);
      dbg_put(p, 13, w_e);
      dbg_put(p, 14, w_s);
    }
    epilogue<EPI>(p, tmem, warp, lane, m0, n0, split, n_tile * gridDim.x + m_tile, gridDim.x * gridDim.y,
                  last_flag, acc_full, SA ? tmem + (uint32_t)BNMAX : 0u);
    if (threadIdx.x == 64) dbg_mark(p, 7);
  }

  tc_fence_before();
  cluster_sync_all();  // no CTA leaves while the pair's MMAs may still touch its smem / TMEM
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// Split-K reduction for many splits (ext_reduce): one thread per output (n, m), the
// partials of all splits loaded independently (4 at a time) and summed in fixed split
// order 0..S−1 — the same order as the in-kernel fix-up — then the fused epilogue.
// The last-CTA fix-up walks the splits serially (one memory latency per split and
// chunk), which dominated GEMMs with a long K (e.g. the LSTM dh GEMM, K = 4H = 6000).
template <int EPI>
__global__ void splitk_epilogue_kernel(const float* __restrict__ ws, int splits, int tiles, int mt_grid, int M, int N,
                                       float* __restrict__ out, const float* __restrict__ aux, int relu, int row) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the partials of the preceding GEMM
  const int64_t total = (int64_t)M * N;
  const size_t split_stride = (size_t)tiles * BNMAX * BM;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i % M);
    const int n = (int)(i / M);
    const int tile = (n / BNMAX) * mt_grid + m / BM;
    const float* src = ws + ((size_t)tile * BNMAX + n % BNMAX) * BM + m % BM;
    float acc = 0.f;
    int s = 0;
    for (; s + 4 <= splits; s += 4) {
      const float a0 = __ldcg(src + (size_t)s * split_stride), a1 = __ldcg(src + (size_t)(s + 1) * split_stride);
      const float a2 = __ldcg(src + (size_t)(s + 2) * split_stride), a3 = __ldcg(src + (size_t)(s + 3) * split_stride);
      acc += a0;
      acc += a1;
      acc += a2;
      acc += a3;
    }
    for (; s < splits; ++s) acc += __ldcg(src + (size_t)s * split_stride);
    const int64_t o = row ? (int64_t)m * N + n : i;  // row: out[m·N + n]
    if (EPI == EPI_FWD) {
      if (aux) acc += aux[row ? n : m];
      if (relu) acc = fmaxf(acc, 0.f);
    } else if (EPI == EPI_DX) {
      if (aux && !(aux[o] > 0.f)) acc = 0.f;
    }
    out[o] = acc;
  }
}

// cudaLaunchKernelEx with programmatic stream serialization when pdl (GemmArgs::pdl)
template <typename... KArgs, typename... Args>
st_status launch_maybe_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                           Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  if (pdl) {
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  ST_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
  return ST_OK;
}

template <int EPI>
st_status launch_splitk_epilogue(const TcParams& p, int tiles, int mt_grid, cudaStream_t s, bool pdl = false) {
  const int64_t total = (int64_t)p.M * p.N;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)device_sm_count() * 8);
  return launch_maybe_pdl(pdl, splitk_epilogue_kernel<EPI>, dim3(blocks), dim3(256), 0, s, p.ws, p.splits, tiles,
                          mt_grid, p.M, p.N, p.out, p.aux, p.relu, p.row);
}

// lo = x − trunc_tf32(x) of a whole [rows × pitch] activation matrix (the B operand
// of the FP32X3 forward / dX GEMMs), computed once per GEMM.
__global__ void split_lo_kernel(const float4* __restrict__ x, float4* __restrict__ lo, size_t n4) {
  // programmatic dependent launch (no-ops without the attribute): successor may launch;
  // x is complete only after the wait
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = x[i];
    lo[i] = make_float4(lo_part(v.x), lo_part(v.y), lo_part(v.z), lo_part(v.w));
  }
}



// K-B update of J elements at o0 + j·stride (j < J) of one parameter block given their
// gradients g[j]: all loads first (J·2 in flight), then the Eq. 1 / apply / Eq. 4 math.
template <int J>
__device__ __forceinline__ void update_cols(const UpdateArgs& u, size_t o0, size_t stride, const float* g) {
  float w[J], v[J];
  const float* pw = u.W + o0;
  const float* pv = u.V + o0;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    w[j] = __ldcs(pw + j * stride);
    v[j] = __ldcs(pv + j * stride);
  }
  float* qw = u.W + o0;
  float* qv = u.V + o0;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    v[j] = __fmaf_rn(u.c.c_gamma, v[j], __fmul_rn(u.c.c_one, g[j]));
    w[j] = __fmaf_rn(-u.c.c_eta, v[j], w[j]);
    __stcs(qw + j * stride, w[j]);
    __stcs(qv + j * stride, v[j]);
  }
  if (u.WF) {
    float* qf = u.WF + o0;
#pragma unroll
    for (int j = 0; j < J; ++j) qf[j * stride] = __fmaf_rn(-u.c.c_f, v[j], w[j]);
  }
  if (u.WB) {
    float* qb = u.WB + o0;
#pragma unroll
    for (int j = 0; j < J; ++j) qb[j * stride] = __fmaf_rn(-u.c.c_b, v[j], w[j]);
  }
}


// 4×4 transpose inside each lane quad: lane r (= lane & 3) holds row r of a 4×4 block
// (a[x] = M[r][x]); afterwards it holds column r (a[x] = M[x][r]).
__device__ __forceinline__ void quad_transpose4(float* a, int r) {
  float x0 = (r & 1) ? a[0] : a[1];
  float x1 = (r & 1) ? a[2] : a[3];
  x0 = __shfl_xor_sync(0xffffffffu, x0, 1);
  x1 = __shfl_xor_sync(0xffffffffu, x1, 1);
  if (r & 1) {
    a[0] = x0;
    a[2] = x1;
  } else {
    a[1] = x0;
    a[3] = x1;
  }
  float y0 = (r & 2) ? a[0] : a[2];
  float y1 = (r & 2) ? a[1] : a[3];
  y0 = __shfl_xor_sync(0xffffffffu, y0, 2);
  y1 = __shfl_xor_sync(0xffffffffu, y1, 2);
  if (r & 2) {
    a[0] = y0;
    a[1] = y1;
  } else {
    a[2] = y0;
    a[3] = y1;
  }
}

// Fused K-B on a full 32-row × 16-column block held by one warp after tcgen05.ld
// (lane = row m0w + lane, v[j] = g of column n0c + j). Each lane quad transposes so
// that lane q·4 + r owns rows m0w + 4q .. +3 of columns n0c + 4i + r (i = 0..3):
// float4 loads / stores, 4× fewer memory instructions than the lane-per-row form.
__device__ __forceinline__ void update_block16_vec(const UpdateArgs& u, size_t M, int m0w, int n0c, int lane,
                                                   float* v) {
  const int q = lane >> 2, r = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i) quad_transpose4(v + 4 * i, r);
  float4 w4[4], v4[4];
  size_t o[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    o[i] = (size_t)(n0c + 4 * i + r) * M + m0w + 4 * q;
    w4[i] = __ldcs(reinterpret_cast<const float4*>(u.W + o[i]));
    v4[i] = __ldcs(reinterpret_cast<const float4*>(u.V + o[i]));
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float* g = v + 4 * i;
    float* pw = reinterpret_cast<float*>(&w4[i]);
    float* pv = reinterpret_cast<float*>(&v4[i]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      pv[e] = __fmaf_rn(u.c.c_gamma, pv[e], __fmul_rn(u.c.c_one, g[e]));
      pw[e] = __fmaf_rn(-u.c.c_eta, pv[e], pw[e]);
    }
    __stcs(reinterpret_cast<float4*>(u.W + o[i]), w4[i]);
    __stcs(reinterpret_cast<float4*>(u.V + o[i]), v4[i]);
    if (u.WF) {
      float4 f;
      f.x = __fmaf_rn(-u.c.c_f, pv[0], pw[0]);
      f.y = __fmaf_rn(-u.c.c_f, pv[1], pw[1]);
      f.z = __fmaf_rn(-u.c.c_f, pv[2], pw[2]);
      f.w = __fmaf_rn(-u.c.c_f, pv[3], pw[3]);
      *reinterpret_cast<float4*>(u.WF + o[i]) = f;
    }
    if (u.WB) {
      float4 f;
      f.x = __fmaf_rn(-u.c.c_b, pv[0], pw[0]);
      f.y = __fmaf_rn(-u.c.c_b, pv[1], pw[1]);
      f.z = __fmaf_rn(-u.c.c_b, pv[2], pw[2]);
      f.w = __fmaf_rn(-u.c.c_b, pv[3], pw[3]);
      *reinterpret_cast<float4*>(u.WB + o[i]) = f;
    }
  }
}

// ============================================================================
// FP32X3 / TF32 dW kernel (persistent): G = Xᵀ·dZ as Gᵀ tiles (M = out, N = in, K = B).
//
// K = batch is short (≤ 128 here), the output (one fp32 per parameter) dominates.
// Each CTA walks a contiguous range of 128 × 128 output tiles in m-major order.
// The A operand (dZᵀ rows of the current m-tile, all of K) is staged once per m-tile
// (TMA → smem), split by converter warps into hi / lo and kept RESIDENT IN TMEM
// (A-from-TMEM MMA); B (X columns, hi + lo precomputed) streams through a 2-stage smem
// ring. TMEM: accumulators [0, 256) (two buffers), A hi [256, 384), A lo [384, 512).
// Epilogue: 16 warps in two groups, group g drains accumulator g (tiles local ≡ g mod 2).
// With kUPD it applies the K-B update in place of storing G. The update is an HBM
// stream (W, V read and written once): two loader warps keep W / V chunks
// (128 rows × 16 columns, 16 KB) in flight by TMA into a 3-slot ring per group — 96 KB
// continuously in flight per SM, independent of registers — and the epilogue reads them
// from smem, applies Eq. 1 / apply / Eq. 4 with g from TMEM and stores from registers
// (warp-coalesced, write-through). Register-staged loads (one 4 KB batch per warp in
// flight) reached only ~4.7 TB/s on the same stream.
// ============================================================================
constexpr int DW_KMAX = 128;                       // K (= batch) capacity of the resident A
#ifndef ST_DW_RB
#define ST_DW_RB 3
#endif
constexpr int DW_RB = ST_DW_RB;                    // B ring stages (hi + lo, 32 KB)
constexpr int DW_EPI_WARPS = 16;                   // 2 groups × 2 warps per TMEM lane quadrant
constexpr int DW_CONV_WARPS = 4;
constexpr int DW_LOAD_WARPS = 2;                   // W / V stream loaders, one per group
constexpr int DW_THREADS = 64 + 32 * (DW_EPI_WARPS + DW_CONV_WARPS + DW_LOAD_WARPS);
constexpr int DW_A_BYTES = (DW_KMAX / BK) * TILE_BYTES;  // raw A staging: 64 KB
constexpr int DW_B_STAGE = 2 * TILE_BYTES;
constexpr int DW_WV_COLS = 16;                     // columns (n) per W / V chunk
#ifndef ST_DW_WV_SLOTS
#define ST_DW_WV_SLOTS 4
#endif
constexpr int DW_WV_SLOTS = ST_DW_WV_SLOTS;        // ring slots per group
constexpr int DW_WV_HALF = DW_WV_COLS * BM * 4;    // 8 KB: one tensor's chunk [16][128]
constexpr int DW_WV_SLOT = 2 * DW_WV_HALF;         // W + V
constexpr int DW_WV_BYTES = 2 * DW_WV_SLOTS * DW_WV_SLOT;  // 96 KB
// The A staging (needed once per m-tile, i.e. once or twice per CTA) ALIASES the B ring:
// the producer drains the ring before loading A and resumes B only after the converter
// has read A. The 64 KB this frees deepen the B ring (X hi + lo, 128 KB per tile from
// L2: with 2 stages the MMAs starved on the L2 round trip and the epilogue waited on
// the accumulator).
static_assert(DW_RB * DW_B_STAGE >= DW_A_BYTES, "A staging aliases the B ring");
constexpr int dw_smem_bytes() { return DW_RB * DW_B_STAGE + DW_WV_BYTES + 1024 + 512; }

template <bool kX3, bool kUPD>
__global__ void __launch_bounds__(DW_THREADS, 1)
    tc_dw_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                 const __grid_constant__ CUtensorMap mapBlo, const __grid_constant__ CUtensorMap mapW,
                 const __grid_constant__ CUtensorMap mapV, TcParams p, int m_tiles, int n_tiles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  char* smem = align_smem_1k(smem_raw);
  char* Astage = smem;
  char* ringB = smem;  // aliased with the A staging (see dw_smem_bytes)
  char* ringWV = smem + DW_RB * DW_B_STAGE;  // [group][slot] W chunk, V chunk
  uint64_t* bars = reinterpret_cast<uint64_t*>(ringWV + DW_WV_BYTES);
  const uint32_t a_full = smem_u32(bars);          // A staging landed (TMA)
  const uint32_t a_sfree = a_full + 8;             // converter done reading the staging (4 warps)
  const uint32_t a_tfull = a_sfree + 8;            // A hi / lo written to TMEM (4 warps)
  const uint32_t a_tempty = a_tfull + 8;           // MMAs on the old A done (commit)
  const uint32_t b_full = a_tempty + 8;            // [RB]
  const uint32_t b_empty = b_full + 8 * DW_RB;     // [RB]
  const uint32_t c_full = b_empty + 8 * DW_RB;     // [2] accumulator ready
  const uint32_t c_empty = c_full + 16;            // [2] epilogue group drained it (8 warps)
  const uint32_t wv_full = c_empty + 16;           // [2][SLOTS] W / V chunk landed (TMA)
  const uint32_t wv_empty = wv_full + 8 * 2 * DW_WV_SLOTS;  // [2][SLOTS] consumed (the group's 8 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4 + 2 * DW_RB + 4 + 4 * DW_WV_SLOTS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tiles = m_tiles * n_tiles;
  int t_begin = (int)((long long)blockIdx.x * tiles / gridDim.x);
  int t_end = (int)((long long)(blockIdx.x + 1) * tiles / gridDim.x);
  if (p.lockstep) {
    const int parts = gridDim.x / m_tiles, m_t = blockIdx.x % m_tiles, part = blockIdx.x / m_tiles;
    t_begin = m_t * n_tiles + part * n_tiles / parts;
    t_end = m_t * n_tiles + (part + 1) * n_tiles / parts;
  }
  const int nkb = p.kb_total;  // K blocks (K ≤ 128)
  const int bn = p.bn;
  const int conv_w0 = 2 + DW_EPI_WARPS;
  const int load_w0 = conv_w0 + DW_CONV_WARPS;
  const int nch = (bn + DW_WV_COLS - 1) / DW_WV_COLS;  // W / V chunks per tile

  if (threadIdx.x == 0) {
    mbar_init(a_full, 1);
    mbar_init(a_sfree, DW_CONV_WARPS);
    mbar_init(a_tfull, DW_CONV_WARPS);
    mbar_init(a_tempty, 1);
    for (int s = 0; s < DW_RB; ++s) {
      mbar_init(b_full + 8 * s, 1);
      mbar_init(b_empty + 8 * s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(c_full + 8 * s, 1);
      mbar_init(c_empty + 8 * s, DW_EPI_WARPS / 2);
    }
    for (int s = 0; s < 2 * DW_WV_SLOTS; ++s) {
      mbar_init(wv_full + 8 * s, 1);
      mbar_init(wv_empty + 8 * s, DW_EPI_WARPS / 4);  // the chunk's 4 warps wrote w', v' back
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tA_hi = tmem + 256, tA_lo = tmem + 384;
  // programmatic dependent launch (no-ops without the attribute): the successor may launch;
  // dZ / X / X-lo are read only after the predecessor completed (warp 0), while the W / V
  // stream — written by no earlier kernel still in flight — may start at once
  if (threadIdx.x == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0) {
    // ---------------- TMA producer: A staging per m-tile, B ring per tile × K-block
    // (warp-converged loop, elected lane issues)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    {
      int cur_m = -1, a_loads = 0, it = 0;
      for (int t = t_begin; t < t_end; ++t) {
        const int m_t = t / n_tiles, n_t = t % n_tiles;
        if (m_t != cur_m) {
          // drain the B ring (the staging aliases it): the MMAs of every issued B stage are done
          for (int j = max(0, it - DW_RB); j < it; ++j) mbar_wait(b_empty + 8 * (j % DW_RB), (j / DW_RB) & 1);
          if (elect_one()) {
            mbar_expect_tx(a_full, (uint32_t)(nkb * TILE_BYTES));
            for (int kb = 0; kb < nkb; ++kb) {
              const uint32_t dA = smem_u32(Astage + kb * TILE_BYTES);
#pragma unroll
              for (int c = 0; c < BM / 32; ++c) tma_load_2d(dA + c * 4096, &mapA, m_t * BM + 32 * c, kb * BK, a_full);
            }
          }
          __syncwarp();
          // B may overwrite the staging only once the converter has read it
          mbar_wait(a_sfree, a_loads & 1);
          cur_m = m_t;
          ++a_loads;
        }
        const int nbox = (bn + 31) / 32;
        const uint32_t bytes = (uint32_t)((kX3 ? 2 : 1) * nbox * 4096);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % DW_RB;
          mbar_wait(b_empty + 8 * s, ((it / DW_RB) & 1) ^ 1);
          const uint32_t full = b_full + 8 * s;
          const uint32_t dB = smem_u32(ringB + s * DW_B_STAGE);
          if (elect_one()) {
            if (p.dev_flags & 4) {  // development: skip the B loads
              mbar_arrive(full);
            } else {
              mbar_expect_tx(full, bytes);
              for (int c = 0; c < nbox; ++c) {
                tma_load_2d(dB + c * 4096, &mapB, n_t * BNMAX + 32 * c, kb * BK, full);
                if (kX3) tma_load_2d(dB + TILE_BYTES + c * 4096, &mapBlo, n_t * BNMAX + 32 * c, kb * BK, full);
              }
            }
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: A (dZᵀ hi / lo) from TMEM, B (X hi / lo) from smem.
    // The whole warp walks the loop (operands stay warp-uniform), one elected lane issues.
    {
      int cur_m = -1, a_loads = 0, it = 0, local = 0;
      for (int t = t_begin; t < t_end; ++t, ++local) {
        const int m_t = t / n_tiles;
        if (m_t != cur_m) {
          if (a_loads > 0) {
            if (elect_one()) tc_commit(a_tempty);  // every MMA on the old A has been issued
            __syncwarp();
          }
          mbar_wait(a_tfull, a_loads & 1);
          cur_m = m_t;
          ++a_loads;
        }
        const int buf = local & 1;
        mbar_wait(c_empty + 8 * buf, ((local >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t acc_t = tmem + buf * BNMAX;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % DW_RB;
          mbar_wait(b_full + 8 * s, (it / DW_RB) & 1);
          tc_fence_after();
          const uint32_t b_hi = smem_u32(ringB + s * DW_B_STAGE), b_lo = b_hi + TILE_BYTES;
          const uint32_t acc0 = kb > 0 ? 1u : 0u;
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              if (p.dev_flags & 1) break;
              const uint32_t ka = kb * BK + kk * 8;
              tc_mma_ts(acc_t, tA_hi + ka, desc_mnmajor(b_hi + kk * 1024), p.idesc, kk > 0 ? 1u : acc0);
              if (kX3) {
                tc_mma_ts(acc_t, tA_lo + ka, desc_mnmajor(b_hi + kk * 1024), p.idesc, 1u);
                if (!(p.dev_flags & 256)) tc_mma_ts(acc_t, tA_hi + ka, desc_mnmajor(b_lo + kk * 1024), p.idesc, 1u);
              }
            }
            tc_commit(b_empty + 8 * s);
          }
          __syncwarp();
        }
        if (elect_one()) tc_commit(c_full + 8 * buf);
        __syncwarp();
      }
    }
  } else if (warp >= load_w0) {
    // ---------------- W / V stream of group (warp − load_w0), one thread: TMA loads into
    // the ring and TMA stores of the updated chunks out of it. Chunk q lives in slot
    // q % SLOTS; once the group's 8 warps have written w', v' back into it (wv_empty[q],
    // 8 arrivals) the chunk is stored, and once that store has read the slot, chunk
    // q + SLOTS is loaded into it. The epilogue warps never wait for one another.
    if (kUPD && p.wv_stream) {
      const int group = warp - load_w0;
      const bool leader = elect_one();
      const uint32_t full0 = wv_full + 8 * DW_WV_SLOTS * group, done0 = wv_empty + 8 * DW_WV_SLOTS * group;
      char* ring = ringWV + group * DW_WV_SLOTS * DW_WV_SLOT;
      const int my_tiles = (t_end - (t_begin + group) + 1) / 2;
      const int nq = my_tiles > 0 ? my_tiles * nch : 0;
      auto coords = [&](int q, int& cm, int& cn) {
        const int t = t_begin + group + 2 * (q / nch), c = q % nch;
        cm = (t / n_tiles) * BM;
        cn = (t % n_tiles) * BNMAX + c * DW_WV_COLS;
      };
      auto load = [&](int q) {
        const int sl = q % DW_WV_SLOTS;
        int cm, cn;
        coords(q, cm, cn);
        const uint32_t dst = smem_u32(ring + sl * DW_WV_SLOT);
        if (leader) {
          if (p.dev_flags & 64) {  // development: skip the W / V loads
            mbar_arrive(full0 + 8 * sl);
          } else {
            mbar_expect_tx(full0 + 8 * sl, DW_WV_SLOT);
            tma_load_2d(dst, &mapW, cm, cn, full0 + 8 * sl);
            tma_load_2d(dst + DW_WV_HALF, &mapV, cm, cn, full0 + 8 * sl);
          }
        }
        __syncwarp();
      };
      for (int q = 0; q < min(nq, DW_WV_SLOTS); ++q) load(q);
      if (p.wv_direct) {
        // the epilogue stores w', v' itself: refill a slot as soon as its 4 warps have read it
        for (int q = 0; q + DW_WV_SLOTS < nq; ++q) {
          mbar_wait(done0 + 8 * (q % DW_WV_SLOTS), (q / DW_WV_SLOTS) & 1);
          load(q + DW_WV_SLOTS);
        }
      } else
      for (int q = 0; q < nq; ++q) {
        const int sl = q % DW_WV_SLOTS;
        mbar_wait(done0 + 8 * sl, (q / DW_WV_SLOTS) & 1);  // w', v' of chunk q are in the slot
        int cm, cn;
        coords(q, cm, cn);
        const uint32_t src = smem_u32(ring + sl * DW_WV_SLOT);
        if (leader) {
          tma_store_2d(&mapW, src, cm, cn);
          tma_store_2d(&mapV, src + DW_WV_HALF, cm, cn);
          bulk_commit();
          // refill the slot as soon as its store has read it (the global writes stay in flight)
          bulk_wait_read<0>();
        }
        __syncwarp();
        if (q + DW_WV_SLOTS < nq) load(q + DW_WV_SLOTS);
      }
      if (leader) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // updates in memory before exit
      __syncwarp();
    }
  } else if (warp >= conv_w0) {
    // ---------------- converter: staged dZᵀ (MN-major boxes) → TMEM hi / lo, once per m-tile
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // tile row (out index) = TMEM lane
    int cur_m = -1, a_loads = 0;
    for (int t = t_begin; t < t_end; ++t) {
      const int m_t = t / n_tiles;
      if (m_t == cur_m) continue;
      cur_m = m_t;
      mbar_wait(a_full, a_loads & 1);
      mbar_wait(a_tempty, (a_loads & 1) ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < nkb; ++kb) {
        const char* box = Astage + kb * TILE_BYTES + (r >> 5) * 4096;
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float x = *reinterpret_cast<const float*>(box + k * 128 + ((((r & 31) >> 3) ^ (k & 3)) << 5) +
                                                          (r & 7) * 4);
          hi[k] = __float_as_uint(x);
          lo[k] = __float_as_uint(lo_part(x));
        }
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        tc_st32(tA_hi + lane_off + kb * BK, hi);
        if (kX3) tc_st32(tA_lo + lane_off + kb * BK, lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(a_sfree);
        mbar_arrive(a_tfull);
      }
      ++a_loads;
    }
  } else {
    // ---------------- epilogue (warps 2..17): accumulator → G[n·M + m], or (kUPD) the
    // K-B update of W / V / WF / WB at the same index; g never leaves the chip.
    const int quad = warp & 3;
    const int group = (warp - 2) >> 3;       // accumulator / tile parity
    const int half = ((warp - 2) >> 2) & 1;  // which 64 columns of the tile (G store) / 8 of each chunk's 16 (stream)
    int local = group;
    if (kUPD && p.wv_stream) {
      // W / V from the smem ring: chunk c of a tile is consumed by the 4 warps (one per
      // TMEM lane quadrant) of parity c & 1, so two chunks are in flight per group; this
      // warp takes rows quad·32 + lane, all 16 columns. w', v' are written back INTO the
      // slot and leave by TMA store (issued by the group's stream thread once the 4 warps
      // have arrived on wv_empty): no per-warp global stores for W / V. WF / WB (only when
      // s > 0) are stored from registers.
      const uint32_t full0 = wv_full + 8 * DW_WV_SLOTS * group, empty0 = wv_empty + 8 * DW_WV_SLOTS * group;
      char* ring = ringWV + group * DW_WV_SLOTS * DW_WV_SLOT;
      const UpdateArgs& u = p.upd;
      int q = 0;
      for (int t = t_begin + group; t < t_end; t += 2, local += 2) {
        const int m_t = t / n_tiles, n_t = t % n_tiles;
        mbar_wait(c_full + 8 * group, (local >> 1) & 1);
        tc_fence_after();
        const int m = m_t * BM + quad * 32 + lane;
        const uint32_t trow = tmem + group * BNMAX + ((uint32_t)(quad * 32) << 16);
        const int n0 = n_t * BNMAX;
        for (int c = 0; c < nch; ++c, ++q) {
          if ((c & 1) != half) continue;
          const int sl = q % DW_WV_SLOTS;
          const int c0 = c * DW_WV_COLS;  // first tile column of the chunk
          uint32_t rr[16];
          tc_ld16_nowait(trow + c0, rr);
          mbar_wait(full0 + 8 * sl, (q / DW_WV_SLOTS) & 1);
          float* sw = reinterpret_cast<float*>(ring + sl * DW_WV_SLOT) + quad * 32 + lane;
          float* sv = sw + DW_WV_HALF / 4;
          float w[16], v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            w[j] = sw[j * BM];
            v[j] = sv[j * BM];
          }
          tc_wait_ld();
          const int nc = n0 + c0;
          if (p.wv_direct) {
            // the slot is free once all lanes have read it; w', v' go out from registers
            // (per j: 32 consecutive m = one 128-byte line per warp, write-through)
            __syncwarp();
            if (lane == 0) mbar_arrive(empty0 + 8 * sl);
            if (m < p.M) {
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                if (nc + j >= p.N) break;
                const float g = __uint_as_float(rr[j]);
                const float vn = __fmaf_rn(u.c.c_gamma, v[j], __fmul_rn(u.c.c_one, g));
                const float wn = __fmaf_rn(-u.c.c_eta, vn, w[j]);
                const size_t o = (size_t)(nc + j) * p.M + m;
                __stcs(u.W + o, wn);
                __stcs(u.V + o, vn);
                if (u.WF) __stcs(u.WF + o, __fmaf_rn(-u.c.c_f, vn, wn));
                if (u.WB) __stcs(u.WB + o, __fmaf_rn(-u.c.c_b, vn, wn));
              }
            }
            continue;
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float g = __uint_as_float(rr[j]);
            const float vn = __fmaf_rn(u.c.c_gamma, v[j], __fmul_rn(u.c.c_one, g));
            const float wn = __fmaf_rn(-u.c.c_eta, vn, w[j]);
            sw[j * BM] = wn;  // out-of-range rows / columns are clipped by the TMA store
            sv[j * BM] = vn;
            if ((u.WF || u.WB) && m < p.M && nc + j < p.N) {
              const size_t o = (size_t)(nc + j) * p.M + m;
              if (u.WF) __stcs(u.WF + o, __fmaf_rn(-u.c.c_f, vn, wn));
              if (u.WB) __stcs(u.WB + o, __fmaf_rn(-u.c.c_b, vn, wn));
            }
          }
          fence_proxy_async();  // the generic-proxy writes above are read by the TMA store
          __syncwarp();
          if (lane == 0) mbar_arrive(empty0 + 8 * sl);  // this warp's part of chunk q is written back
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(c_empty + 8 * group);
      }
    } else
    for (int t = t_begin + group; t < t_end; t += 2, local += 2) {
      const int m_t = t / n_tiles, n_t = t % n_tiles;
      const int buf = group;
      mbar_wait(c_full + 8 * buf, (local >> 1) & 1);
      tc_fence_after();
      const int m = m_t * BM + quad * 32 + lane;
      const uint32_t trow = tmem + buf * BNMAX + ((uint32_t)(quad * 32) << 16);
      const int n0 = n_t * BNMAX;
      const int cbeg = half * (BNMAX / 2);
      const int cend = min(bn, cbeg + BNMAX / 2);
      const bool full_tile = (n0 + cend <= p.N) && (m_t * BM + BM <= p.M);
      for (int c = cbeg; c < cend; c += 16) {
        if (p.dev_flags & 16) break;
        uint32_t rr[16];
        tc_ld16_nowait(trow + c, rr);
        tc_wait_ld();
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(rr[j]);
        const size_t o0 = (size_t)(n0 + c) * p.M + m;  // element (n0 + c + j, m) at o0 + j·M
        if (kUPD) {
          const UpdateArgs& u = p.upd;
          if (full_tile) {
            update_block16_vec(u, (size_t)p.M, m_t * BM + quad * 32, n0 + c, lane, v);
          } else if (m < p.M) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (n0 + c + j < p.N) update_cols<1>(u, o0 + (size_t)j * p.M, 0, v + j);
          }
        } else if (m < p.M) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (n0 + c + j < p.N) __stcs(p.out + o0 + (size_t)j * p.M, v[j]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(c_empty + 8 * buf);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
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

// 2D fp32 tensor [outer][inner] (row pitch = inner), box {box_inner, box_outer}, no swizzle
// (plain row-major staging for the W / V stream of the fused update).
bool make_plain_map(CUtensorMap* m, const float* base, int inner, int outer, int box_inner, int box_outer) {
  EncodeFn enc = get_encode();
  if (!enc || ((uintptr_t)base & 15u)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)inner * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Upper bound on the CTAs of one persistent / split-K launch: workspace_bytes sizes the
// partial-tile buffers for it, independent of the device it is queried on.
constexpr int kWsSms = 160;

// SM count of the current device (cached per device ordinal: contexts may live on
// different GPUs of one process)
int num_sms() {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  int sms = cache[dev].load(std::memory_order_relaxed);
  if (sms <= 0) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
    sms = std::min(sms, kWsSms);  // the split-K workspaces are sized for at most kWsSms CTAs
    cache[dev].store(sms, std::memory_order_relaxed);
  }
  return sms;
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device setting: opt each kernel in
// once per (device, kernel, size), thread-safe (stage threads launch concurrently).
st_status ensure_max_smem(const void* fn, int bytes) {
  static std::mutex mu;
  static std::set<std::tuple<int, const void*, int>> done;
  int dev = 0;
  ST_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (done.count(std::make_tuple(dev, fn, bytes))) return ST_OK;
  ST_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.insert(std::make_tuple(dev, fn, bytes));
  return ST_OK;
}

uint32_t make_idesc(int bn, bool a_mn, bool b_mn, int mma_m = BM) {
  uint32_t d = 0;
  d |= 1u << 4;                       // D format F32
  d |= 2u << 7;                       // A format TF32
  d |= 2u << 10;                      // B format TF32
  d |= (a_mn ? 1u : 0u) << 15;        // A major (0 = K, 1 = MN)
  d |= (b_mn ? 1u : 0u) << 16;        // B major
  d |= (uint32_t)(bn >> 3) << 17;     // N >> 3
  d |= (uint32_t)(mma_m >> 4) << 24;  // M >> 4
  return d;
}

// MMA N of a tile: the tile's columns rounded up to a multiple of 16 (≤ 128); the
// B box of K-major operands has exactly bn rows (OOB rows are zero-filled by TMA).
int bn_for(int N) { return std::max(16, (std::min(N, BNMAX) + 15) / 16 * 16); }

int dev_flags() {
  static int f = -1;
  if (f < 0) {
    f = dev_knob("ST_GEMM_DEV_FLAGS", 0);
  }
  return f;
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

static thread_local int g_launches = 0;
constexpr size_t kCounterBytes = 64 * 1024;
constexpr int kExtReduceSplits = 2;  // from this many K splits on, reduce in a separate parallel kernel (ST_EXT_REDUCE overrides)

int ext_reduce_splits() {
  static int f = -1;
  if (f < 0) {
    f = dev_knob("ST_EXT_REDUCE", kExtReduceSplits);
  }
  return f;
}


// Fused dW + update with m-tile-aligned CTA ranges (TcParams::lockstep): standalone on the
// whole GPU (8192²: 128 CTAs) 222 → 206 µs; in the overlapped backward (80-SM budget) only
// 64 CTAs fit whole m-tile columns and it is slower. Default (2): on when the launch has
// the whole GPU; ST_DW_LOCKSTEP=1 always, 0 never.
int dw_lockstep_mode() {
  static int f = -1;
  if (f < 0) {
    f = dev_knob("ST_DW_LOCKSTEP", 2);
  }
  return f;
}

// TMEM-A kernel, dW launches: K-blocks per accumulator segment (0 = one accumulator per work
// unit). Measured on VGG-16 (10 mini-batches, fp64 oracle): V spread 0.054 → 0.0007 at 1
// stage (the CUDA-core fp32 GEMMs: 0.00014), 0.093 → 0.035 at 8 stages (fp32: 0.039).
// ST_TSG_SEG overrides (development).
int tsg_segment_kblocks() {
  static int f = -1;
  if (f < 0) f = std::max(0, dev_knob("ST_TSG_SEG", 0));
  return f;
}

// The fused update stores w', v' from registers and frees each W / V slot as soon as
// the epilogue has read it (default): standalone 8192² 202.9 → 191.8 µs (5.29 → 5.60
// TB/s), 16384² 710 → 689 µs (6.05 → 6.24 TB/s) against TMA stores out of the slot,
// whose refill had to wait for the store to read the slot. ST_DW_DIRECT=0: TMA stores.
int dw_direct_mode() {
  static int f = -1;
  if (f < 0) f = dev_knob("ST_DW_DIRECT", 1) != 0 ? 1 : 0;
  return f;
}

// ST_TSG_NARROW=0: N ≤ 64 TMEM-A launches on the 4-stage ring (A/B timing)
bool tsg_narrow_on() {
  static int f = -1;
  if (f < 0) {
    f = dev_knob("ST_TSG_NARROW", 1) != 0 ? 1 : 0;
  }
  return f != 0;
}

// ST_CONV_TS=0: FP32X3 implicit-conv fwd / dX without the TMEM-A kernel (A/B timing)
bool conv_ts_on() {
  static int f = -1;
  if (f < 0) {
    f = dev_knob("ST_CONV_TS", 1) != 0 ? 1 : 0;
  }
  return f != 0;
}

// ST_CONV_PERSISTENT=0: implicit-conv fwd / dX on the one-tile-per-CTA kernel (A/B timing)
bool conv_persistent_off() {
  static int f = -1;
  if (f < 0) {
    f = dev_knob("ST_CONV_PERSISTENT", 1) == 0 ? 1 : 0;
  }
  return f != 0;
}

template <int EPI, bool A_MN, bool B_MN, int CV = CV_NONE>
st_status launch(const GemmArgs& g, int M, int N, int K, const CUtensorMap& ma, const CUtensorMap& mb, float* out,
                 const float* aux, int relu, int cvH = 0, int cvW = 0, int cvC = 0, bool tall_fwd = false) {
  TcParams p{};
  p.dev_flags = dev_flags();
  p.row = (CV == CV_FWD || CV == CV_DX || CV == CV_ROWS || CV == CV_DWT) ? 1 : 0;
  p.cv_H = cvH;
  p.cv_W = cvW;
  p.cv_C = cvC;
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
  const size_t ws_cap = (size_t)2 * kWsSms * BNMAX * BM * 4;
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
  auto kern = (g.mode == ST_GEMM_FP32X3) ? tc_gemm_kernel<EPI, A_MN, B_MN, true, S, CV>
                                         : tc_gemm_kernel<EPI, A_MN, B_MN, false, S, CV>;
  const int ai = g.mode == ST_GEMM_FP32X3 ? 1 : 0;
  (void)ai;
  ST_TRY(ensure_max_smem((const void*)kern, smem_bytes(S)));
  p.ext_reduce = p.splits >= ext_reduce_splits();
  if (g.mode == ST_GEMM_FP32X3 && conv_ts_on() && (CV != CV_NONE || EPI == EPI_DW || tall_fwd)) {
    // persistent TMEM-A kernel: implicit conv (all passes), the tall dense dW and the tall
    // dense forward (many row tiles: the epilogue of one tile overlaps the next one's MMAs)
    const bool narrow = p.bn <= 64 && tsg_narrow_on();
    auto ck = narrow ? tc_tsg_kernel<EPI, A_MN, B_MN, CV, true> : tc_tsg_kernel<EPI, A_MN, B_MN, CV, false>;
    const int smem = narrow ? tsg_smem_bytes<true>() : tsg_smem_bytes<false>();
    ST_TRY(ensure_max_smem((const void*)ck, smem));
    p.idesc = make_idesc(p.bn, false, B_MN);
    p.ext_reduce = p.splits > 1;
    // dW: K = pixels / T·B rows, long accumulation chains (measured error 2.9e-5 → 9.7e-6
    // rel-L2 on an 8192-row dW, LSTM step unchanged); fwd / dX keep the double-buffered
    // accumulators that overlap the epilogue (ST_GEMM_DEV_FLAGS=1024 forces it everywhere)
    p.split_acc = (EPI == EPI_DW || (p.dev_flags & 1024)) ? 1 : 0;
    p.seg = tsg_segment_kblocks();
    const int budget = g.max_ctas > 0 ? std::min(g.max_ctas, num_sms()) : num_sms();
    ST_TRY(launch_maybe_pdl(g.pdl, ck, dim3(std::min(tiles * p.splits, budget)), dim3(kPThreads), (size_t)smem,
                            g.stream, ma, mb, p, mt, tiles));
    g_launches = 1;
    if (p.ext_reduce) {
      ST_TRY(launch_splitk_epilogue<EPI>(p, tiles, mt, g.stream, g.pdl));
      g_launches = 2;
    }
    return ST_OK;
  }
  if ((CV == CV_FWD || CV == CV_DX || CV == CV_ROWS) && p.splits == 1 && !conv_persistent_off()) {
    auto pk = (g.mode == ST_GEMM_FP32X3) ? tc_gemm_persistent_kernel<EPI, A_MN, B_MN, true, S, CV>
                                         : tc_gemm_persistent_kernel<EPI, A_MN, B_MN, false, S, CV>;
    ST_TRY(ensure_max_smem((const void*)pk, smem_bytes(S)));
    const int budget = g.max_ctas > 0 ? std::min(g.max_ctas, num_sms()) : num_sms();
    pk<<<std::min(tiles, budget), kPThreads, smem_bytes(S), g.stream>>>(ma, mb, p, mt, tiles);
    ST_CUDA_TRY(cudaGetLastError());
    g_launches = 1;
    return ST_OK;
  }
  kern<<<grid, kThreads, smem_bytes(S), g.stream>>>(ma, mb, p);
  ST_CUDA_TRY(cudaGetLastError());
  g_launches = 1;
  if (p.ext_reduce) {
    ST_TRY(launch_splitk_epilogue<EPI>(p, mt * nt, mt, g.stream));
    g_launches = 2;
  }
  return ST_OK;
}

bool tma_ok(const void* p, int pitch) { return aligned16(p) && (pitch % 4) == 0; }

// split-K plan shared by both kernels
void plan_splits(TcParams& p, int M, int N, int K, int budget) {
  p.M = M;
  p.N = N;
  p.K = K;
  p.kb_total = (K + BK - 1) / BK;
  const int mt = (M + BM - 1) / BM, nt = (N + BNMAX - 1) / BNMAX;
  const int tiles = mt * nt;
  int splits = 1;
  if (tiles < budget) splits = std::min(budget / tiles, p.kb_total);
  if (const int f = dev_knob("ST_FORCE_SPLITS", 0)) splits = std::min(f, p.kb_total);  // development: accuracy vs K
  if (splits < 1) splits = 1;
  const size_t part_bytes = (size_t)BNMAX * BM * 4;
  const size_t ws_cap = (size_t)2 * kWsSms * BNMAX * BM * 4;
  while (splits > 1 && ((size_t)splits * tiles * part_bytes > ws_cap || tiles > (int)(kCounterBytes / 4))) --splits;
  p.kb_per_split = (p.kb_total + splits - 1) / splits;
  p.splits = (p.kb_total + p.kb_per_split - 1) / p.kb_per_split;
  p.bn = bn_for(N);
}

// CTA-pair kernel for fwd / dX (default; ST_GEMM_PAIR=0 selects the single-CTA kernel).
// With the MMA issue loop warp-converged (operands in uniform registers) the pair's
// faster MMA rate shows: 8192² fwd 101 → 87 µs, dX 104 → 88 µs; wide-FCN step 3.05 → 2.88 ms.
// Stream-K is opt-in (ST_STREAM_K=1): measured on the 8192² fwd / dX it is no faster
// than the K-split grid (102 vs 105 µs standalone, 3.14 vs 3.18 ms per wide-FCN step) —
// the GEMM is bound chip-wide, not by the 20 SMs the split leaves idle — and it loses
// badly when a tile is cut into many segments (784-wide dX: 25 → 80 µs).
bool stream_k_off() {
  static int f = -1;
  if (f < 0) {
    f = dev_knob("ST_STREAM_K", 0) == 1 ? 0 : 1;
  }
  return f != 0;
}

// The CTA-pair fwd / dX kernel keeps the small 3xTF32 terms in a second accumulator (D24):
// 8192² fwd rel-L2 1.7e-5 → 5.7e-6, dX 3.0e-5 → 9.9e-6 against fp64; wide-FCN step
// unchanged (45.0–45.4k vs 45.1–45.3k samples/s). ST_TS_SPLIT_ACC=0 restores one accumulator.
int ts_split_acc() {
  static int f = -1;
  if (f < 0) {
    f = dev_knob("ST_TS_SPLIT_ACC", 1) != 0 ? 1 : 0;
  }
  return f;
}

bool use_pair() {
  static int f = -1;
  if (f < 0) {
    f = dev_knob("ST_GEMM_PAIR", 1);
  }
  return f != 0;
}

// FP32X3 fwd / dX through the TMEM-A kernels. Bact: the activation operand [N rows × K]
// (row pitch K); its lo part goes to the workspace tail.
template <int EPI, bool A_MN>
st_status launch_ts(const GemmArgs& g, int M, int N, int K, const CUtensorMap& ma, const float* Bact, float* out,
                    const float* aux, int relu) {
  TcParams p{};
  const bool pair = use_pair();
  const int budget = g.max_ctas > 0 ? std::min(g.max_ctas, num_sms()) : num_sms();
  // pair: the m-tile count is padded to even (the padding CTA's rows are masked)
  const int mt = (M + BM - 1) / BM, mt_grid = pair ? (mt + 1) / 2 * 2 : mt;
  plan_splits(p, mt_grid * BM, N, K, pair ? budget / 2 * 2 : budget);
  const int nt = (N + BNMAX - 1) / BNMAX;
  p.mt = mt_grid;
  p.tiles = mt_grid * nt;
  // stream-K when the tiles alone cannot fill the CTA budget: every CTA gets the same
  // number of K-blocks (a K split leaves budget − tiles·splits SMs idle)
  p.sk = (!pair && p.tiles < budget && !stream_k_off()) ? 1 : 0;
  p.M = M;
  p.out = out;
  p.aux = aux;
  p.relu = relu;
  p.counters = reinterpret_cast<int*>(g.work);
  p.ws = reinterpret_cast<float*>(static_cast<char*>(g.work) + kCounterBytes);
  p.idesc = make_idesc(p.bn, false, false, pair ? 2 * BM : BM);
  p.dev_flags = dev_flags();
  p.ext_reduce = p.splits >= ext_reduce_splits();
  float* blo = reinterpret_cast<float*>(static_cast<char*>(g.work) + kCounterBytes +
                                        (size_t)2 * kWsSms * BNMAX * BM * 4);
  int launches = 1;
  if (g.act_lo) {
    blo = const_cast<float*>(g.act_lo);  // the producer already split the operand
  } else {
    const size_t n4 = (size_t)N * K / 4;
    ST_TRY(launch_maybe_pdl(g.pdl, split_lo_kernel, dim3((unsigned)std::min<size_t>(4 * (size_t)num_sms(), (n4 + 255) / 256)),
                            dim3(256), 0, g.stream, reinterpret_cast<const float4*>(Bact),
                            reinterpret_cast<float4*>(blo), n4));
    ++launches;
  }
  const int brows = pair ? p.bn / 2 : p.bn;
  CUtensorMap mb, mblo;
  if (!make_map(&mb, Bact, K, N, K, brows, false) || !make_map(&mblo, blo, K, N, K, brows, false))
    return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (activation operand)");
  dim3 grid(mt_grid, nt, p.splits);
  if (p.sk) {
    const long long U = (long long)p.tiles * p.kb_total;
    grid = dim3((unsigned)std::min<long long>(budget, U), 1, 1);
    p.splits = 1;
    p.ext_reduce = 0;
  }
  if (pair) {
    auto kern = ts_split_acc() ? tc_ts2_kernel<EPI, A_MN, true> : tc_ts2_kernel<EPI, A_MN, false>;
    ST_TRY(ensure_max_smem((const void*)kern, ts2_smem_bytes()));
    if (g.pdl) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = grid;
      cfg.blockDim = dim3(TS_THREADS);
      cfg.dynamicSmemBytes = ts2_smem_bytes();
      cfg.stream = g.stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      ST_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ma, mb, mblo, p));
    } else {
      kern<<<grid, TS_THREADS, ts2_smem_bytes(), g.stream>>>(ma, mb, mblo, p);
    }
  } else {
    auto kern = tc_ts_kernel<EPI, A_MN>;
    ST_TRY(ensure_max_smem((const void*)kern, ts_smem_bytes()));
    kern<<<grid, TS_THREADS, ts_smem_bytes(), g.stream>>>(ma, mb, mblo, p);
  }
  ST_CUDA_TRY(cudaGetLastError());
  g_launches = launches;
  if (p.ext_reduce && g.defer) {
    g.defer->ws = p.ws;
    g.defer->splits = p.splits;
    g.defer->tiles = mt_grid * nt;
    g.defer->mt = mt_grid;
    g.defer->bm = BM;
    g.defer->bn = BNMAX;
  } else if (p.ext_reduce) {
    ST_TRY(launch_splitk_epilogue<EPI>(p, mt_grid * nt, mt_grid, g.stream, g.pdl));
    g_launches = launches + 1;
  }
  return ST_OK;
}

}  // namespace

int device_sm_count() { return num_sms(); }

// exported for the persistent LSTM recurrence (k_lstm_rec.cu)
bool tc_make_map(CUtensorMap* m, const float* base, int inner, int outer, int pitch, int box_outer, bool mn_major) {
  return make_map(m, base, inner, outer, pitch, box_outer, mn_major);
}
st_status tc_ensure_max_smem(const void* fn, int bytes) { return ensure_max_smem(fn, bytes); }
uint32_t make_idesc_tf32(int bn, int mma_m) { return make_idesc(bn, false, false, mma_m); }

int tc_last_launches() { return g_launches; }
// counters (64 KB, zero-initialised by the owner, self-resetting) + split-K partials
// for up to 2 × #SMs output tiles of 128 × 128 fp32.
// + the lo part of the activation operand (B × max width fp32) for the FP32X3 fwd / dX.
// lo tails: dW needs both dZ and X (B × (out + in), each padded to 64 floats).
int64_t tc_workspace_bytes(int B, int max_in, int max_out) {
  const int64_t lo = ((int64_t)B * max_out + 63) / 64 * 64 + ((int64_t)B * max_in + 63) / 64 * 64;
  return (int64_t)kCounterBytes + (int64_t)2 * kWsSms * BNMAX * BM * 4 + std::max<int64_t>(64, lo) * 4 + 256;
}

st_status simt_fwd(const GemmArgs& g, const float* X, const float* W, const float* bias, float* Z, int relu);
st_status simt_dx(const GemmArgs& g, const float* dZ, const float* W, const float* mask, float* D);
st_status simt_dw(const GemmArgs& g, const float* X, const float* dZ, float* G, float* gb);
int simt_last_launches();

// Forward GEMMs with many row tiles (N = T·B ≥ 8 × 128: the LSTM input projections, the LM
// softmax, explicit-im2col convs) on the persistent TMEM-A kernel instead of one CTA pair per
// tile: a CTA's next tile fills one accumulator while the epilogue drains the other. LM
// per-layer profile: softmax forward 653 → 610 µs, LSTM forward 1048 → 1000 µs
// (gpurun_out/r2ft). ST_FWD_TSG=0 (development build): the CTA-pair kernel.
bool tall_fwd_tsg() {
  static int f = -1;
  if (f < 0) f = dev_knob("ST_FWD_TSG", 1) != 0 ? 1 : 0;
  return f != 0;
}

// fwd: M = out, N = B, K = in
st_status tc_fwd(const GemmArgs& g, const float* X, const float* W, const float* bias, float* Z, int relu) {
  if (!tma_ok(W, g.n_out) || !tma_ok(X, g.n_in) || !get_encode()) {
    // TMA needs 16-byte pitches (e.g. the 10-wide output layer): CUDA-core split-K path
    st_status s = simt_fwd(g, X, W, bias, Z, relu);
    g_launches = simt_last_launches();
    return s;
  }
  CUtensorMap ma, mb;
  if (g.mode == ST_GEMM_FP32X3 && !(tall_fwd_tsg() && g.B >= 8 * BNMAX && !g.defer)) {
    if (!make_map(&ma, W, g.n_out, g.n_in, g.n_out, 32, true))
      return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (fwd)");
    return launch_ts<EPI_FWD, true>(g, g.n_out, g.B, g.n_in, ma, X, Z, bias, relu);
  }
  if (g.mode == ST_GEMM_FP32X3) {  // tall forward (T·B rows: LSTM input projection, LM softmax)
    if (!make_map(&ma, W, g.n_out, g.n_in, g.n_out, 32, true) || !make_map(&mb, X, g.n_in, g.B, g.n_in, BNMAX, false))
      return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (fwd)");
    return launch<EPI_FWD, true, false>(g, g.n_out, g.B, g.n_in, ma, mb, Z, bias, relu, 0, 0, 0, true);
  }
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
  if (g.mode == ST_GEMM_FP32X3) {
    if (!make_map(&ma, W, g.n_out, g.n_in, g.n_out, BM, false))
      return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (dX)");
    return launch_ts<EPI_DX, false>(g, g.n_in, g.B, g.n_out, ma, dZ, D, mask, 0);
  }
  if (!make_map(&ma, W, g.n_out, g.n_in, g.n_out, BM, false) || !make_map(&mb, dZ, g.n_out, g.B, g.n_out, bn_for(g.B), false))
    return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (dX)");
  return launch<EPI_DX, false, false>(g, g.n_in, g.B, g.n_out, ma, mb, D, mask, 0);
}

// dW: M = out, N = in, K = B. upd != NULL: fused K-B update of the weight block
// (and, via gb_upd, of the bias block) instead of writing G / gb.
st_status tc_dw_impl(const GemmArgs& g, const float* X, const float* dZ, float* G, float* gb, const UpdateArgs* upd,
                     const UpdateArgs* gb_upd);
st_status tc_dw(const GemmArgs& g, const float* X, const float* dZ, float* G, float* gb) {
  return tc_dw_impl(g, X, dZ, G, gb, nullptr, nullptr);
}
bool tc_dw_fusable(const GemmArgs& g, const float* X, const float* dZ) {
  return aligned16(dZ) && g.n_out % 4 == 0 && aligned16(X) && g.n_in % 4 == 0 && get_encode() && g.B <= DW_KMAX &&
         g.mode != ST_GEMM_SIMT;
}
st_status tc_dw_update(const GemmArgs& g, const float* X, const float* dZ, const UpdateArgs& w, const UpdateArgs& b) {
  return tc_dw_impl(g, X, dZ, nullptr, nullptr, &w, b.W ? &b : nullptr);
}
bool tc_dw_update_aligned(const UpdateArgs& w) {
  return aligned16(w.W) && aligned16(w.V) && (!w.WF || aligned16(w.WF)) && (!w.WB || aligned16(w.WB));
}
st_status tc_dw_impl(const GemmArgs& g, const float* X, const float* dZ, float* G, float* gb, const UpdateArgs* upd,
                     const UpdateArgs* gb_upd) {
  if (!tma_ok(dZ, g.n_out) || !tma_ok(X, g.n_in) || !get_encode()) {
    st_status s = simt_dw(g, X, dZ, G, gb);
    g_launches = simt_last_launches();
    return s;
  }
  if (g.B <= DW_KMAX) {
    // persistent kernel: lo of dZ and X precomputed into the workspace tail
    const bool x3 = g.mode == ST_GEMM_FP32X3;
    float* lo_base = reinterpret_cast<float*>(static_cast<char*>(g.work) + kCounterBytes +
                                              (size_t)2 * kWsSms * BNMAX * BM * 4);
    float* dzlo = lo_base;
    float* xlo = lo_base + (((size_t)g.B * g.n_out + 63) / 64 * 64);
    int launches = 1;
    (void)dzlo;
    if (x3) {
      const size_t n4b = (size_t)g.B * g.n_in / 4;
      ST_TRY(launch_maybe_pdl(g.pdl, split_lo_kernel, dim3((unsigned)std::min<size_t>(4 * (size_t)num_sms(), (n4b + 255) / 256)),
                              dim3(256), 0, g.stream, reinterpret_cast<const float4*>(X),
                              reinterpret_cast<float4*>(xlo), n4b));
      launches += 1;
    }
    CUtensorMap ma, mb, mblo;
    if (!make_map(&ma, dZ, g.n_out, g.B, g.n_out, 32, true) || !make_map(&mb, X, g.n_in, g.B, g.n_in, 32, true) ||
        !make_map(&mblo, xlo, g.n_in, g.B, g.n_in, 32, true))
      return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (dW)");
    TcParams p{};
    p.M = g.n_out;
    p.N = g.n_in;
    p.K = g.B;
    p.kb_total = (g.B + BK - 1) / BK;
    p.splits = 1;
    p.bn = bn_for(g.n_in);
    p.out = G;
    p.dev_flags = dev_flags();
    CUtensorMap mw, mv;
    memset(&mw, 0, sizeof(mw));
    memset(&mv, 0, sizeof(mv));
    if (upd) {
      p.upd = *upd;
      // W / V block [N rows][M cols] (element (n, m) at n·M + m), box 128 (m) × 16 (n), no swizzle
      p.wv_stream = (g.n_out % 4 == 0) && make_plain_map(&mw, upd->W, g.n_out, g.n_in, BM, DW_WV_COLS) &&
                    make_plain_map(&mv, upd->V, g.n_out, g.n_in, BM, DW_WV_COLS);
    }
    p.idesc = make_idesc(p.bn, false, true);  // A from TMEM, B MN-major
    const int mt = (g.n_out + BM - 1) / BM, nt = (g.n_in + BNMAX - 1) / BNMAX;
    const int budget = g.max_ctas > 0 ? std::min(g.max_ctas, num_sms()) : num_sms();
    int grid = std::min(mt * nt, budget);
    p.wv_direct = p.wv_stream ? dw_direct_mode() : 0;
    const int lm = dw_lockstep_mode();
    if ((lm == 1 || (lm == 2 && g.max_ctas <= 0)) && mt <= budget && nt >= budget / mt) {
      grid = (budget / mt) * mt;  // whole m-tile columns (see TcParams::lockstep)
      p.lockstep = 1;
    }
    auto kern = upd ? (x3 ? tc_dw_kernel<true, true> : tc_dw_kernel<false, true>)
                    : (x3 ? tc_dw_kernel<true, false> : tc_dw_kernel<false, false>);
    ST_TRY(ensure_max_smem((const void*)kern, dw_smem_bytes()));
    ST_TRY(launch_maybe_pdl(g.pdl, kern, dim3(grid), dim3(DW_THREADS), (size_t)dw_smem_bytes(), g.stream, ma, mb,
                            mblo, mw, mv, p, mt, nt));
    if (gb_upd) {
      ST_TRY(launch_bias_grad_update(dZ, g.B, g.n_out, *gb_upd, g.stream));
      ++launches;
    } else if (gb) {
      const int n = launch_bias_grad(dZ, g.B, g.n_out, gb, nullptr, 0, g.stream);
      if (n < 0) return set_error(ST_ERR_CUDA, "bias gradient launch failed");
      launches += n;
    }
    g_launches = launches;
    return ST_OK;
  }
  CUtensorMap ma, mb;
  if (!make_map(&ma, dZ, g.n_out, g.B, g.n_out, 32, true) || !make_map(&mb, X, g.n_in, g.B, g.n_in, 32, true))
    return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (dW)");
  ST_TRY((launch<EPI_DW, true, true>(g, g.n_out, g.n_in, g.B, ma, mb, G, nullptr, 0)));
  if (gb) {
    // the GEMM's split-K partials are consumed by the time this runs (same stream)
    const int n = launch_bias_grad(dZ, g.B, g.n_out, gb, g.work, g.work_bytes, g.stream);
    if (n < 0) return set_error(ST_ERR_CUDA, "bias gradient launch failed");
    g_launches = 1 + n;
  }
  return ST_OK;
}

// ---------------------------------------------------------------- implicit-GEMM conv
namespace {

// Pixel box of `rows` consecutive NHWC pixels (a tile never straddles a partial image
// row): {w, h, b} extents, or false when the geometry cannot be tiled that way.
bool act_box(int H, int W, int rows, cuuint32_t* box) {
  if (W >= rows) {
    if (W % rows) return false;
    box[0] = rows, box[1] = 1, box[2] = 1;
  } else {
    if (rows % W) return false;
    const int hb = rows / W;
    if (hb <= H) {
      if (H % hb) return false;
      box[0] = W, box[1] = hb, box[2] = 1;
    } else {
      if (hb % H) return false;
      box[0] = W, box[1] = H, box[2] = hb / H;
    }
  }
  return box[0] <= 256 && box[1] <= 256 && box[2] <= 256;
}

// NHWC tensor [B][H][W][C] (fp32) as a 4-D map (dims C, W, H, B), box {32 channels,
// `rows` pixels}; SWIZZLE_128B (K-major operand) or SWIZZLE_128B_ATOM_32B (MN-major):
// the box lands in smem exactly like the 2-D box {32, rows} of a [pixels × C] matrix.
bool make_act_map(CUtensorMap* m, const float* base, int B, int H, int W, int C, int rows, bool mn_major) {
  EncodeFn enc = get_encode();
  cuuint32_t pb[3];
  if (!enc || !aligned16(base) || (C % 32) || !act_box(H, W, rows, pb)) return false;
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)C * 4, (cuuint64_t)W * C * 4, (cuuint64_t)H * W * C * 4};
  cuuint32_t box[4] = {32, pb[0], pb[1], pb[2]};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// HWIO weights viewed as [9][Cin][Cout] (dims Cout, Cin, 9), box {32 co, bn ci, 1 tap}:
// the K-major B operand of the conv dX (K = (tap, co)).
bool make_w3_map(CUtensorMap* m, const float* base, int Cin, int Cout, int bn) {
  EncodeFn enc = get_encode();
  if (!enc || !aligned16(base) || (Cout % 4)) return false;
  cuuint64_t dims[3] = {(cuuint64_t)Cout, (cuuint64_t)Cin, 9};
  cuuint64_t strides[2] = {(cuuint64_t)Cout * 4, (cuuint64_t)Cin * Cout * 4};
  cuuint32_t box[3] = {32, (cuuint32_t)bn, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool implicit_conv_off() {
  static int f = -1;
  if (f < 0) {
    f = dev_knob("ST_CONV_IM2COL", 0) == 1 ? 1 : 0;
  }
  return f != 0;
}

}  // namespace

bool tc_conv_ok(int mode, int H, int W, int Cin, int Cout) {
  cuuint32_t b[3];
  return !implicit_conv_off() && (mode == ST_GEMM_FP32X3 || mode == ST_GEMM_TF32) && get_encode() &&
         Cin % 32 == 0 && Cout % 32 == 0 && act_box(H, W, BM, b) && act_box(H, W, 32, b);
}

// Conv forward on the CTA-pair TMEM-A kernel (tc_ts2_kernel<…, CONV>): weights on M
// (Cout ≥ 256, so every pair tile is full), pixels on N — the pair's MMAs run at ~1.5× the
// per-SM rate of the single-CTA N ≤ 128 ones (profiles/r1_probe_mma_rate_tf32.txt). The
// activation lo is split once into the workspace tail. Default since round 2 (with PDL and
// graph sessions in the step): VGG-16 62.3k → 63.4k samples/s (two runs each, one box);
// round 1 had measured it neutral (58.9k vs 59.0k). ST_CONV_PAIR=0: single-CTA conv forward.
bool conv_pair_on() {
  static int f = -1;
  if (f < 0) {
    f = dev_knob("ST_CONV_PAIR", 1) != 0 ? 1 : 0;
  }
  return f != 0;
}

st_status tc_conv_fwd_pair(const GemmArgs& g, const float* X, int H, int W, int Cin, int Cout, const float* Wt,
                           const float* bias, float* Y, int relu) {
  const int P = g.B * H * W, K = 9 * Cin;
  TcParams p{};
  const int budget = g.max_ctas > 0 ? std::min(g.max_ctas, num_sms()) : num_sms();
  const int mt = (Cout + BM - 1) / BM, mt_grid = (mt + 1) / 2 * 2;
  plan_splits(p, mt_grid * BM, P, K, budget / 2 * 2);
  const int nt = (P + BNMAX - 1) / BNMAX;
  if (p.bn != BNMAX) return set_error(ST_ERR_INPUT, "conv fwd pair: needs P >= %d pixels (got %d)", BNMAX, P);
  p.mt = mt_grid;
  p.tiles = mt_grid * nt;
  p.M = Cout;
  p.out = Y;
  p.aux = bias;
  p.relu = relu;
  p.cv_H = H;
  p.cv_W = W;
  p.cv_C = Cin;
  p.counters = reinterpret_cast<int*>(g.work);
  p.ws = reinterpret_cast<float*>(static_cast<char*>(g.work) + kCounterBytes);
  p.idesc = make_idesc(p.bn, false, false, 2 * BM);
  p.dev_flags = dev_flags();
  p.ext_reduce = p.splits >= ext_reduce_splits();
  float* xlo = reinterpret_cast<float*>(static_cast<char*>(g.work) + kCounterBytes +
                                        (size_t)2 * kWsSms * BNMAX * BM * 4);
  const size_t n4 = (size_t)P * Cin / 4;
  split_lo_kernel<<<std::min<size_t>(4 * (size_t)num_sms(), (n4 + 255) / 256), 256, 0, g.stream>>>(
      reinterpret_cast<const float4*>(X), reinterpret_cast<float4*>(xlo), n4);
  ST_CUDA_TRY(cudaGetLastError());
  CUtensorMap ma, mb, mblo;
  if (!make_map(&ma, Wt, Cout, K, Cout, 32, true) || !make_act_map(&mb, X, g.B, H, W, Cin, BNMAX / 2, false) ||
      !make_act_map(&mblo, xlo, g.B, H, W, Cin, BNMAX / 2, false))
    return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (conv fwd, pair)");
  auto kern = ts_split_acc() ? tc_ts2_kernel<EPI_FWD, true, true, true> : tc_ts2_kernel<EPI_FWD, true, false, true>;
  ST_TRY(ensure_max_smem((const void*)kern, ts2_smem_bytes()));
  dim3 grid(mt_grid, nt, p.splits);
  kern<<<grid, TS_THREADS, ts2_smem_bytes(), g.stream>>>(ma, mb, mblo, p);
  ST_CUDA_TRY(cudaGetLastError());
  g_launches = 2;
  if (p.ext_reduce) {
    ST_TRY(launch_splitk_epilogue<EPI_FWD>(p, mt_grid * nt, mt_grid, g.stream));
    g_launches = 3;
  }
  return ST_OK;
}

// Y[P × Cout] = conv3x3(X) + b, optional ReLU (NHWC; g.B = images)
st_status tc_conv_fwd(const GemmArgs& g, const float* X, int H, int W, int Cin, int Cout, const float* Wt,
                      const float* bias, float* Y, int relu) {
  const int P = g.B * H * W;
  cuuint32_t pb[3];
  // P ≥ 128: the pair's N tile is the full 128 pixels, so each CTA's window box is exactly the
  // 64 pixels its TMA map describes (a narrower tile would expect fewer bytes than it loads)
  if (g.mode == ST_GEMM_FP32X3 && Cout >= 2 * BM && P >= BNMAX && use_pair() && conv_pair_on() &&
      act_box(H, W, BNMAX / 2, pb))
    return tc_conv_fwd_pair(g, X, H, W, Cin, Cout, Wt, bias, Y, relu);
  CUtensorMap ma, mb;
  if (!make_act_map(&ma, X, g.B, H, W, Cin, BM, false) || !make_map(&mb, Wt, Cout, 9 * Cin, Cout, 32, true))
    return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (conv fwd)");
  return launch<EPI_FWD, false, true, CV_FWD>(g, P, Cout, 9 * Cin, ma, mb, Y, bias, relu, H, W, Cin);
}

// D[P × Cin] = conv3x3ᵀ(dZ) ⊙ 1[mask > 0] (mask may be null)
st_status tc_conv_dx(const GemmArgs& g, const float* dZ, int H, int W, int Cin, int Cout, const float* Wt,
                     const float* mask, float* D) {
  const int P = g.B * H * W;
  CUtensorMap ma, mb;
  if (!make_act_map(&ma, dZ, g.B, H, W, Cout, BM, false) || !make_w3_map(&mb, Wt, Cin, Cout, bn_for(Cin)))
    return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (conv dX)");
  return launch<EPI_DX, false, false, CV_DX>(g, P, Cin, 9 * Cout, ma, mb, D, mask, 0, H, W, Cout);
}

// G[9·Cin × Cout] = Σ_p col(X)[p]ᵀ dZ[p]; gb[Cout] = Σ_p dZ[p] (gb may be null).
// Cout ≥ 128: M = Cout (full 128-row tiles), N = 9·Cin; else M = 9·Cin, N = Cout.
st_status tc_conv_dw(const GemmArgs& g, const float* X, const float* dZ, int H, int W, int Cin, int Cout, float* G,
                     float* gb) {
  const int P = g.B * H * W;
  CUtensorMap ma, mb;
  if (Cout < BM) {
    if (!make_act_map(&ma, X, g.B, H, W, Cin, 32, true) || !make_map(&mb, dZ, Cout, P, Cout, 32, true))
      return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (conv dW)");
    ST_TRY((launch<EPI_DW, true, true, CV_DWT>(g, 9 * Cin, Cout, P, ma, mb, G, nullptr, 0, H, W, Cin)));
  } else {
    if (!make_map(&ma, dZ, Cout, P, Cout, 32, true) || !make_act_map(&mb, X, g.B, H, W, Cin, 32, true))
      return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (conv dW)");
    ST_TRY((launch<EPI_DW, true, true, CV_DW>(g, Cout, 9 * Cin, P, ma, mb, G, nullptr, 0, H, W, Cin)));
  }
  int launches = g_launches;
  if (gb) {
    const int n = launch_bias_grad(dZ, P, Cout, gb, g.work, g.work_bytes, g.stream);
    if (n < 0) return set_error(ST_ERR_CUDA, "bias gradient launch failed");
    launches += n;
  }
  g_launches = launches;
  return ST_OK;
}

// First conv (Cin·9 < 32, e.g. RGB): explicit im2col into rows padded to 32 columns
// (col[p][k], k ≥ 9·Cin zero) so both GEMMs take the TMA / tcgen05 path; the weight
// rows past 9·Cin are outside the [9·Cin × Cout] map, so TMA zero-fills them.
bool tc_conv_small_ok(int mode, int Cin, int Cout) {
  return !implicit_conv_off() && (mode == ST_GEMM_FP32X3 || mode == ST_GEMM_TF32) && get_encode() && 9 * Cin <= 32 &&
         Cout % 4 == 0;
}

st_status tc_conv_small_fwd(const GemmArgs& g, const float* col, int H, int W, int Cin, int Cout, const float* Wt,
                            const float* bias, float* Y, int relu) {
  const int P = g.B * H * W;
  CUtensorMap ma, mb;
  if (!make_map(&ma, col, 32, P, 32, BM, false) || !make_map(&mb, Wt, Cout, 9 * Cin, Cout, 32, true))
    return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (first conv fwd)");
  return launch<EPI_FWD, false, true, CV_ROWS>(g, P, Cout, 32, ma, mb, Y, bias, relu);
}

st_status tc_conv_small_dw(const GemmArgs& g, const float* col, const float* dZ, int H, int W, int Cin, int Cout,
                           float* G, float* gb) {
  const int P = g.B * H * W;
  CUtensorMap ma, mb;
  if (!make_map(&ma, dZ, Cout, P, Cout, 32, true) || !make_map(&mb, col, 9 * Cin, P, 32, 32, true))
    return set_error(ST_ERR_CUDA, "cuTensorMapEncodeTiled failed (first conv dW)");
  ST_TRY((launch<EPI_DW, true, true>(g, Cout, 9 * Cin, P, ma, mb, G, nullptr, 0)));
  int launches = g_launches;
  if (gb) {
    const int n = launch_bias_grad(dZ, P, Cout, gb, g.work, g.work_bytes, g.stream);
    if (n < 0) return set_error(ST_ERR_CUDA, "bias gradient launch failed");
    launches += n;
  }
  g_launches = launches;
  return ST_OK;
}

}  // namespace st
