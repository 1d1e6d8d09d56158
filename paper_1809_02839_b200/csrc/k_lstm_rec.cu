// K-D2: persistent LSTM recurrence (P:377-380 LM workload, reading D18).
// DEVELOPMENT VARIANT (opt-in ST_LSTM_PERSIST=1 in the -DST_DEV_KNOBS build; the product
// library keeps the per-step GEMM + cell path, measured faster: DESIGN.md §5).
//
// One launch runs all T time steps of one LSTM layer in one direction. Per step the
// recurrent product is a small GEMM (B × H by H × 4H) whose result every CTA needs before
// the next step, so a launch per step (GEMM, then cell) pays launch, ramp and split-K
// reduce latency 2T times. Here the grid stays resident (cooperative launch, one CTA per
// SM) and a step is:
//   1. MMA phase   : CTA (q, s) computes tile q of the recurrent product over K split s
//                    (3xTF32: W_hh tile → TMEM hi / lo by the converter warps, the activation
//                    hi / lo tiles by TMA, three kind::tf32 MMAs per K step of 8; the two small
//                    terms in a second accumulator) and writes its partial to the workspace.
//   2. tile sync   : the S CTAs of tile q meet on a per-tile counter.
//   3. cell phase  : each of them applies the cell to its 1/S of the batch rows of tile q,
//                    summing the S partials in split order (deterministic).
//   4. grid sync   : a monotonic grid counter; the TMA producer waits on it before loading
//                    the step's activation (h_t / dG_t, written by every CTA). The W_hh tiles
//                    of the first ring stages are loaded and converted before the wait.
// Forward  (t = 0 .. T−1): rec = h_{t−1}·W_hh; tiles are gate-interleaved: tile q owns the
//   hidden units j ∈ [32q, 32q+32) and M row m = g·32 + (j − 32q) is column g·H + j of W_hh,
//   so one tile holds all four gates of its units and the cell needs nothing else.
//   A = W_hh [k][g·H + j] (MN-major, four 32-column boxes), B = h_{t−1} [b][k] (K-major).
// Backward (t = T−1 .. 0): dh_t = dG_{t+1}·W_hhᵀ; tile q owns units j ∈ [128q, 128q+128);
//   A = W_hh [j][k] (K-major), B = dG_{t+1} [b][k] (K-major), K = 4H.
// The cell arithmetic is the one of lstm_cell_fwd_kernel / lstm_cell_bwd_kernel (k_lstm.cu).
#include "kernels.hpp"
#include "knobs.hpp"
#include "tc_ptx.cuh"

#ifdef ST_DEV_KNOBS
namespace st {

bool tc_make_map(CUtensorMap* m, const float* base, int inner, int outer, int pitch, int box_outer, bool mn_major);
st_status tc_ensure_max_smem(const void* fn, int bytes);
uint32_t make_idesc_tf32(int bn, int mma_m);

namespace {
using namespace ptx;

constexpr int RS = 4;                     // ring stages = TMEM A slots
constexpr int R_TILE = 128 * 32 * 4;      // 16 KB: one 128 × 32 fp32 operand tile
constexpr int R_STAGE = 3 * R_TILE;       // A raw, B hi, B lo
constexpr int R_THREADS = 320;            // producer, MMA, 4 converter warps, 4 epilogue / cell warps
constexpr int R_SMEM = RS * R_STAGE + 1024 + 256;
constexpr int R_CELL_U = 6;               // cells per thread per batch of loads (latency hiding)
constexpr int R_SPC = 3;                  // fwd: K-split partials (× 4 gates) loaded per round trip
constexpr int R_SPC_B = 12;               // bwd: K-split partials loaded per round trip
constexpr size_t R_BAR_OFFSET = 16 * 1024;  // counters inside the GEMM workspace's counter block

struct RecParams {
  int B, H, T;
  int nt, splits, kb_total, kb_per_split;
  uint32_t idesc;
  float* ws;          // partials [nt][splits][128 n (= b)][128 m]
  unsigned* bar;      // [0] grid counter, [1 + q] tile counters (zeroed before the launch)
  float* gates;       // fwd: [T][B][4H] Gx_t in, activated gates out; bwd: activated gates (read)
  float* hbuf;        // fwd: [(T+1)][B][H], hbuf[0] = h_{−1} = 0
  float* cbuf;        // [T][B][H] (fwd: written, bwd: read)
  float* lo;          // fwd: h lo [2][B][H]; bwd: dG lo [2][B][4H] (slot t & 1)
  const float* dOut;  // bwd: [T][B][H]
  float* dG;          // bwd: [T][B][4H]
  float* dc;          // bwd: [B][H]
  int dbg;            // development timeline (rec_mark)
};

#ifdef ST_DEV_KNOBS
// development timeline (ST_LSTM_DBG=1): %globaltimer at 5 points of iteration i of CTA b
constexpr int kDbgIters = 40, kDbgCtas = 160;
__device__ uint64_t g_rec_dbg[kDbgIters * kDbgCtas * 8];
__device__ __forceinline__ void rec_mark(int on, int i, int k) {
  if (on && i < kDbgIters && blockIdx.x < kDbgCtas) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_rec_dbg[((size_t)i * kDbgCtas + blockIdx.x) * 8 + k] = t;
  }
}
#else
__device__ __forceinline__ void rec_mark(int, int, int) {}
#endif

__device__ __forceinline__ float sigm(float x) { return 1.0f / (1.0f + expf(-x)); }

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// Spin until *p ≥ target: relaxed polls with a short sleep between them (a tight loop of
// acquire loads from the producer warp slows the cell warps' loads on the same SM), then
// one acquire. A peer that never arrives (it cannot: the launch is cooperative, every CTA
// is resident) would hang the GPU: trap after ~4 s instead.
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_geq(const unsigned* p, unsigned target) {
  if (ld_acquire(p) >= target) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (ld_relaxed(p) < target) {
    __nanosleep(64);
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 4000000000ull) __trap();
  }
  (void)ld_acquire(p);
}
// 4 epilogue / cell warps (warps 6..9)
__device__ __forceinline__ void cell_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

template <bool BWD>
__global__ void __launch_bounds__(R_THREADS, 1)
    lstm_rec_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                    const __grid_constant__ CUtensorMap mapBlo, RecParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  char* smem = align_smem_1k(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + RS * R_STAGE);
  const uint32_t full_a = smem_u32(bars);      // A landed                       [RS]
  const uint32_t full_b = full_a + 8 * RS;     // B hi + lo landed               [RS]
  const uint32_t b_ready = full_b + 8 * RS;    // TMEM hi / lo written (4 warps) [RS]
  const uint32_t b_empty = b_ready + 8 * RS;   // MMAs done with stage + slot    [RS]
  const uint32_t acc_full = b_empty + 8 * RS;
  const uint32_t acc_empty = acc_full + 8;     // 4 epilogue warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4 * RS + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = blockIdx.x / p.splits, s = blockIdx.x % p.splits;
  const int kb0 = s * p.kb_per_split, kb1 = min(p.kb_total, kb0 + p.kb_per_split);
  const int nkb = kb1 - kb0;
  const int B = p.B, H = p.H, T = p.T;
  const unsigned G = gridDim.x;

  if (threadIdx.x == 0) {
    for (int i = 0; i < RS; ++i) {
      mbar_init(full_a + 8 * i, 1);
      mbar_init(full_b + 8 * i, 1);
      mbar_init(b_ready + 8 * i, 4);
      mbar_init(b_empty + 8 * i, 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 4);
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
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapBlo)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem2 = tmem + 128;  // the two small 3xTF32 terms
  const uint32_t tmemA = tmem + 256;  // RS slots of 64 columns (32 hi + 32 lo)

  if (warp == 0) {
    // ---------------- TMA producer. Iteration i ≥ 1 reads the activation written in
    // iteration i − 1 (fwd: h_{t−1} = hbuf[t]; bwd: dG_{t+1}) and its lo slot.
    int it = 0;
    for (int i = 1; i < T; ++i) {
      const int t = BWD ? T - 1 - i : i;
      const int brow = BWD ? (t + 1) * B : t * B;        // activation rows of this step
      const int lrow = (BWD ? ((t + 1) & 1) : ((t - 1) & 1)) * B;
      const int pre = min(RS, nkb);
      // W_hh tiles of the first stages do not depend on the previous step: load them first
      for (int u = 0; u < pre; ++u) {
        const int si = (it + u) % RS;
        mbar_wait(b_empty + 8 * si, (((it + u) / RS) & 1) ^ 1);
        if (elect_one()) {
          const uint32_t dA = smem_u32(smem + si * R_STAGE);
          mbar_expect_tx(full_a + 8 * si, R_TILE);
          const int k0 = (kb0 + u) * 32;
          if (BWD) {
            tma_load_2d(dA, &mapA, k0, q * 128, full_a + 8 * si);
          } else {
#pragma unroll
            for (int g = 0; g < 4; ++g) tma_load_2d(dA + g * 4096, &mapA, g * H + q * 32, k0, full_a + 8 * si);
          }
        }
        __syncwarp();
      }
      // the previous step's cells, on every CTA
      if (lane == 0) {
        wait_geq(p.bar, G * (unsigned)i);
        rec_mark(p.dbg, i, 0);
      }
      __syncwarp();
      fence_proxy_async_global();
      for (int u = 0; u < nkb; ++u, ++it) {
        const int si = it % RS;
        const int k0 = (kb0 + u) * 32;
        const uint32_t dA = smem_u32(smem + si * R_STAGE);
        if (u >= pre) {
          mbar_wait(b_empty + 8 * si, ((it / RS) & 1) ^ 1);
          if (elect_one()) {
            mbar_expect_tx(full_a + 8 * si, R_TILE);
            if (BWD) {
              tma_load_2d(dA, &mapA, k0, q * 128, full_a + 8 * si);
            } else {
#pragma unroll
              for (int g = 0; g < 4; ++g) tma_load_2d(dA + g * 4096, &mapA, g * H + q * 32, k0, full_a + 8 * si);
            }
          }
          __syncwarp();
        }
        if (elect_one()) {
          mbar_expect_tx(full_b + 8 * si, 2 * R_TILE);
          tma_load_2d(dA + R_TILE, &mapB, k0, brow, full_b + 8 * si);
          tma_load_2d(dA + 2 * R_TILE, &mapBlo, k0, lrow, full_b + 8 * si);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: A hi / lo from TMEM slot, B hi / lo from smem
    int it = 0;
    for (int i = 1; i < T; ++i) {
      mbar_wait(acc_empty, ((i - 1) & 1) ^ 1);
      tc_fence_after();
      for (int u = 0; u < nkb; ++u, ++it) {
        const int si = it % RS;
        mbar_wait(b_ready + 8 * si, (it / RS) & 1);
        mbar_wait(full_b + 8 * si, (it / RS) & 1);
        tc_fence_after();
        const uint32_t b_hi = smem_u32(smem + si * R_STAGE) + R_TILE, b_lo = b_hi + R_TILE;
        const uint32_t a_hi = tmemA + si * 64, a_lo = a_hi + 32;
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t acc = (u > 0 || kk > 0) ? 1u : 0u;
            tc_mma_ts(tmem, a_hi + kk * 8, desc_kmajor(b_hi + kk * 32), p.idesc, acc);
            tc_mma_ts(tmem2, a_lo + kk * 8, desc_kmajor(b_hi + kk * 32), p.idesc, acc);
            tc_mma_ts(tmem2, a_hi + kk * 8, desc_kmajor(b_lo + kk * 32), p.idesc, 1u);
          }
          tc_commit(b_empty + 8 * si);
          if (u == nkb - 1) {
            tc_commit(acc_full);
            rec_mark(p.dbg, i, 1);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp < 6) {
    // ---------------- converters: A row r → TMEM lane r (hi, lo)
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    int it = 0;
    for (int i = 1; i < T; ++i) {
      for (int u = 0; u < nkb; ++u, ++it) {
        const int si = it % RS;
        mbar_wait(full_a + 8 * si, (it / RS) & 1);
        const char* st = smem + si * R_STAGE;
        uint32_t hi[32], lo[32];
        if (!BWD) {
          // MN-major: element (k, r) in box r / 32, row k, 32-byte atoms swizzled by k % 4
          const char* box = st + (r >> 5) * 4096;
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const float x =
                *reinterpret_cast<const float*>(box + k * 128 + ((((r & 31) >> 3) ^ (k & 3)) << 5) + (r & 7) * 4);
            hi[k] = __float_as_uint(x);
            lo[k] = __float_as_uint(lo_part(x));
          }
        } else {
          // K-major SWIZZLE_128B: row r, 16-byte chunk c at (c ^ (r & 7))
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
        // TMEM slot si is free: the producer refilled the stage only after b_empty, which
        // commits after every MMA that read the slot
        tc_fence_after();
        const uint32_t taddr = tmemA + si * 64 + ((uint32_t)(quad * 32) << 16);
        tc_st32(taddr, hi);
        tc_st32(taddr + 32, lo);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(b_ready + 8 * si);
      }
    }
  } else {
    // ---------------- epilogue + cell (warps 6..9 → TMEM quadrants 2, 3, 0, 1)
    const int quad = warp & 3;
    const int ctid = (warp - 6) * 32 + lane;
    const int m = quad * 32 + lane;
    float* wsq = p.ws + (size_t)q * p.splits * (128 * 128);
    const int S = p.splits;
    const int b0 = s * B / S, b1 = (s + 1) * B / S;
    const int nj = BWD ? min(128, H - q * 128) : min(32, H - q * 32);
    const int j0 = BWD ? q * 128 : q * 32;
    const int ncell = (b1 - b0) * nj;
    const size_t BH = (size_t)B * H, B4H = (size_t)B * 4 * H;
    if (ctid == 0) rec_mark(p.dbg, 0, 6);  // kernel start (slot 6 is unused at i = 0)
    for (int i = 0; i < T; ++i) {
      const int t = BWD ? T - 1 - i : i;
      // while the MMAs run: pull this step's cell inputs that do not depend on them (Gx_t /
      // the stashed gates, c, dOut — long evicted to HBM) into L2
      for (int e = ctid; e < ncell; e += 128) {
        const int b = b0 + e / nj, j = j0 + e % nj;
        const float* g = p.gates + (size_t)t * B4H + (size_t)b * 4 * H + j;
#pragma unroll
        for (int gg = 0; gg < 4; ++gg) prefetch_l2(g + gg * H);
        if (BWD) {
          const size_t o = (size_t)b * H + j;
          prefetch_l2(p.cbuf + (size_t)t * BH + o);
          if (t) prefetch_l2(p.cbuf + (size_t)(t - 1) * BH + o);
          prefetch_l2(p.dOut + (size_t)t * BH + o);
        }
      }
      if (i > 0) {
        mbar_wait(acc_full, (i - 1) & 1);
        tc_fence_after();
        if (ctid == 0) rec_mark(p.dbg, i, 2);
        const uint32_t trow = tmem + ((uint32_t)(quad * 32) << 16), trow2 = tmem2 + ((uint32_t)(quad * 32) << 16);
        float* wsp = wsq + (size_t)s * (128 * 128);
#pragma unroll 1
        for (int c = 0; c < 128; c += 16) {
          uint32_t v[16], w[16];
          tc_ld16_nowait(trow + c, v);
          tc_ld16_nowait(trow2 + c, w);
          tc_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e)
            wsp[(size_t)(c + e) * 128 + m] = __uint_as_float(v[e]) + __uint_as_float(w[e]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty);
        if (ctid == 0) rec_mark(p.dbg, i, 6);
        __threadfence();
        cell_bar();
        if (ctid == 0) {
          atomicAdd(p.bar + 1 + q, 1u);
          wait_geq(p.bar + 1 + q, (unsigned)S * (unsigned)i);
          rec_mark(p.dbg, i, 3);
        }
        cell_bar();
      }
      // cells of (b ∈ [b0, b1), j ∈ [j0, j0 + nj)), R_CELL_U per thread with every load of
      // a batch issued before its arithmetic
      for (int e0 = ctid; e0 < ncell; e0 += 128 * R_CELL_U) {
        if (!BWD) {
          float gx[R_CELL_U][4], rc[R_CELL_U][4], cp[R_CELL_U];
#pragma unroll
          for (int u = 0; u < R_CELL_U; ++u) {
            const int e = e0 + u * 128;
#pragma unroll
            for (int gg = 0; gg < 4; ++gg) rc[u][gg] = 0.f;
            if (e < ncell) {
              const int b = b0 + e / nj, jj = e % nj, j = j0 + jj;
              const float* g = p.gates + (size_t)t * B4H + (size_t)b * 4 * H + j;
#pragma unroll
              for (int gg = 0; gg < 4; ++gg) gx[u][gg] = g[gg * H];
              cp[u] = t ? p.cbuf[(size_t)(t - 1) * BH + (size_t)b * H + j] : 0.f;
            }
          }
          // the S partials of every gate, in split order; R_SPC splits' loads in flight at once
          for (int sp0 = 0; i > 0 && sp0 < S; sp0 += R_SPC) {
            float v[R_CELL_U][R_SPC][4];
#pragma unroll
            for (int u = 0; u < R_CELL_U; ++u) {
              const int e = e0 + u * 128;
              const int b = b0 + e / nj, jj = e % nj;
#pragma unroll
              for (int k = 0; k < R_SPC; ++k)
#pragma unroll
                for (int gg = 0; gg < 4; ++gg)
                  v[u][k][gg] = (e < ncell && sp0 + k < S)
                                    ? __ldcg(wsq + ((size_t)(sp0 + k) * 128 + b) * 128 + jj + gg * 32)
                                    : 0.f;
            }
#pragma unroll
            for (int u = 0; u < R_CELL_U; ++u)
#pragma unroll
              for (int k = 0; k < R_SPC; ++k)
                if (sp0 + k < S) {
#pragma unroll
                  for (int gg = 0; gg < 4; ++gg) rc[u][gg] += v[u][k][gg];
                }
          }
#ifdef ST_DEV_KNOBS
          if (e0 == 0 && p.dbg) {  // the first batch's loads have landed
            asm volatile("" ::"f"(rc[0][0]), "f"(gx[0][0]), "f"(cp[0]));
            rec_mark(p.dbg, i, 7);
          }
#endif
#pragma unroll
          for (int u = 0; u < R_CELL_U; ++u) {
            const int e = e0 + u * 128;
            if (e < ncell) {
              const int b = b0 + e / nj, j = j0 + e % nj;
              const float gi = sigm(gx[u][0] + rc[u][0]);
              const float gf = sigm(gx[u][1] + rc[u][1]);
              const float gg = tanhf(gx[u][2] + rc[u][2]);
              const float go = sigm(gx[u][3] + rc[u][3]);
              const float c = gf * cp[u] + gi * gg;
              float* g = p.gates + (size_t)t * B4H + (size_t)b * 4 * H + j;
              g[0] = gi;
              g[H] = gf;
              g[2 * H] = gg;
              g[3 * H] = go;
              const size_t o = (size_t)b * H + j;
              p.cbuf[(size_t)t * BH + o] = c;
              const float h = go * tanhf(c);
              p.hbuf[(size_t)(t + 1) * BH + o] = h;
              p.lo[(size_t)(t & 1) * BH + o] = lo_part(h);
            }
          }
        } else {
          float ga[R_CELL_U][4], ct[R_CELL_U], cp[R_CELL_U], dO[R_CELL_U], dcn[R_CELL_U], dhn[R_CELL_U];
#pragma unroll
          for (int u = 0; u < R_CELL_U; ++u) {
            const int e = e0 + u * 128;
            dhn[u] = 0.f;
            if (e < ncell) {
              const int b = b0 + e / nj, jj = e % nj, j = j0 + jj;
              const float* g = p.gates + (size_t)t * B4H + (size_t)b * 4 * H + j;
#pragma unroll
              for (int gg = 0; gg < 4; ++gg) ga[u][gg] = g[gg * H];
              const size_t o = (size_t)b * H + j;
              ct[u] = p.cbuf[(size_t)t * BH + o];
              cp[u] = t ? p.cbuf[(size_t)(t - 1) * BH + o] : 0.f;
              dO[u] = p.dOut[(size_t)t * BH + o];
              dcn[u] = (i > 0) ? p.dc[o] : 0.f;
            }
          }
          for (int sp0 = 0; i > 0 && sp0 < S; sp0 += R_SPC_B) {
            float v[R_CELL_U][R_SPC_B];
#pragma unroll
            for (int u = 0; u < R_CELL_U; ++u) {
              const int e = e0 + u * 128;
              const int b = b0 + e / nj, jj = e % nj;
#pragma unroll
              for (int k = 0; k < R_SPC_B; ++k)
                v[u][k] = (e < ncell && sp0 + k < S) ? __ldcg(wsq + ((size_t)(sp0 + k) * 128 + b) * 128 + jj) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < R_CELL_U; ++u)
#pragma unroll
              for (int k = 0; k < R_SPC_B; ++k)
                if (sp0 + k < S) dhn[u] += v[u][k];
          }
#pragma unroll
          for (int u = 0; u < R_CELL_U; ++u) {
            const int e = e0 + u * 128;
            if (e < ncell) {
              const int b = b0 + e / nj, j = j0 + e % nj;
              const float gi = ga[u][0], gf = ga[u][1], gg = ga[u][2], go = ga[u][3];
              const float dh = dO[u] + dhn[u];
              const float tc = tanhf(ct[u]);
              const float dcv = dcn[u] + dh * go * (1.f - tc * tc);
              const float d0 = dcv * gg * gi * (1.f - gi);
              const float d1 = dcv * cp[u] * gf * (1.f - gf);
              const float d2 = dcv * gi * (1.f - gg * gg);
              const float d3 = dh * tc * go * (1.f - go);
              float* d = p.dG + (size_t)t * B4H + (size_t)b * 4 * H + j;
              d[0] = d0;
              d[H] = d1;
              d[2 * H] = d2;
              d[3 * H] = d3;
              float* l = p.lo + (size_t)(t & 1) * B4H + (size_t)b * 4 * H + j;
              l[0] = lo_part(d0);
              l[H] = lo_part(d1);
              l[2 * H] = lo_part(d2);
              l[3 * H] = lo_part(d3);
              p.dc[(size_t)b * H + j] = dcv * gf;
            }
          }
        }
      }
      if (ctid == 0) rec_mark(p.dbg, i, 5);
      // this CTA's cells of step t are written: grid counter (the producers wait on it)
      fence_proxy_async_global();
      __threadfence();
      cell_bar();
      if (ctid == 0) {
        rec_mark(p.dbg, i, 4);
        atomicAdd(p.bar, 1u);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// Cooperative launch of one direction; ST_ERR_UNSUPPORTED when the shapes or the device
// do not allow it (the caller then runs the per-step GEMM + cell path).
template <bool BWD>
st_status launch_rec(const GemmArgs& g, RecParams p, const float* Whh, const float* act, size_t act_rows) {
  const int H = p.H, B = p.B;
  int sms = device_sm_count();
  if (g.max_ctas > 0) sms = std::min(sms, g.max_ctas);
  p.nt = BWD ? (H + 127) / 128 : (H + 31) / 32;
  const int K = BWD ? 4 * H : H;
  p.kb_total = (K + 31) / 32;
  int S = std::min(sms / p.nt, p.kb_total);
  if (S < 1) return ST_ERR_UNSUPPORTED;
  p.kb_per_split = (p.kb_total + S - 1) / S;
  p.splits = (p.kb_total + p.kb_per_split - 1) / p.kb_per_split;
  const int grid = p.nt * p.splits;
  auto kern = lstm_rec_kernel<BWD>;
  ST_TRY(tc_ensure_max_smem((const void*)kern, R_SMEM));
  int per_sm = 0;
  ST_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, R_THREADS, R_SMEM));
  if (per_sm < 1 || grid > per_sm * device_sm_count()) return ST_ERR_UNSUPPORTED;
  CUtensorMap ma, mb, mblo;
  bool ok;
  if (BWD)  // W_hh [H rows j][4H k], box {32 k, 128 j}, K-major
    ok = tc_make_map(&ma, Whh, 4 * H, H, 4 * H, 128, false);
  else      // W_hh [H rows k][4H cols], box {32 cols, 32 k}, MN-major
    ok = tc_make_map(&ma, Whh, 4 * H, H, 4 * H, 32, true);
  ok = ok && tc_make_map(&mb, act, K, (int)act_rows, K, 128, false) && tc_make_map(&mblo, p.lo, K, 2 * B, K, 128, false);
  if (!ok) return ST_ERR_UNSUPPORTED;
  p.idesc = make_idesc_tf32(128, 128);
  p.dbg = dev_knob("ST_LSTM_DBG", 0) == (BWD ? 2 : 1);
  p.bar = reinterpret_cast<unsigned*>(static_cast<char*>(g.work) + R_BAR_OFFSET);
  p.ws = reinterpret_cast<float*>(static_cast<char*>(g.work) + 64 * 1024);
  ST_CUDA_TRY(cudaMemsetAsync(p.bar, 0, (size_t)(1 + p.nt) * 4, g.stream));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(R_THREADS);
  cfg.dynamicSmemBytes = R_SMEM;
  cfg.stream = g.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  ST_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ma, mb, mblo, p));
  return ST_OK;
}

// ST_LSTM_PERSIST: 1 = both directions, 2 = backward only, 3 = forward only
bool rec_shapes_ok(const GemmArgs& g, int B, int H, int T, bool bwd) {
  const int v = dev_knob("ST_LSTM_PERSIST", 0);
  const bool on = v == 1 || v == (bwd ? 2 : 3);
  return on && g.mode == ST_GEMM_FP32X3 && B >= 1 && B <= 128 && H % 4 == 0 && T >= 1 && g.work;
}

}  // namespace

st_status lstm_rec_fwd(const GemmArgs& g, int B, int H, int T, const float* Whh, float* gates, float* hbuf,
                       float* cbuf, float* hlo2) {
  if (!rec_shapes_ok(g, B, H, T, false)) return ST_ERR_UNSUPPORTED;
  RecParams p{};
  p.B = B;
  p.H = H;
  p.T = T;
  p.gates = gates;
  p.hbuf = hbuf;
  p.cbuf = cbuf;
  p.lo = hlo2;
  return launch_rec<false>(g, p, Whh, hbuf, (size_t)(T + 1) * B);
}

st_status lstm_rec_bwd(const GemmArgs& g, int B, int H, int T, const float* Whh, const float* gates,
                       const float* cbuf, const float* dOut, float* dG, float* dglo2, float* dc) {
  if (!rec_shapes_ok(g, B, H, T, true)) return ST_ERR_UNSUPPORTED;
  RecParams p{};
  p.B = B;
  p.H = H;
  p.T = T;
  p.gates = const_cast<float*>(gates);
  p.cbuf = const_cast<float*>(cbuf);
  p.dOut = dOut;
  p.dG = dG;
  p.lo = dglo2;
  p.dc = dc;
  return launch_rec<true>(g, p, Whh, dG, (size_t)T * B);
}

#ifdef ST_DEV_KNOBS
// development: copy the last launch's timeline out (n ≥ kDbgIters · kDbgCtas · 8)
extern "C" __attribute__((visibility("default"))) int st_dev_lstm_rec_timeline(uint64_t* out, int n) {
  if (n < kDbgIters * kDbgCtas * 8) return -1;
  cudaDeviceSynchronize();
  return cudaMemcpyFromSymbol(out, g_rec_dbg, sizeof(uint64_t) * kDbgIters * kDbgCtas * 8) == cudaSuccess ? 0 : -2;
}
#endif

}  // namespace st
#else  // product build: the per-step path (measured faster)

namespace st {
st_status lstm_rec_fwd(const GemmArgs&, int, int, int, const float*, float*, float*, float*, float*) {
  return ST_ERR_UNSUPPORTED;
}
st_status lstm_rec_bwd(const GemmArgs&, int, int, int, const float*, const float*, const float*, const float*, float*,
                       float*, float*) {
  return ST_ERR_UNSUPPORTED;
}
}  // namespace st
#endif
