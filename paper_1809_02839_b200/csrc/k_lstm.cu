// K-D / K-E: LSTM cell and embedding kernels of the LM stages.
//
// LSTM (reading D18: gate order i, f, g, o; one bias; h_{-1} = c_{-1} = 0):
//   forward step t : G = Gx_t + h_{t−1}·W_hh  (the GEMM runs in k_gemm_tc.cu)
//                    i, f, o = σ(G), g = tanh(G); c_t = f⊙c_{t−1} + i⊙g; h_t = o⊙tanh(c_t)
//   backward step t: dh = dOut_t + dh_next; dc = dc_next + dh⊙o⊙(1 − tanh²c_t)
//                    dG = [dc⊙g⊙i(1−i), dc⊙c_{t−1}⊙f(1−f), dc⊙i⊙(1−g²), dh⊙tanh(c_t)⊙o(1−o)]
//                    dc_next = dc⊙f      (dh_next = dG·W_hhᵀ is a GEMM)
// Embedding: forward gathers rows of E; the gradient is a deterministic segmented
// sum (tokens bucketed by a counting sort, each bucket summed in row order).
#include "kernels.hpp"

namespace st {
namespace {

__device__ __forceinline__ float sigm(float x) { return 1.0f / (1.0f + expf(-x)); }

// x − trunc_tf32(x): the lo half of the 3xTF32 split of the next GEMM's activation
// operand (the same expression as k_gemm_tc.cu split_lo_kernel, written independently)
__device__ __forceinline__ float tf32_lo(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// Elements (row n, columns m + j·step, j < J) of a GEMM output [rows × ld]: direct, or
// the sums of the deferred split-K partials (SplitPlan, kernels.hpp) — each in split order
// from 0.f (bit-identical to the reduce kernel), with every load of a 4-split group issued
// before its adds (the partials come from L2: latency, not bandwidth, bounds this).
template <int J>
__device__ __forceinline__ void gemm_out(const float* direct, const SplitPlan& p, int n, int m, int step, int ld,
                                         float* out) {
  if (p.splits <= 1) {
#pragma unroll
    for (int j = 0; j < J; ++j) out[j] = direct[(size_t)n * ld + m + j * step];
    return;
  }
  const size_t stride = (size_t)p.tiles * p.bn * p.bm;
  const float* src[J];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int mj = m + j * step;
    src[j] = p.ws + ((size_t)((n / p.bn) * p.mt + mj / p.bm) * p.bn + n % p.bn) * p.bm + mj % p.bm;
    out[j] = 0.f;
  }
  int s = 0;
  for (; s + 4 <= p.splits; s += 4) {
    float v[4][J];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < J; ++j) v[u][j] = __ldcg(src[j] + (size_t)(s + u) * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int j = 0; j < J; ++j) out[j] += v[u][j];
  }
  for (; s < p.splits; ++s) {
    float v[J];
#pragma unroll
    for (int j = 0; j < J; ++j) v[j] = __ldcg(src[j] + (size_t)s * stride);
#pragma unroll
    for (int j = 0; j < J; ++j) out[j] += v[j];
  }
}

// gates [B × 4H]: in = Gx_t (pre-activation input projection incl. bias), overwritten
// with the activated i, f, g, o; rec [B × 4H] = h_{t−1}·W_hh (or its deferred partials).
// h_lo (optional): tf32 lo of h_t for the next step's recurrent GEMM.
__global__ void lstm_cell_fwd_kernel(float* __restrict__ gates, const float* __restrict__ rec, SplitPlan rp,
                                     const float* __restrict__ c_prev, float* __restrict__ c_out,
                                     float* __restrict__ h_out, float* __restrict__ h_lo, int B, int H) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * H) return;
  const int b = idx / H, j = idx % H;
  float* g = gates + (size_t)b * 4 * H;
  float r[4];
  gemm_out<4>(rec, rp, b, j, H, 4 * H, r);
  const float gi = sigm(g[j] + r[0]);
  const float gf = sigm(g[H + j] + r[1]);
  const float gg = tanhf(g[2 * H + j] + r[2]);
  const float go = sigm(g[3 * H + j] + r[3]);
  const float cp = c_prev ? c_prev[idx] : 0.f;
  const float c = gf * cp + gi * gg;
  g[j] = gi;
  g[H + j] = gf;
  g[2 * H + j] = gg;
  g[3 * H + j] = go;
  c_out[idx] = c;
  const float h = go * tanhf(c);
  h_out[idx] = h;
  if (h_lo) h_lo[idx] = tf32_lo(h);
}

// dOut_t [B × H] (gradient w.r.t. h_t from above), dh_next [B × H] (from step t+1, or its
// deferred partials; NULL with splits = 0 at t = T−1), dc [B × H] in: dc_next (ignored when
// first), out: dc⊙f for step t−1. dG_lo (optional): tf32 lo of dG_t for the dh GEMM.
__global__ void lstm_cell_bwd_kernel(const float* __restrict__ gates, const float* __restrict__ c_t,
                                     const float* __restrict__ c_prev, const float* __restrict__ dOut,
                                     const float* __restrict__ dh_next, SplitPlan hp, float* __restrict__ dc,
                                     int first, float* __restrict__ dG, float* __restrict__ dG_lo, int B, int H) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * H) return;
  const int b = idx / H, j = idx % H;
  const float* g = gates + (size_t)b * 4 * H;
  const float gi = g[j], gf = g[H + j], gg = g[2 * H + j], go = g[3 * H + j];
  const float c = c_t[idx];
  const float cp = c_prev ? c_prev[idx] : 0.f;
  float dhn = 0.f;
  if (dh_next || hp.splits > 1) gemm_out<1>(dh_next, hp, b, j, 0, H, &dhn);
  const float dh = dOut[idx] + dhn;
  const float tc = tanhf(c);
  const float dcv = (first ? 0.f : dc[idx]) + dh * go * (1.f - tc * tc);
  float* d = dG + (size_t)b * 4 * H;
  const float d0 = dcv * gg * gi * (1.f - gi);
  const float d1 = dcv * cp * gf * (1.f - gf);
  const float d2 = dcv * gi * (1.f - gg * gg);
  const float d3 = dh * tc * go * (1.f - go);
  d[j] = d0;
  d[H + j] = d1;
  d[2 * H + j] = d2;
  d[3 * H + j] = d3;
  if (dG_lo) {
    float* l = dG_lo + (size_t)b * 4 * H;
    l[j] = tf32_lo(d0);
    l[H + j] = tf32_lo(d1);
    l[2 * H + j] = tf32_lo(d2);
    l[3 * H + j] = tf32_lo(d3);
  }
  dc[idx] = dcv * gf;
}

__global__ void embed_gather_kernel(const float* __restrict__ E, const int32_t* __restrict__ tok, int rows, int D,
                                    float* __restrict__ out) {
  const int r = blockIdx.x;
  if (r >= rows) return;
  const float* src = E + (size_t)tok[r] * D;
  float* dst = out + (size_t)r * D;
  for (int d = threadIdx.x; d < D; d += blockDim.x) dst[d] = src[d];
}

__global__ void count_kernel(const int32_t* __restrict__ tok, int rows, int* __restrict__ counts) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rows) atomicAdd(counts + tok[r], 1);
}

// exclusive scan of counts[V] → offs[V + 1] (single CTA, fixed order)
__global__ void __launch_bounds__(1024) scan_kernel(const int* __restrict__ counts, int V, int* __restrict__ offs) {
  __shared__ int part[1024];
  const int per = (V + 1023) / 1024;
  const int b0 = threadIdx.x * per;
  int s = 0;
  for (int v = b0; v < min(V, b0 + per); ++v) s += counts[v];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int i = 0; i < 1024; ++i) {
      const int t = part[i];
      part[i] = acc;
      acc += t;
    }
    offs[V] = acc;
  }
  __syncthreads();
  int acc = part[threadIdx.x];
  for (int v = b0; v < min(V, b0 + per); ++v) {
    offs[v] = acc;
    acc += counts[v];
  }
}

__global__ void fill_kernel(const int32_t* __restrict__ tok, int rows, const int* __restrict__ offs,
                            int* __restrict__ cursor, int* __restrict__ list) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rows) list[offs[tok[r]] + atomicAdd(cursor + tok[r], 1)] = r;
}

// each bucket sorted ascending (insertion sort; buckets are short except the top tokens)
__global__ void sort_buckets_kernel(const int* __restrict__ offs, int V, int* __restrict__ list) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= V) return;
  const int a = offs[v], b = offs[v + 1];
  for (int i = a + 1; i < b; ++i) {
    const int x = list[i];
    int j = i - 1;
    while (j >= a && list[j] > x) {
      list[j + 1] = list[j];
      --j;
    }
    list[j + 1] = x;
  }
}

// gE[v][d] = Σ_{rows r with tok[r] = v, ascending r} dA[r][d]   (dense: untouched rows get 0)
__global__ void embed_grad_kernel(const float* __restrict__ dA, const int* __restrict__ offs,
                                  const int* __restrict__ list, int V, int D, float* __restrict__ gE) {
  const int v = blockIdx.x;
  if (v >= V) return;
  const int a = offs[v], b = offs[v + 1];
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float s = 0.f;
    for (int i = a; i < b; ++i) s += dA[(size_t)list[i] * D + d];
    gE[(size_t)v * D + d] = s;
  }
}

}  // namespace

st_status launch_lstm_cell_fwd(float* gates, const float* rec, const SplitPlan* rp, const float* c_prev, float* c_out,
                               float* h_out, float* h_lo, int B, int H, cudaStream_t s) {
  const int n = B * H;
  const SplitPlan p = rp ? *rp : SplitPlan{};
  lstm_cell_fwd_kernel<<<(n + 255) / 256, 256, 0, s>>>(gates, rec, p, c_prev, c_out, h_out, h_lo, B, H);
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

st_status launch_lstm_cell_bwd(const float* gates, const float* c_t, const float* c_prev, const float* dOut,
                               const float* dh_next, const SplitPlan* hp, float* dc, int first, float* dG,
                               float* dG_lo, int B, int H, cudaStream_t s) {
  const int n = B * H;
  const SplitPlan p = hp ? *hp : SplitPlan{};
  lstm_cell_bwd_kernel<<<(n + 255) / 256, 256, 0, s>>>(gates, c_t, c_prev, dOut, dh_next, p, dc, first, dG, dG_lo,
                                                        B, H);
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

st_status launch_embed_gather(const float* E, const int32_t* tok, int rows, int D, float* out, cudaStream_t s) {
  embed_gather_kernel<<<rows, 256, 0, s>>>(E, tok, rows, D, out);
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int64_t embed_grad_scratch_bytes(int rows, int V) { return (int64_t)(3 * V + 1 + rows) * 4 + 256; }

// scratch: embed_grad_scratch_bytes(rows, V) bytes. Launches 6 kernels (+1 memset).
st_status launch_embed_grad(const float* dA, const int32_t* tok, int rows, int V, int D, float* gE, void* scratch,
                            cudaStream_t s) {
  int* counts = static_cast<int*>(scratch);
  int* cursor = counts + V;
  int* offs = cursor + V;
  int* list = offs + V + 1;
  ST_CUDA_TRY(cudaMemsetAsync(counts, 0, (size_t)2 * V * 4, s));
  count_kernel<<<(rows + 255) / 256, 256, 0, s>>>(tok, rows, counts);
  scan_kernel<<<1, 1024, 0, s>>>(counts, V, offs);
  fill_kernel<<<(rows + 255) / 256, 256, 0, s>>>(tok, rows, offs, cursor, list);
  sort_buckets_kernel<<<(V + 255) / 256, 256, 0, s>>>(offs, V, list);
  embed_grad_kernel<<<V, 256, 0, s>>>(dA, offs, list, V, D, gE);
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // namespace st
