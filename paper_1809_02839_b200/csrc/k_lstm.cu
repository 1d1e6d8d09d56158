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
  // programmatic dependent launch: the next recurrent GEMM may launch now; this kernel's
  // inputs (the previous GEMM's partials) are complete only after the wait
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
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
  // programmatic dependent launch: the next recurrent GEMM may launch now; this kernel's
  // inputs (the previous GEMM's partials) are complete only after the wait
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
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

// float4 variants (H % 4 == 0, 16-B aligned buffers): each thread owns 4 consecutive
// units j..j+3 of one row b — the same arithmetic per element, 4× the bytes per load
// instruction (the cells are latency-bound: ~1.4 TB/s with one float per load).
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float& at(float4& v, int i) { return reinterpret_cast<float*>(&v)[i]; }

// out[g] (g < G) = the GEMM output at (row n, columns m + g·step .. +3), direct or the
// fixed-order sum of the deferred split partials (4 consecutive columns stay inside one
// bm-wide tile because m and step are multiples of 4 and bm % 4 == 0)
template <int G>
__device__ __forceinline__ void gemm_out4(const float* direct, const SplitPlan& p, int n, int m, int step, int ld,
                                          float4* out) {
  if (p.splits <= 1) {
#pragma unroll
    for (int g = 0; g < G; ++g) out[g] = ld4(direct + (size_t)n * ld + m + g * step);
    return;
  }
  const size_t stride = (size_t)p.tiles * p.bn * p.bm;
  const float* src[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int mg = m + g * step;
    src[g] = p.ws + ((size_t)((n / p.bn) * p.mt + mg / p.bm) * p.bn + n % p.bn) * p.bm + mg % p.bm;
    out[g] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  int s = 0;
  for (; s + 2 <= p.splits; s += 2) {
    float4 v[2][G];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int g = 0; g < G; ++g) v[u][g] = __ldcg(reinterpret_cast<const float4*>(src[g] + (size_t)(s + u) * stride));
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int g = 0; g < G; ++g) {
        out[g].x += v[u][g].x;
        out[g].y += v[u][g].y;
        out[g].z += v[u][g].z;
        out[g].w += v[u][g].w;
      }
  }
  for (; s < p.splits; ++s) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(src[g] + (size_t)s * stride));
      out[g].x += v.x;
      out[g].y += v.y;
      out[g].z += v.z;
      out[g].w += v.w;
    }
  }
}

__global__ void lstm_cell_fwd4_kernel(float* __restrict__ gates, const float* __restrict__ rec, SplitPlan rp,
                                      const float* __restrict__ c_prev, float* __restrict__ c_out,
                                      float* __restrict__ h_out, float* __restrict__ h_lo, int B, int H) {
  // programmatic dependent launch: the next recurrent GEMM may launch now; this kernel's
  // inputs (the previous GEMM's partials) are complete only after the wait
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int H4 = H / 4;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * H4) return;
  const int b = idx / H4, j = (idx % H4) * 4;
  float* g = gates + (size_t)b * 4 * H;
  float4 r[4], x[4];
  gemm_out4<4>(rec, rp, b, j, H, 4 * H, r);
#pragma unroll
  for (int q = 0; q < 4; ++q) x[q] = ld4(g + q * H + j);
  const float4 cp = c_prev ? ld4(c_prev + (size_t)b * H + j) : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 oi, of, og, oo, oc, oh, ol;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float gi = sigm(at(x[0], e) + at(r[0], e));
    const float gf = sigm(at(x[1], e) + at(r[1], e));
    const float gg = tanhf(at(x[2], e) + at(r[2], e));
    const float go = sigm(at(x[3], e) + at(r[3], e));
    const float c = gf * reinterpret_cast<const float*>(&cp)[e] + gi * gg;
    const float h = go * tanhf(c);
    at(oi, e) = gi;
    at(of, e) = gf;
    at(og, e) = gg;
    at(oo, e) = go;
    at(oc, e) = c;
    at(oh, e) = h;
    at(ol, e) = tf32_lo(h);
  }
  st4(g + j, oi);
  st4(g + H + j, of);
  st4(g + 2 * H + j, og);
  st4(g + 3 * H + j, oo);
  st4(c_out + (size_t)b * H + j, oc);
  st4(h_out + (size_t)b * H + j, oh);
  if (h_lo) st4(h_lo + (size_t)b * H + j, ol);
}

__global__ void lstm_cell_bwd4_kernel(const float* __restrict__ gates, const float* __restrict__ c_t,
                                      const float* __restrict__ c_prev, const float* __restrict__ dOut,
                                      const float* __restrict__ dh_next, SplitPlan hp, float* __restrict__ dc,
                                      int first, float* __restrict__ dG, float* __restrict__ dG_lo, int B, int H) {
  // programmatic dependent launch: the next recurrent GEMM may launch now; this kernel's
  // inputs (the previous GEMM's partials) are complete only after the wait
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int H4 = H / 4;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * H4) return;
  const int b = idx / H4, j = (idx % H4) * 4;
  const size_t o = (size_t)b * H + j;
  const float* g = gates + (size_t)b * 4 * H;
  float4 gv[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) gv[q] = ld4(g + q * H + j);
  float4 dhn = make_float4(0.f, 0.f, 0.f, 0.f);
  if (dh_next || hp.splits > 1) gemm_out4<1>(dh_next, hp, b, j, 0, H, &dhn);
  float4 cv = ld4(c_t + o), cp = c_prev ? ld4(c_prev + o) : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 dov = ld4(dOut + o), dcv4 = first ? make_float4(0.f, 0.f, 0.f, 0.f) : ld4(dc + o);
  float4 d0, d1, d2, d3, dcn;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float gi = at(gv[0], e), gf = at(gv[1], e), gg = at(gv[2], e), go = at(gv[3], e);
    const float dh = at(dov, e) + at(dhn, e);
    const float tc = tanhf(at(cv, e));
    const float dcx = at(dcv4, e) + dh * go * (1.f - tc * tc);
    at(d0, e) = dcx * gg * gi * (1.f - gi);
    at(d1, e) = dcx * at(cp, e) * gf * (1.f - gf);
    at(d2, e) = dcx * gi * (1.f - gg * gg);
    at(d3, e) = dh * tc * go * (1.f - go);
    at(dcn, e) = dcx * gf;
  }
  float* d = dG + (size_t)b * 4 * H;
  st4(d + j, d0);
  st4(d + H + j, d1);
  st4(d + 2 * H + j, d2);
  st4(d + 3 * H + j, d3);
  if (dG_lo) {
    float* l = dG_lo + (size_t)b * 4 * H;
    st4(l + j, make_float4(tf32_lo(d0.x), tf32_lo(d0.y), tf32_lo(d0.z), tf32_lo(d0.w)));
    st4(l + H + j, make_float4(tf32_lo(d1.x), tf32_lo(d1.y), tf32_lo(d1.z), tf32_lo(d1.w)));
    st4(l + 2 * H + j, make_float4(tf32_lo(d2.x), tf32_lo(d2.y), tf32_lo(d2.z), tf32_lo(d2.w)));
    st4(l + 3 * H + j, make_float4(tf32_lo(d3.x), tf32_lo(d3.y), tf32_lo(d3.z), tf32_lo(d3.w)));
  }
  st4(dc + o, dcn);
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

// 256-thread launch of a cell kernel as a programmatic dependent of the preceding kernel
static cudaLaunchConfig_t pdl_config(int blocks, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  return cfg;
}
static void pdl_attr(cudaLaunchConfig_t& cfg, cudaLaunchAttribute* at) {
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
}

st_status launch_lstm_cell_fwd(float* gates, const float* rec, const SplitPlan* rp, const float* c_prev, float* c_out,
                               float* h_out, float* h_lo, int B, int H, cudaStream_t s) {
  const int n = B * H;
  const SplitPlan p = rp ? *rp : SplitPlan{};
  const bool v4 = H % 4 == 0 && ((uintptr_t)gates | (uintptr_t)rec | (uintptr_t)c_prev | (uintptr_t)c_out |
                                 (uintptr_t)h_out | (uintptr_t)h_lo | (uintptr_t)p.ws) % 16 == 0;
  cudaLaunchConfig_t cfg = pdl_config(v4 ? (n / 4 + 255) / 256 : (n + 255) / 256, s);
  cudaLaunchAttribute at[1];
  pdl_attr(cfg, at);
  if (v4)
    ST_CUDA_TRY(cudaLaunchKernelEx(&cfg, lstm_cell_fwd4_kernel, gates, rec, p, c_prev, c_out, h_out, h_lo, B, H));
  else
    ST_CUDA_TRY(cudaLaunchKernelEx(&cfg, lstm_cell_fwd_kernel, gates, rec, p, c_prev, c_out, h_out, h_lo, B, H));
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

st_status launch_lstm_cell_bwd(const float* gates, const float* c_t, const float* c_prev, const float* dOut,
                               const float* dh_next, const SplitPlan* hp, float* dc, int first, float* dG,
                               float* dG_lo, int B, int H, cudaStream_t s) {
  const int n = B * H;
  const SplitPlan p = hp ? *hp : SplitPlan{};
  const bool v4 = H % 4 == 0 && ((uintptr_t)gates | (uintptr_t)c_t | (uintptr_t)c_prev | (uintptr_t)dOut |
                                 (uintptr_t)dh_next | (uintptr_t)dc | (uintptr_t)dG | (uintptr_t)dG_lo |
                                 (uintptr_t)p.ws) % 16 == 0;
  cudaLaunchConfig_t cfg = pdl_config(v4 ? (n / 4 + 255) / 256 : (n + 255) / 256, s);
  cudaLaunchAttribute at[1];
  pdl_attr(cfg, at);
  if (v4)
    ST_CUDA_TRY(cudaLaunchKernelEx(&cfg, lstm_cell_bwd4_kernel, gates, c_t, c_prev, dOut, dh_next, p, dc, first, dG,
                                   dG_lo, B, H));
  else
    ST_CUDA_TRY(cudaLaunchKernelEx(&cfg, lstm_cell_bwd_kernel, gates, c_t, c_prev, dOut, dh_next, p, dc, first, dG,
                                   dG_lo, B, H));
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
