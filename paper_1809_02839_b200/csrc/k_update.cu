// K-B: the fused SpecTrain update kernel.
//
// One HBM stream over the stage arena, per parameter:
//   v' = γ·v + (1−γ)·g            Eq. 1     [heavy-ball: γ·v + g, D2]
//   w' = w − η·v'                 Momentum-SGD apply (D1)
//   WF = w' − s_F·η·v'            Eq. 4 with s_F of Eq. 5, if s_F > 0
//   WB = w' − s_B·η·v'            Eq. 4 with s_B of Eq. 6, if s_B > 0 and s_B ≠ s_F
// i.e. the update of this backward fused with the predictions the NEXT forward
// and backward of this stage will use (no update intervenes between them in
// 1F1B). Algorithmic traffic: reads G, W, V (12 B) + writes W,
// V (8 B) [+ WF 4 B] [+ WB 4 B] = 20 / 24 / 28 B per parameter.
//
// Arithmetic is pinned to explicit round-to-nearest intrinsics so the compiler
// cannot re-associate: v' = fma(γ, v, (1−γ)·g), w' = fma(−η, v', w),
// wf = fma(−s_F·η, v', w').
#include "kernels.hpp"

namespace st {

UpdateConsts make_update_consts(float lr, float gamma, int sF, int sB, int momentum) {
  UpdateConsts c;
  c.c_gamma = gamma;
  c.c_one = (momentum == ST_MOMENTUM_HEAVY_BALL) ? 1.0f : (float)(1.0 - (double)gamma);
  c.c_eta = lr;
  c.c_f = (float)((double)sF * (double)lr);
  c.c_b = (float)((double)sB * (double)lr);
  return c;
}

namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 2;  // float4 per array per thread per iteration

__device__ __forceinline__ float4 ld_stream(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(float4* p, const float4& v) { __stcs(p, v); }

template <bool kWF, bool kWB>
__device__ __forceinline__ void upd1(float& w, float& v, float g, float& wf, float& wb, const UpdateConsts& c) {
  const float vn = __fmaf_rn(c.c_gamma, v, __fmul_rn(c.c_one, g));
  const float wn = __fmaf_rn(-c.c_eta, vn, w);
  if (kWF) wf = __fmaf_rn(-c.c_f, vn, wn);
  if (kWB) wb = __fmaf_rn(-c.c_b, vn, wn);
  v = vn;
  w = wn;
}

template <bool kWF, bool kWB>
__global__ void __launch_bounds__(kThreads) update_predict_kernel(float4* __restrict__ W, float4* __restrict__ V,
                                                                  const float4* __restrict__ G,
                                                                  float4* __restrict__ WF, float4* __restrict__ WB,
                                                                  size_t n4, UpdateConsts c, float* __restrict__ Ws,
                                                                  float* __restrict__ Vs, const float* __restrict__ Gs,
                                                                  float* __restrict__ WFs, float* __restrict__ WBs,
                                                                  int head, size_t tail0, int tail) {
  PDL_PROLOGUE();
  const size_t stride = (size_t)gridDim.x * kThreads * kUnroll;
  for (size_t base = (size_t)blockIdx.x * kThreads * kUnroll + threadIdx.x; base < n4; base += stride) {
    float4 w[kUnroll], v[kUnroll], g[kUnroll], wf[kUnroll], wb[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const size_t i = base + (size_t)u * kThreads;
      if (i < n4) {
        g[u] = ld_stream(G + i);
        w[u] = ld_stream(W + i);
        v[u] = ld_stream(V + i);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const size_t i = base + (size_t)u * kThreads;
      if (i < n4) {
        upd1<kWF, kWB>(w[u].x, v[u].x, g[u].x, wf[u].x, wb[u].x, c);
        upd1<kWF, kWB>(w[u].y, v[u].y, g[u].y, wf[u].y, wb[u].y, c);
        upd1<kWF, kWB>(w[u].z, v[u].z, g[u].z, wf[u].z, wb[u].z, c);
        upd1<kWF, kWB>(w[u].w, v[u].w, g[u].w, wf[u].w, wb[u].w, c);
        st_stream(W + i, w[u]);
        st_stream(V + i, v[u]);
        if (kWF) WF[i] = wf[u];
        if (kWB) WB[i] = wb[u];
      }
    }
  }
  // scalar head (to reach 16-byte alignment) and tail (n % 4) elements — block 0
  if (blockIdx.x == 0 && (int)threadIdx.x < head + tail) {
    const size_t t = (int)threadIdx.x < head ? (size_t)threadIdx.x : tail0 + (threadIdx.x - head);
    float w = Ws[t], v = Vs[t], wf = 0.f, wb = 0.f;
    upd1<kWF, kWB>(w, v, Gs[t], wf, wb, c);
    Ws[t] = w;
    Vs[t] = v;
    if (kWF) WFs[t] = wf;
    if (kWB) WBs[t] = wb;
  }
}

int grid_for(size_t n4) {
  const int sms = device_sm_count();
  // persistent grid-stride: up to 8 resident 256-thread CTAs per SM
  const size_t per_cta = (size_t)kThreads * kUnroll;
  size_t want = (n4 + per_cta - 1) / per_cta;
  size_t cap = (size_t)sms * 8;
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  return (int)want;
}

}  // namespace

st_status launch_update_predict(float* W, float* V, const float* G, float* WF, float* WB, size_t n,
                                const UpdateConsts& c, cudaStream_t s) {
  if (n == 0) return ST_OK;
  // W, V, G, WF, WB share their alignment (same offset into 256-byte aligned arenas, or
  // 16-byte aligned raw buffers): peel up to 3 scalar elements to reach float4 alignment.
  int head = (int)(((16 - ((uintptr_t)W & 15)) & 15) / 4);
  if ((size_t)head > n) head = (int)n;
  const size_t n4 = (n - head) / 4;
  const int tail = (int)((n - head) % 4);
  const size_t tail0 = head + n4 * 4;
  const int grid = grid_for(n4 ? n4 : 1);
  auto W4 = reinterpret_cast<float4*>(W + head);
  auto V4 = reinterpret_cast<float4*>(V + head);
  auto G4 = reinterpret_cast<const float4*>(G + head);
  auto F4 = WF ? reinterpret_cast<float4*>(WF + head) : nullptr;
  auto B4 = WB ? reinterpret_cast<float4*>(WB + head) : nullptr;
  st_status st = ST_OK;
  if (WF && WB)
    st = launch_pdl(pdl_enabled(), update_predict_kernel<true, true>, dim3(grid), dim3(kThreads), 0, s, W4, V4, G4, F4, B4, n4, c, W, V, G, WF, WB, head,
                                                                tail0, tail);
  else if (WF)
    st = launch_pdl(pdl_enabled(), update_predict_kernel<true, false>, dim3(grid), dim3(kThreads), 0, s, W4, V4, G4, F4, B4, n4, c, W, V, G, WF, WB, head,
                                                                 tail0, tail);
  else if (WB)
    st = launch_pdl(pdl_enabled(), update_predict_kernel<false, true>, dim3(grid), dim3(kThreads), 0, s, W4, V4, G4, F4, B4, n4, c, W, V, G, WF, WB, head,
                                                                 tail0, tail);
  else
    st = launch_pdl(pdl_enabled(), update_predict_kernel<false, false>, dim3(grid), dim3(kThreads), 0, s, W4, V4, G4, F4, B4, n4, c, W, V, G, WF, WB, head,
                                                                  tail0, tail);
  ST_TRY(st);
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

namespace {
// g_b[o] = Σ_b dZ[b][o] (fixed order: 8 row groups, then a fixed combine), then
// the same K-B arithmetic as update_predict_kernel on the bias entries.
__global__ void __launch_bounds__(256) bias_grad_update_kernel(const float* __restrict__ dZ, int B, int n_out,
                                                               UpdateArgs u) {
  PDL_PROLOGUE();
  __shared__ float part[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int o = blockIdx.x * 32 + tx;
  float s = 0.f;
  if (o < n_out)
    for (int b = ty; b < B; b += 8) s += dZ[(size_t)b * n_out + o];
  part[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && o < n_out) {
    float g = part[0][tx];
#pragma unroll
    for (int r = 1; r < 8; ++r) g += part[r][tx];
    float w = u.W[o], v = u.V[o], wf = 0.f, wb = 0.f;
    const float vn = __fmaf_rn(u.c.c_gamma, v, __fmul_rn(u.c.c_one, g));
    const float wn = __fmaf_rn(-u.c.c_eta, vn, w);
    if (u.WF) wf = __fmaf_rn(-u.c.c_f, vn, wn);
    if (u.WB) wb = __fmaf_rn(-u.c.c_b, vn, wn);
    u.W[o] = wn;
    u.V[o] = vn;
    if (u.WF) u.WF[o] = wf;
    if (u.WB) u.WB[o] = wb;
  }
}
}  // namespace

st_status launch_bias_grad_update(const float* dZ, int B, int n_out, const UpdateArgs& u, cudaStream_t s) {
  ST_TRY(launch_pdl(pdl_enabled(), bias_grad_update_kernel, dim3((n_out + 31) / 32), dim3(256), 0, s, dZ, B, n_out,
                    u));
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // namespace st

// ---- Fig. 7 prediction accuracy -----------------------
// e_pred = W_old − s·η·V_old − W_now (Eq. 4 prediction vs the actual weights s updates
// later), e_stale = W_old − W_now; Σ e² of both in fp64. Pass 1: CTA b sums a fixed
// contiguous chunk (per-thread strided sums, then a fixed smem tree); pass 2: one thread
// adds the CTA partials in order — deterministic for a given n.
namespace st {
namespace {

constexpr int kErrBlocks = 592;

__global__ void __launch_bounds__(256) pred_err_partial_kernel(const float* __restrict__ Wo,
                                                               const float* __restrict__ Vo,
                                                               const float* __restrict__ Wn, size_t n, double c,
                                                               double* __restrict__ part) {
  __shared__ double sp[256], ss[256];
  const size_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const size_t i0 = (size_t)blockIdx.x * chunk, i1 = min(n, i0 + chunk);
  double ap = 0.0, as = 0.0;
  for (size_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const double wo = Wo[i], wn = Wn[i];
    const double ep = (wo - c * (double)Vo[i]) - wn, es = wo - wn;
    ap += ep * ep;
    as += es * es;
  }
  sp[threadIdx.x] = ap;
  ss[threadIdx.x] = as;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (threadIdx.x < h) {
      sp[threadIdx.x] += sp[threadIdx.x + h];
      ss[threadIdx.x] += ss[threadIdx.x + h];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = sp[0];
    part[2 * blockIdx.x + 1] = ss[0];
  }
}

__global__ void pred_err_final_kernel(const double* __restrict__ part, int nb, double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double p = 0.0, q = 0.0;
  for (int b = 0; b < nb; ++b) {
    p += part[2 * b];
    q += part[2 * b + 1];
  }
  out[0] = p;
  out[1] = q;
}

// Hybrid DP × PP (NEXT-4): in-place sum of the gradient arenas of a stage's R
// co-located replicas over elements [begin, end): every arena receives Σ_j G_j, summed
// in the fixed order j = 0..R−1 (all replicas end bit-identical). Each replica reduces
// its own slice of the arenas, so the R launches touch disjoint memory.
constexpr int kMaxReplicas = 16;
struct GPtrs {
  float* g[kMaxReplicas];
};

__global__ void replica_sum_kernel(GPtrs p, int R, size_t begin, size_t end) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = begin + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < end; i += stride) {
    float acc = p.g[0][i];
    for (int j = 1; j < R; ++j) acc = __fadd_rn(acc, p.g[j][i]);
    for (int j = 0; j < R; ++j) p.g[j][i] = acc;
  }
}

}  // namespace

st_status launch_replica_sum(float* const* Gs, int R, size_t begin, size_t end, cudaStream_t s) {
  if (R < 1 || R > kMaxReplicas) return set_error(ST_ERR_INPUT, "replica sum: %d replicas (max %d)", R, kMaxReplicas);
  if (end <= begin) return ST_OK;
  GPtrs p{};
  for (int j = 0; j < R; ++j) p.g[j] = Gs[j];
  const size_t n = end - begin;
  const int grid = (int)std::min<size_t>((size_t)device_sm_count() * 8, (n + 255) / 256);
  replica_sum_kernel<<<std::max(1, grid), 256, 0, s>>>(p, R, begin, end);
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

int64_t prediction_error_work_bytes() { return (int64_t)(2 * kErrBlocks + 2) * 8; }

st_status launch_prediction_error(const float* W_old, const float* V_old, const float* W_now, size_t n, double s_eta,
                                  double* work, cudaStream_t s) {
  const int nb = (int)std::min<size_t>(kErrBlocks, std::max<size_t>(1, (n + 255) / 256));
  pred_err_partial_kernel<<<nb, 256, 0, s>>>(W_old, V_old, W_now, n, s_eta, work);
  pred_err_final_kernel<<<1, 32, 0, s>>>(work, nb, work + 2 * kErrBlocks);
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // namespace st
