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
                                                                  size_t n4, UpdateConsts c, float* __restrict__ Wt,
                                                                  float* __restrict__ Vt, const float* __restrict__ Gt,
                                                                  float* __restrict__ WFt, float* __restrict__ WBt,
                                                                  int tail) {
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
  // scalar tail (n % 4 elements) — one block handles it
  if (blockIdx.x == 0 && threadIdx.x < tail) {
    const int t = threadIdx.x;
    float w = Wt[t], v = Vt[t], wf = 0.f, wb = 0.f;
    upd1<kWF, kWB>(w, v, Gt[t], wf, wb, c);
    Wt[t] = w;
    Vt[t] = v;
    if (kWF) WFt[t] = wf;
    if (kWB) WBt[t] = wb;
  }
}

int grid_for(size_t n4) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
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
  const size_t n4 = n / 4;
  const int tail = (int)(n % 4);
  const size_t t0 = n4 * 4;
  float* WFt = WF ? WF + t0 : nullptr;
  float* WBt = WB ? WB + t0 : nullptr;
  const int grid = grid_for(n4 ? n4 : 1);
  auto W4 = reinterpret_cast<float4*>(W);
  auto V4 = reinterpret_cast<float4*>(V);
  auto G4 = reinterpret_cast<const float4*>(G);
  auto F4 = reinterpret_cast<float4*>(WF);
  auto B4 = reinterpret_cast<float4*>(WB);
  if (WF && WB)
    update_predict_kernel<true, true><<<grid, kThreads, 0, s>>>(W4, V4, G4, F4, B4, n4, c, W + t0, V + t0, G + t0,
                                                                WFt, WBt, tail);
  else if (WF)
    update_predict_kernel<true, false><<<grid, kThreads, 0, s>>>(W4, V4, G4, F4, B4, n4, c, W + t0, V + t0,
                                                                 G + t0, WFt, WBt, tail);
  else if (WB)
    update_predict_kernel<false, true><<<grid, kThreads, 0, s>>>(W4, V4, G4, F4, B4, n4, c, W + t0, V + t0,
                                                                 G + t0, WFt, WBt, tail);
  else
    update_predict_kernel<false, false><<<grid, kThreads, 0, s>>>(W4, V4, G4, F4, B4, n4, c, W + t0, V + t0,
                                                                  G + t0, WFt, WBt, tail);
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // namespace st
