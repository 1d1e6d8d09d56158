// CUDA-core fp32 GEMMs of a dense stage (ST_GEMM_SIMT: bring-up / diagnostic
// mode; the product path is the tcgen05 kernel in k_gemm_tc.cu).
//
// One generic 64×64×16 tiled kernel, C(m,n) = Σ_k A(m,k)·B(k,n) with arbitrary
// element strides, sequential fp32 FMA over k (deterministic), fused epilogues:
//   EPI_BIAS : C = acc + bias[n], optional ReLU       (forward)
//   EPI_MASK : C = acc · 1[aux(m,n) > 0]              (dX with the ReLU mask, D12)
//   EPI_PLAIN: C = acc                                (dW)
// plus the bias-gradient column sum g_b[o] = Σ_b dZ[b][o].
#include "kernels.hpp"

namespace st {
namespace {

enum { EPI_PLAIN = 0, EPI_BIAS = 1, EPI_MASK = 2 };

constexpr int TM = 64, TN = 64, TK = 16;

template <int EPI>
__global__ void __launch_bounds__(256) sgemm_kernel(int M, int N, int K, const float* __restrict__ A, int64_t a_sm,
                                                    int64_t a_sk, const float* __restrict__ Bm, int64_t b_sk,
                                                    int64_t b_sn, float* __restrict__ C, int64_t c_sm, int64_t c_sn,
                                                    const float* __restrict__ aux, int relu) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;  // 16×16 threads, 4×4 outputs each
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
    // A tile TM×TK: 1024 elements, 4 per thread. Map the contiguous dimension to tid.
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = tid + r * 256;
      int mm, kk;
      if (a_sk == 1) { kk = e % TK; mm = e / TK; } else { mm = e % TM; kk = e / TM; }
      const int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? A[gm * a_sm + gk * a_sk] : 0.f;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = tid + r * 256;
      int nn, kk;
      if (b_sn == 1) { nn = e % TN; kk = e / TN; } else { kk = e % TK; nn = e / TK; }
      const int gn = n0 + nn, gk = k0 + kk;
      Bs[kk][nn] = (gn < N && gk < K) ? Bm[gk * b_sk + gn * b_sn] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty + 16 * i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx + 16 * j;
      if (gn >= N) continue;
      float v = acc[i][j];
      if (EPI == EPI_BIAS) {
        if (aux) v += aux[gn];
        if (relu) v = fmaxf(v, 0.f);
      } else if (EPI == EPI_MASK) {
        if (aux && !(aux[gm * c_sm + gn * c_sn] > 0.f)) v = 0.f;
      }
      C[gm * c_sm + gn * c_sn] = v;
    }
  }
}

__global__ void bias_grad_kernel(const float* __restrict__ dZ, int B, int n_out, float* __restrict__ gb) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= n_out) return;
  float s = 0.f;
  for (int b = 0; b < B; ++b) s += dZ[(size_t)b * n_out + o];
  gb[o] = s;
}

template <int EPI>
st_status run(int M, int N, int K, const float* A, int64_t a_sm, int64_t a_sk, const float* Bm, int64_t b_sk,
              int64_t b_sn, float* C, int64_t c_sm, int64_t c_sn, const float* aux, int relu, cudaStream_t s) {
  dim3 grid((N + TN - 1) / TN, (M + TM - 1) / TM);
  sgemm_kernel<EPI><<<grid, 256, 0, s>>>(M, N, K, A, a_sm, a_sk, Bm, b_sk, b_sn, C, c_sm, c_sn, aux, relu);
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // namespace

// forward: Z[b][o] = Σ_i X[b][i]·W[i][o] + bias[o]
st_status simt_fwd(const GemmArgs& g, const float* X, const float* W, const float* bias, float* Z, int relu) {
  return run<EPI_BIAS>(g.B, g.n_out, g.n_in, X, g.n_in, 1, W, g.n_out, 1, Z, g.n_out, 1, bias, relu, g.stream);
}

// dX: D[b][i] = Σ_o dZ[b][o]·W[i][o], masked by mask[b][i] > 0
st_status simt_dx(const GemmArgs& g, const float* dZ, const float* W, const float* mask, float* D) {
  return run<EPI_MASK>(g.B, g.n_in, g.n_out, dZ, g.n_out, 1, W, 1, g.n_out, D, g.n_in, 1, mask, 0, g.stream);
}

// dW: G[i][o] = Σ_b X[b][i]·dZ[b][o];  gb[o] = Σ_b dZ[b][o]
st_status simt_dw(const GemmArgs& g, const float* X, const float* dZ, float* G, float* gb) {
  ST_TRY(run<EPI_PLAIN>(g.n_in, g.n_out, g.B, X, 1, g.n_in, dZ, g.n_out, 1, G, g.n_out, 1, nullptr, 0, g.stream));
  if (gb) {
    bias_grad_kernel<<<(g.n_out + 255) / 256, 256, 0, g.stream>>>(dZ, g.B, g.n_out, gb);
    ST_CUDA_TRY(cudaGetLastError());
  }
  return ST_OK;
}

st_status launch_bias_grad(const float* dZ, int B, int n_out, float* gb, cudaStream_t s) {
  bias_grad_kernel<<<(n_out + 255) / 256, 256, 0, s>>>(dZ, B, n_out, gb);
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // namespace st
