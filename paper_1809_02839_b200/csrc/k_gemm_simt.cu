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

enum { EPI_PLAIN = 0, EPI_BIAS = 1, EPI_MASK = 2, EPI_PARTIAL = 3 };

constexpr int TM = 64, TN = 64, TK = 16;

template <int EPI>
__global__ void __launch_bounds__(256) sgemm_kernel(int M, int N, int K, const float* __restrict__ A, int64_t a_sm,
                                                    int64_t a_sk, const float* __restrict__ Bm, int64_t b_sk,
                                                    int64_t b_sn, float* __restrict__ C, int64_t c_sm, int64_t c_sn,
                                                    const float* __restrict__ aux, int relu, int k_chunk) {
  PDL_PROLOGUE();
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;  // 16×16 threads, 4×4 outputs each
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  float acc[4][4] = {};
  // split-K: blockIdx.z owns [kb, ke); partials go to C + z·M·N (EPI_PARTIAL)
  const int kb = blockIdx.z * k_chunk;
  const int ke = min(K, kb + k_chunk);
  if (EPI == EPI_PARTIAL) C += (size_t)blockIdx.z * M * N;
  for (int k0 = kb; k0 < ke; k0 += TK) {
    // A tile TM×TK: 1024 elements, 4 per thread. Map the contiguous dimension to tid.
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = tid + r * 256;
      int mm, kk;
      if (a_sk == 1) { kk = e % TK; mm = e / TK; } else { mm = e % TM; kk = e / TM; }
      const int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < ke) ? A[gm * a_sm + gk * a_sk] : 0.f;
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = tid + r * 256;
      int nn, kk;
      if (b_sn == 1) { nn = e % TN; kk = e / TN; } else { kk = e % TK; nn = e / TK; }
      const int gn = n0 + nn, gk = k0 + kk;
      Bs[kk][nn] = (gn < N && gk < ke) ? Bm[gk * b_sk + gn * b_sn] : 0.f;
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
      if (EPI == EPI_PARTIAL)
        C[(size_t)gm * N + gn] = v;
      else
        C[gm * c_sm + gn * c_sn] = v;
    }
  }
}

// Fixed-order reduction of split-K partials + the real epilogue.
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int splits, int M, int N, float* __restrict__ C,
                                     int64_t c_sm, int64_t c_sn, int epi, const float* __restrict__ aux, int relu) {
  PDL_PROLOGUE();
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= M * N) return;
  const int m = idx / N, n = idx % N;
  float v = 0.f;
  for (int z = 0; z < splits; ++z) v += ws[(size_t)z * M * N + idx];
  if (epi == EPI_BIAS) {
    if (aux) v += aux[n];
    if (relu) v = fmaxf(v, 0.f);
  } else if (epi == EPI_MASK) {
    if (aux && !(aux[m * c_sm + n * c_sn] > 0.f)) v = 0.f;
  }
  C[m * c_sm + n * c_sn] = v;
}

// g_b[o] = Σ_b dZ[b][o]: 32 columns per CTA × 8 row groups, fixed-order combine.
__global__ void __launch_bounds__(256) bias_grad_kernel(const float* __restrict__ dZ, int B, int n_out,
                                                        float* __restrict__ gb) {
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
    float t = part[0][tx];
#pragma unroll
    for (int r = 1; r < 8; ++r) t += part[r][tx];
    gb[o] = t;
  }
}

// Tall column sums (conv layers: rows = B·H·W pixels): pass 1 gives each CTA a fixed
// contiguous row block (block rb of `rpb` rows, 8 row groups, fixed combine) and writes
// part[rb][o]; pass 2 sums the blocks in order. The partition depends only on the
// shape, so the result is deterministic.
__global__ void __launch_bounds__(256) colsum_partial_kernel(const float* __restrict__ dZ, int rows, int n_out,
                                                             int rpb, float* __restrict__ part) {
  __shared__ float sm[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int o = blockIdx.x * 32 + tx;
  const int r0 = blockIdx.y * rpb, r1 = min(rows, r0 + rpb);
  float s = 0.f;
  if (o < n_out)
    for (int r = r0 + ty; r < r1; r += 8) s += dZ[(size_t)r * n_out + o];
  sm[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && o < n_out) {
    float t = sm[0][tx];
#pragma unroll
    for (int q = 1; q < 8; ++q) t += sm[q][tx];
    part[(size_t)blockIdx.y * n_out + o] = t;
  }
}

// float4 variant (n_out % 4 == 0, 16-B aligned): 8 threads × 4 columns = 32 columns per
// CTA, 32 row groups, each thread 4 independent accumulators (rows r ≡ j mod 4 of its
// group) combined in fixed order, then the 32 groups in fixed order — deterministic, and
// 16 B × 4 loads in flight per thread instead of one 4-B load.
__global__ void __launch_bounds__(256) colsum4_partial_kernel(const float* __restrict__ dZ, int rows, int n_out,
                                                              int rpb, float* __restrict__ part) {
  __shared__ float4 sm[32][9];
  PDL_PROLOGUE();
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;
  const int o = blockIdx.x * 32 + tx * 4;
  const int r0 = blockIdx.y * rpb, r1 = min(rows, r0 + rpb);
  float4 a[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) a[j] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (o < n_out) {
    const float* base = dZ + o;
    int r = r0 + ty;
    for (; r + 96 < r1; r += 128) {
      float4 v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = __ldg(reinterpret_cast<const float4*>(base + (size_t)(r + 32 * j) * n_out));
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        a[j].x += v[j].x;
        a[j].y += v[j].y;
        a[j].z += v[j].z;
        a[j].w += v[j].w;
      }
    }
    for (int j = 0; r < r1; r += 32, ++j) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(base + (size_t)r * n_out));
      a[j & 3].x += v.x;
      a[j & 3].y += v.y;
      a[j & 3].z += v.z;
      a[j & 3].w += v.w;
    }
  }
  float4 t = a[0];
#pragma unroll
  for (int j = 1; j < 4; ++j) {
    t.x += a[j].x;
    t.y += a[j].y;
    t.z += a[j].z;
    t.w += a[j].w;
  }
  sm[ty][tx] = t;
  __syncthreads();
  if (ty == 0 && o < n_out) {
    float4 u = sm[0][tx];
    for (int q = 1; q < 32; ++q) {
      const float4 w = sm[q][tx];
      u.x += w.x;
      u.y += w.y;
      u.z += w.z;
      u.w += w.w;
    }
    *reinterpret_cast<float4*>(part + (size_t)blockIdx.y * n_out + o) = u;
  }
}

}  // namespace

// scratch: workspace whose bytes past the 64 KB counter block may be used for the
// per-block partials of tall inputs (NULL: one-pass kernel). Returns the launch count.
int launch_bias_grad(const float* dZ, int rows, int n_out, float* gb, void* work, int64_t work_bytes,
                     cudaStream_t s) {
  const int cb = (n_out + 31) / 32;
  // tall sums: enough row blocks for ~8 CTAs per SM (the LSTM / LM bias gradients: 6000 or
  // 10 000 columns over T·B = 4480 rows were one pass of 188 / 313 CTAs, ~60 µs each)
  int nb = rows > 1024 ? std::min(1024, std::max(2, (8 * device_sm_count() + cb - 1) / cb)) : 1;
  nb = std::min(nb, (rows + 255) / 256);
  if (nb > 1 && work && (int64_t)nb * n_out * 4 <= work_bytes - 64 * 1024) {
    const int rpb = (rows + nb - 1) / nb;
    nb = (rows + rpb - 1) / rpb;
    float* part = reinterpret_cast<float*>(static_cast<char*>(work) + 64 * 1024);
    // pass 2 is the same column sum over the [nb × n_out] partials as one row block
    if ((n_out & 3) == 0 && (((uintptr_t)dZ | (uintptr_t)gb) & 15) == 0) {
      if (launch_pdl(pdl_enabled(), colsum4_partial_kernel, dim3(cb, nb), dim3(256), 0, s, dZ, rows, n_out, rpb,
                     part) != ST_OK ||
          launch_pdl(pdl_enabled(), colsum4_partial_kernel, dim3(cb, 1), dim3(256), 0, s, part, nb, n_out, nb, gb) !=
              ST_OK)
        return -1;
    } else {
      colsum_partial_kernel<<<dim3(cb, nb), 256, 0, s>>>(dZ, rows, n_out, rpb, part);
      colsum_partial_kernel<<<dim3(cb, 1), 256, 0, s>>>(part, nb, n_out, nb, gb);
    }
    return cudaGetLastError() == cudaSuccess ? 2 : -1;
  }
  if (launch_pdl(pdl_enabled(), bias_grad_kernel, dim3(cb), dim3(256), 0, s, dZ, rows, n_out, gb) != ST_OK) return -1;
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

namespace {

thread_local int g_simt_launches = 0;

// Tiles that cannot fill the GPU (e.g. the 10-wide output layer: 2 tiles, K = 8192)
// are split along K into ≤ #SM/tiles chunks; partials (workspace, after the 64 KB
// counter block) are reduced in fixed order by a second kernel — deterministic.
template <int EPI>
st_status run(int M, int N, int K, const float* A, int64_t a_sm, int64_t a_sk, const float* Bm, int64_t b_sk,
              int64_t b_sn, float* C, int64_t c_sm, int64_t c_sn, const float* aux, int relu, cudaStream_t s,
              void* work, int64_t work_bytes) {
  const int tiles = ((N + TN - 1) / TN) * ((M + TM - 1) / TM);
  int splits = 1;
  if (work && tiles < 74 && K >= 8 * TK) splits = std::min(device_sm_count() / tiles, K / (4 * TK));
  const int64_t need = (int64_t)splits * M * N * 4;
  while (splits > 1 && need > work_bytes - 64 * 1024) --splits;
  dim3 grid((N + TN - 1) / TN, (M + TM - 1) / TM, std::max(1, splits));
  if (splits <= 1) {
    ST_TRY(launch_pdl(pdl_enabled(), sgemm_kernel<EPI>, grid, dim3(256), 0, s, M, N, K, A, a_sm, a_sk, Bm, b_sk, b_sn,
                      C, c_sm, c_sn, aux, relu, K));
    g_simt_launches = 1;
    return ST_OK;
  }
  const int chunk = ((K + splits - 1) / splits + TK - 1) / TK * TK;
  splits = (K + chunk - 1) / chunk;
  grid.z = splits;
  float* ws = reinterpret_cast<float*>(static_cast<char*>(work) + 64 * 1024);
  ST_TRY(launch_pdl(pdl_enabled(), sgemm_kernel<EPI_PARTIAL>, grid, dim3(256), 0, s, M, N, K, A, a_sm, a_sk, Bm, b_sk,
                    b_sn, ws, c_sm, c_sn, (const float*)nullptr, 0, chunk));
  ST_TRY(launch_pdl(pdl_enabled(), splitk_reduce_kernel, dim3((M * N + 255) / 256), dim3(256), 0, s, ws, splits, M, N,
                    C, c_sm, c_sn, EPI, aux, relu));
  g_simt_launches = 2;
  return ST_OK;
}

}  // namespace

// forward: Z[b][o] = Σ_i X[b][i]·W[i][o] + bias[o]
st_status simt_fwd(const GemmArgs& g, const float* X, const float* W, const float* bias, float* Z, int relu) {
  return run<EPI_BIAS>(g.B, g.n_out, g.n_in, X, g.n_in, 1, W, g.n_out, 1, Z, g.n_out, 1, bias, relu, g.stream, g.work,
                       g.work_bytes);
}

// dX: D[b][i] = Σ_o dZ[b][o]·W[i][o], masked by mask[b][i] > 0
st_status simt_dx(const GemmArgs& g, const float* dZ, const float* W, const float* mask, float* D) {
  return run<EPI_MASK>(g.B, g.n_in, g.n_out, dZ, g.n_out, 1, W, 1, g.n_out, D, g.n_in, 1, mask, 0, g.stream, g.work,
                       g.work_bytes);
}

// dW: G[i][o] = Σ_b X[b][i]·dZ[b][o];  gb[o] = Σ_b dZ[b][o]
st_status simt_dw(const GemmArgs& g, const float* X, const float* dZ, float* G, float* gb) {
  ST_TRY(run<EPI_PLAIN>(g.n_in, g.n_out, g.B, X, 1, g.n_in, dZ, g.n_out, 1, G, g.n_out, 1, nullptr, 0, g.stream,
                        g.work, g.work_bytes));
  if (gb) {
    const int l = g_simt_launches;
    const int n = launch_bias_grad(dZ, g.B, g.n_out, gb, g.work, g.work_bytes, g.stream);
    if (n < 0) return set_error(ST_ERR_CUDA, "bias gradient launch failed");
    g_simt_launches = l + n;
  }
  return ST_OK;
}

int simt_last_launches() { return g_simt_launches; }

}  // namespace st
