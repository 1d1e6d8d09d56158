// K-C: softmax cross-entropy forward+backward at the last stage.
//   loss = mean_b [ logsumexp(Z_b) − Z_b[y_b] ]           (D11 batch mean)
//   dZ   = (softmax(Z) − onehot(y)) / B
// One warp per row (max-subtracted softmax, max and sum in one online pass), then a
// single-CTA fixed-order sum of the per-row losses (deterministic).
#include "kernels.hpp"

namespace st {
namespace {

// (m, s) of a running max-subtracted sum: add x
__device__ __forceinline__ void online_add(float& m, float& s, float x) {
  if (x > m) {
    s = s * expf(m - x) + 1.0f;
    m = x;
  } else {
    s += expf(x - m);
  }
}
// combine two (m, s) pairs
__device__ __forceinline__ void online_merge(float& m, float& s, float m2, float s2) {
  const float mm = fmaxf(m, m2);
  s = (m == -INFINITY ? 0.f : s * expf(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * expf(m2 - mm));
  m = mm;
}

// One warp per row. Pass 1 reads the row once for the max and the max-subtracted sum
// together (online softmax: the running sum is rescaled when the max grows); pass 2 writes
// dZ. float4 loads / stores when C % 4 == 0 (rows 16-B aligned): the LM's 4480 × 10 000
// logits are 179 MB each way, so the row passes, not the arithmetic, set the time.
template <bool VEC>
__global__ void __launch_bounds__(256) ce_rows_kernel(const float* __restrict__ Z, const int32_t* __restrict__ y,
                                                      int B, int C, float inv_b, float* __restrict__ rowloss,
                                                      float* __restrict__ dZ) {
  PDL_PROLOGUE();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= B) return;
  const float* z = Z + (size_t)warp * C;
  float m = -INFINITY, s = 0.f;
  if (VEC) {
    const float4* z4 = reinterpret_cast<const float4*>(z);
    for (int c = lane; c < C / 4; c += 32) {
      const float4 v = z4[c];
      online_add(m, s, v.x);
      online_add(m, s, v.y);
      online_add(m, s, v.z);
      online_add(m, s, v.w);
    }
  } else {
    for (int c = lane; c < C; c += 32) online_add(m, s, z[c]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    online_merge(m, s, m2, s2);
  }
  const int label = y[warp];
  const float inv_s = 1.0f / s;
  float* d = dZ + (size_t)warp * C;
  if (VEC) {
    const float4* z4 = reinterpret_cast<const float4*>(z);
    float4* d4 = reinterpret_cast<float4*>(d);
    for (int c = lane; c < C / 4; c += 32) {
      const float4 v = z4[c];
      const int c0 = 4 * c;
      float4 o;
      o.x = (expf(v.x - m) * inv_s - (c0 == label ? 1.0f : 0.0f)) * inv_b;
      o.y = (expf(v.y - m) * inv_s - (c0 + 1 == label ? 1.0f : 0.0f)) * inv_b;
      o.z = (expf(v.z - m) * inv_s - (c0 + 2 == label ? 1.0f : 0.0f)) * inv_b;
      o.w = (expf(v.w - m) * inv_s - (c0 + 3 == label ? 1.0f : 0.0f)) * inv_b;
      d4[c] = o;
    }
  } else {
    for (int c = lane; c < C; c += 32) {
      const float p = expf(z[c] - m) * inv_s;
      d[c] = (p - (c == label ? 1.0f : 0.0f)) * inv_b;
    }
  }
  if (lane == 0) rowloss[warp] = (logf(s) + m) - z[label];
}

__global__ void __launch_bounds__(1024) mean_kernel(const float* __restrict__ rowloss, int B, float inv_b,
                                                    float* __restrict__ out) {
  PDL_PROLOGUE();
  // fixed-order: thread t sums rows t, t+1024, ...; then a fixed tree
  __shared__ float part[1024];
  float acc = 0.f;
  for (int i = threadIdx.x; i < B; i += 1024) acc += rowloss[i];
  part[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = part[0] * inv_b;
}

}  // namespace

st_status launch_softmax_ce(const float* Z, const int32_t* y, int B, int C, float* rowloss, float* loss_out,
                            float* dZ, cudaStream_t s) {
  if (B <= 0 || C <= 0) return set_error(ST_ERR_INPUT, "softmax_ce: B=%d C=%d", B, C);
  const float inv_b = 1.0f / (float)B;
  const int warps_per_cta = 8;
  const bool vec = (C % 4) == 0 && ((uintptr_t)Z & 15u) == 0 && ((uintptr_t)dZ & 15u) == 0;
  ST_TRY(launch_pdl(pdl_enabled(), vec ? ce_rows_kernel<true> : ce_rows_kernel<false>,
                    dim3((B + warps_per_cta - 1) / warps_per_cta), dim3(32 * warps_per_cta), 0, s, Z, y, B, C, inv_b,
                    rowloss, dZ));
  ST_TRY(launch_pdl(pdl_enabled(), mean_kernel, dim3(1), dim3(1024), 0, s, rowloss, B, inv_b, loss_out));
  return ST_OK;
}

}  // namespace st
