// K-F: the non-GEMM parts of the VGG conv stages, NHWC.
//   conv 3×3, stride 1, pad 1 as an explicit-im2col GEMM: col[P × 9·C] with
//   P = B·H·W pixel rows and columns ordered (kh, kw, c) — the row order of the
//   HWIO weight block — so Y = col·W + b runs on the tcgen05 GEMMs; backward:
//   dW = colᵀ·dY, dcol = dY·Wᵀ, dX = col2im(dcol) (a gather: deterministic) ⊙ mask.
//   2×2 max-pool: the routed input is the first maximum in row-major window order
//   (reading D21); backward recomputes it from the stashed input.
#include "kernels.hpp"

namespace st {
namespace {

// Index math in IDX (int32 when the element count allows it — 64-bit division is
// ~5× slower); channels move as float4 when C % 4 == 0 (VEC = 4), else one by one.
template <typename IDX, int VEC>
__global__ void im2col_kernel(const float* __restrict__ X, int B, int H, int W, int C, float* __restrict__ col) {
  const int CV = C / VEC;
  const IDX total = (IDX)B * H * W * 9 * CV;
  for (IDX i = blockIdx.x * (IDX)blockDim.x + threadIdx.x; i < total; i += (IDX)gridDim.x * blockDim.x) {
    const int cv = (int)(i % CV);
    const IDX t = i / CV;
    const int q = (int)(t % 9);  // kh·3 + kw
    const IDX p = t / 9;         // pixel row b·H·W + h·W + w
    const int w = (int)(p % W);
    const IDX ph = p / W;
    const int h = (int)(ph % H);
    const IDX b = ph / H;
    const int hh = h + q / 3 - 1, ww = w + q % 3 - 1;
    const bool in = hh >= 0 && hh < H && ww >= 0 && ww < W;
    if (VEC == 4) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (in) v = __ldg(reinterpret_cast<const float4*>(X + (((int64_t)b * H + hh) * W + ww) * C) + cv);
      __stcs(reinterpret_cast<float4*>(col) + i, v);
    } else {
      col[i] = in ? __ldg(X + (((int64_t)b * H + hh) * W + ww) * C + cv) : 0.f;
    }
  }
}

// dX[b,h,w,c] = Σ_{kh,kw} dcol[(b, h+1−kh, w+1−kw), (kh, kw, c)] (valid positions),
// then ⊙ 1[mask > 0] if mask (the ReLU of the layer that produced X).
template <typename IDX, int VEC>
__global__ void col2im_kernel(const float* __restrict__ dcol, int B, int H, int W, int C, const float* __restrict__ mask,
                              float* __restrict__ dX) {
  const int CV = C / VEC;
  const IDX total = (IDX)B * H * W * CV;
  for (IDX i = blockIdx.x * (IDX)blockDim.x + threadIdx.x; i < total; i += (IDX)gridDim.x * blockDim.x) {
    const int cv = (int)(i % CV);
    const IDX p = i / CV;
    const int w = (int)(p % W);
    const IDX ph = p / W;
    const int h = (int)(ph % H);
    const IDX b = ph / H;
    if (VEC == 4) {
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const int hh = h + 1 - q / 3, ww = w + 1 - q % 3;
        if (hh >= 0 && hh < H && ww >= 0 && ww < W) {
          const float4 d = __ldg(reinterpret_cast<const float4*>(dcol + ((((int64_t)b * H + hh) * W + ww) * 9 + q) * C) + cv);
          s.x += d.x;
          s.y += d.y;
          s.z += d.z;
          s.w += d.w;
        }
      }
      if (mask) {
        const float4 m = __ldg(reinterpret_cast<const float4*>(mask) + i);
        if (!(m.x > 0.f)) s.x = 0.f;
        if (!(m.y > 0.f)) s.y = 0.f;
        if (!(m.z > 0.f)) s.z = 0.f;
        if (!(m.w > 0.f)) s.w = 0.f;
      }
      reinterpret_cast<float4*>(dX)[i] = s;
    } else {
      float s = 0.f;
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const int hh = h + 1 - q / 3, ww = w + 1 - q % 3;
        if (hh >= 0 && hh < H && ww >= 0 && ww < W)
          s += __ldg(dcol + ((((int64_t)b * H + hh) * W + ww) * 9 + q) * C + cv);
      }
      if (mask && !(mask[i] > 0.f)) s = 0.f;
      dX[i] = s;
    }
  }
}

// col[p][0..31]: the 9·C (≤ 32) window values of pixel p in (kh, kw, c) order, zeros
// after them; one thread per pixel, eight float4 stores (C a template: static indices).
template <int C>
__global__ void im2col_pad32_kernel(const float* __restrict__ X, int B, int H, int W, float* __restrict__ col) {
  PDL_PROLOGUE();
  const int total = B * H * W;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < total; p += gridDim.x * blockDim.x) {
    const int w = p % W, h = (p / W) % H, b = p / (W * H);
    float v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = 0.f;
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      const int hh = h + q / 3 - 1, ww = w + q % 3 - 1;
      if (hh >= 0 && hh < H && ww >= 0 && ww < W) {
        const float* x = X + (((int64_t)b * H + hh) * W + ww) * C;
#pragma unroll
        for (int c = 0; c < C; ++c) v[q * C + c] = __ldg(x + c);
      }
    }
    float4* dst = reinterpret_cast<float4*>(col + (int64_t)p * 32);
#pragma unroll
    for (int k = 0; k < 8; ++k) dst[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
  }
}

template <typename IDX>
__global__ void maxpool_fwd_kernel(const float* __restrict__ X, int B, int H, int W, int C, float* __restrict__ Y) {
  PDL_PROLOGUE();
  const int Ho = H / 2, Wo = W / 2;
  const IDX total = (IDX)B * Ho * Wo * C;
  for (IDX i = blockIdx.x * (IDX)blockDim.x + threadIdx.x; i < total; i += (IDX)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const IDX p = i / C;
    const int wo = (int)(p % Wo);
    const IDX ph = p / Wo;
    const int ho = (int)(ph % Ho);
    const IDX b = ph / Ho;
    const float* x = X + (((int64_t)b * H + 2 * ho) * W + 2 * wo) * C + c;
    float m = x[0];
    m = fmaxf(m, x[C]);
    m = fmaxf(m, x[(int64_t)W * C]);
    m = fmaxf(m, x[(int64_t)W * C + C]);
    Y[i] = m;
  }
}

template <typename IDX>
__global__ void maxpool_bwd_kernel(const float* __restrict__ X, const float* __restrict__ dY, int B, int H, int W,
                                   int C, int relu_mask, float* __restrict__ dX) {
  PDL_PROLOGUE();
  const int Ho = H / 2, Wo = W / 2;
  const IDX total = (IDX)B * Ho * Wo * C;
  for (IDX i = blockIdx.x * (IDX)blockDim.x + threadIdx.x; i < total; i += (IDX)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const IDX p = i / C;
    const int wo = (int)(p % Wo);
    const IDX ph = p / Wo;
    const int ho = (int)(ph % Ho);
    const IDX b = ph / Ho;
    const int64_t base = (((int64_t)b * H + 2 * ho) * W + 2 * wo) * C + c;
    const int64_t off[4] = {0, C, (int64_t)W * C, (int64_t)W * C + C};
    int arg = 0;
    float m = X[base];
#pragma unroll
    for (int q = 1; q < 4; ++q)
      if (X[base + off[q]] > m) {  // strict: the first maximum in row-major order wins
        m = X[base + off[q]];
        arg = q;
      }
    const float g = dY[i];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float v = (q == arg) ? g : 0.f;
      if (relu_mask && !(X[base + off[q]] > 0.f)) v = 0.f;
      dX[base + off[q]] = v;
    }
  }
}

int blocks_for(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return (int)std::min<int64_t>(b, (int64_t)device_sm_count() * 32);
}

}  // namespace

constexpr int64_t kI32 = (int64_t)1 << 30;

st_status launch_im2col(const float* X, int B, int H, int W, int C, float* col, cudaStream_t s) {
  const int64_t n = (int64_t)B * H * W * 9 * C;
  const bool v4 = (C % 4) == 0 && (((uintptr_t)X | (uintptr_t)col) & 15) == 0;
  const int64_t nv = v4 ? n / 4 : n;
  if (v4) {
    if (nv < kI32) im2col_kernel<int, 4><<<blocks_for(nv), 256, 0, s>>>(X, B, H, W, C, col);
    else im2col_kernel<int64_t, 4><<<blocks_for(nv), 256, 0, s>>>(X, B, H, W, C, col);
  } else {
    if (nv < kI32) im2col_kernel<int, 1><<<blocks_for(nv), 256, 0, s>>>(X, B, H, W, C, col);
    else im2col_kernel<int64_t, 1><<<blocks_for(nv), 256, 0, s>>>(X, B, H, W, C, col);
  }
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

st_status launch_im2col_pad32(const float* X, int B, int H, int W, int C, float* col, cudaStream_t s) {
  if (9 * C > 32) return set_error(ST_ERR_INPUT, "im2col_pad32: 9·C = %d > 32", 9 * C);
  const int64_t n = (int64_t)B * H * W;
  switch (C) {
    case 1: ST_TRY(launch_pdl(pdl_enabled(), im2col_pad32_kernel<1>, dim3(blocks_for(n)), dim3(256), 0, s, X, B, H, W, col)); break;
    case 2: ST_TRY(launch_pdl(pdl_enabled(), im2col_pad32_kernel<2>, dim3(blocks_for(n)), dim3(256), 0, s, X, B, H, W, col)); break;
    default: ST_TRY(launch_pdl(pdl_enabled(), im2col_pad32_kernel<3>, dim3(blocks_for(n)), dim3(256), 0, s, X, B, H, W, col)); break;
  }
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

st_status launch_col2im(const float* dcol, int B, int H, int W, int C, const float* mask, float* dX, cudaStream_t s) {
  const int64_t n = (int64_t)B * H * W * C;
  const bool v4 = (C % 4) == 0 && (((uintptr_t)dcol | (uintptr_t)mask | (uintptr_t)dX) & 15) == 0;
  const int64_t nv = v4 ? n / 4 : n;
  if (v4) {
    if (nv * 9 < kI32) col2im_kernel<int, 4><<<blocks_for(nv), 256, 0, s>>>(dcol, B, H, W, C, mask, dX);
    else col2im_kernel<int64_t, 4><<<blocks_for(nv), 256, 0, s>>>(dcol, B, H, W, C, mask, dX);
  } else {
    if (nv * 9 < kI32) col2im_kernel<int, 1><<<blocks_for(nv), 256, 0, s>>>(dcol, B, H, W, C, mask, dX);
    else col2im_kernel<int64_t, 1><<<blocks_for(nv), 256, 0, s>>>(dcol, B, H, W, C, mask, dX);
  }
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

st_status launch_maxpool_fwd(const float* X, int B, int H, int W, int C, float* Y, cudaStream_t s) {
  const int64_t n = (int64_t)B * (H / 2) * (W / 2) * C;
  if (n * 4 < kI32) ST_TRY(launch_pdl(pdl_enabled(), maxpool_fwd_kernel<int>, dim3(blocks_for(n)), dim3(256), 0, s, X, B, H, W, C, Y));
  else ST_TRY(launch_pdl(pdl_enabled(), maxpool_fwd_kernel<int64_t>, dim3(blocks_for(n)), dim3(256), 0, s, X, B, H, W, C, Y));
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

st_status launch_maxpool_bwd(const float* X, const float* dY, int B, int H, int W, int C, int relu_mask, float* dX,
                             cudaStream_t s) {
  const int64_t n = (int64_t)B * (H / 2) * (W / 2) * C;
  if (n * 4 < kI32)
    ST_TRY(launch_pdl(pdl_enabled(), maxpool_bwd_kernel<int>, dim3(blocks_for(n)), dim3(256), 0, s, X, dY, B, H, W, C,
                      relu_mask, dX));
  else
    ST_TRY(launch_pdl(pdl_enabled(), maxpool_bwd_kernel<int64_t>, dim3(blocks_for(n)), dim3(256), 0, s, X, dY, B, H,
                      W, C, relu_mask, dX));
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // namespace st
