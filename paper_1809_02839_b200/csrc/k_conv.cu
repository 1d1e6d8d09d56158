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

__global__ void im2col_kernel(const float* __restrict__ X, int B, int H, int W, int C, float* __restrict__ col) {
  const int64_t total = (int64_t)B * H * W * 9 * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    int64_t t = i / C;
    const int q = (int)(t % 9);  // kh·3 + kw
    const int64_t p = t / 9;     // pixel row b·H·W + h·W + w
    const int w = (int)(p % W);
    const int h = (int)((p / W) % H);
    const int b = (int)(p / ((int64_t)W * H));
    const int hh = h + q / 3 - 1, ww = w + q % 3 - 1;
    col[i] = (hh >= 0 && hh < H && ww >= 0 && ww < W) ? X[(((int64_t)b * H + hh) * W + ww) * C + c] : 0.f;
  }
}

// dX[b,h,w,c] = Σ_{kh,kw} dcol[(b, h+1−kh, w+1−kw), (kh, kw, c)] (valid positions),
// then ⊙ 1[mask > 0] if mask (the ReLU of the layer that produced X).
__global__ void col2im_kernel(const float* __restrict__ dcol, int B, int H, int W, int C, const float* __restrict__ mask,
                              float* __restrict__ dX) {
  const int64_t total = (int64_t)B * H * W * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int64_t p = i / C;
    const int w = (int)(p % W);
    const int h = (int)((p / W) % H);
    const int b = (int)(p / ((int64_t)W * H));
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      const int hh = h + 1 - q / 3, ww = w + 1 - q % 3;
      if (hh >= 0 && hh < H && ww >= 0 && ww < W)
        s += dcol[((((int64_t)b * H + hh) * W + ww) * 9 + q) * C + c];
    }
    if (mask && !(mask[i] > 0.f)) s = 0.f;
    dX[i] = s;
  }
}

__global__ void maxpool_fwd_kernel(const float* __restrict__ X, int B, int H, int W, int C, float* __restrict__ Y) {
  const int Ho = H / 2, Wo = W / 2;
  const int64_t total = (int64_t)B * Ho * Wo * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int64_t p = i / C;
    const int wo = (int)(p % Wo);
    const int ho = (int)((p / Wo) % Ho);
    const int b = (int)(p / ((int64_t)Wo * Ho));
    const float* x = X + (((int64_t)b * H + 2 * ho) * W + 2 * wo) * C + c;
    float m = x[0];
    m = fmaxf(m, x[C]);
    m = fmaxf(m, x[(int64_t)W * C]);
    m = fmaxf(m, x[(int64_t)W * C + C]);
    Y[i] = m;
  }
}

__global__ void maxpool_bwd_kernel(const float* __restrict__ X, const float* __restrict__ dY, int B, int H, int W,
                                   int C, int relu_mask, float* __restrict__ dX) {
  const int Ho = H / 2, Wo = W / 2;
  const int64_t total = (int64_t)B * Ho * Wo * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int64_t p = i / C;
    const int wo = (int)(p % Wo);
    const int ho = (int)((p / Wo) % Ho);
    const int b = (int)(p / ((int64_t)Wo * Ho));
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
  return (int)std::min<int64_t>(b, 148 * 32);
}

}  // namespace

st_status launch_im2col(const float* X, int B, int H, int W, int C, float* col, cudaStream_t s) {
  im2col_kernel<<<blocks_for((int64_t)B * H * W * 9 * C), 256, 0, s>>>(X, B, H, W, C, col);
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

st_status launch_col2im(const float* dcol, int B, int H, int W, int C, const float* mask, float* dX, cudaStream_t s) {
  col2im_kernel<<<blocks_for((int64_t)B * H * W * C), 256, 0, s>>>(dcol, B, H, W, C, mask, dX);
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

st_status launch_maxpool_fwd(const float* X, int B, int H, int W, int C, float* Y, cudaStream_t s) {
  maxpool_fwd_kernel<<<blocks_for((int64_t)B * (H / 2) * (W / 2) * C), 256, 0, s>>>(X, B, H, W, C, Y);
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

st_status launch_maxpool_bwd(const float* X, const float* dY, int B, int H, int W, int C, int relu_mask, float* dX,
                             cudaStream_t s) {
  maxpool_bwd_kernel<<<blocks_for((int64_t)B * (H / 2) * (W / 2) * C), 256, 0, s>>>(X, dY, B, H, W, C, relu_mask,
                                                                                       dX);
  ST_CUDA_TRY(cudaGetLastError());
  return ST_OK;
}

}  // namespace st
