// Launchers of the stage kernels (sm_100a). Every launcher is stream-ordered,
// checks its launch with cudaGetLastError and returns st_status.
#pragma once

#include "common.hpp"

namespace st {

// ---- programmatic dependent launch -------------------------------------------------
// Kernels that begin with PDL_PROLOGUE (trigger the successor, then wait for the
// predecessor's completion before touching memory) may be launched with programmatic
// stream serialization: their launch and ramp overlap the predecessor's tail.
// ST_PDL_DENSE=0 disables it for the stage paths.
#define PDL_PROLOGUE()                                               \
  do {                                                               \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
    asm volatile("griddepcontrol.wait;" ::: "memory");              \
  } while (0)
bool pdl_enabled();
// SMs of the current device (cached per device ordinal; grid sizing of every launcher)
int device_sm_count();
void set_thread_pdl(int on);  // this host thread's launches (−1: the ST_PDL_DENSE default)
template <typename... KArgs, typename... Args>
inline st_status launch_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  if (pdl) {
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  ST_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
  return ST_OK;
}

// ---- K-B: fused smoothed-gradient update + apply + weight prediction --------
// (Eq. 1, D1 apply, Eq. 4 P:326-328 for s_F and s_B)
struct UpdateConsts {
  float c_gamma;  // γ
  float c_one;    // (1−γ) for EMA, 1 for heavy-ball
  float c_eta;    // η
  float c_f;      // s_F·η
  float c_b;      // s_B·η
};
UpdateConsts make_update_consts(float lr, float gamma, int sF, int sB, int momentum);
st_status launch_update_predict(float* W, float* V, const float* G, float* WF, float* WB, size_t n,
                                const UpdateConsts& c, cudaStream_t s);

// Fig. 7 prediction accuracy: work[2·592] partials, then work[2·592 + 0/1] =
// Σ (W_old − s_eta·V_old − W_now)², Σ (W_old − W_now)² (fp64, deterministic order).
int64_t prediction_error_work_bytes();
st_status launch_prediction_error(const float* W_old, const float* V_old, const float* W_now, size_t n, double s_eta,
                                  double* work, cudaStream_t s);

// In-place K-B targets of one parameter block (a layer's weight matrix or bias):
// pointers at the block's offset in the stage arenas; WF / WB NULL when aliased.
struct UpdateArgs {
  float* W;
  float* V;
  float* WF;
  float* WB;
  UpdateConsts c;
};
// g_b = Σ_b dZ[b][o] followed by the K-B update of the bias block (no G write).
st_status launch_bias_grad_update(const float* dZ, int B, int n_out, const UpdateArgs& u, cudaStream_t s);

// ---- GEMMs of a dense stage (row-major fp32 buffers) ---------------------------
// fwd: Z[B×out] = X[B×in]·W[in×out] + b, optional ReLU
// dX : D[B×in]  = (dZ[B×out]·Wᵀ) ⊙ 1[mask > 0] (mask may be null)
// dW : G[in×out] = Xᵀ·dZ ; gb[out] = Σ_b dZ (gb may be null)
// Split-K partials left unreduced for a consumer kernel (the LSTM cells): output element
// (m, n) = Σ_{s < splits} ws[s·tiles·bn·bm + (((n / bn)·mt + m / bm)·bn + n % bn)·bm + m % bm],
// summed in split order from 0.f (bit-identical to the reduce kernel). splits ≤ 1: the
// GEMM wrote its output normally.
struct SplitPlan {
  const float* ws = nullptr;
  int splits = 0, tiles = 0, mt = 0, bm = 128, bn = 128;
};

struct GemmArgs {
  int mode;  // ST_GEMM_*
  int B, n_in, n_out;
  void* work;  // split-K workspace (gemm_workspace_bytes), 64 KB zeroed counters first
  int64_t work_bytes;
  cudaStream_t stream;
  int max_ctas = 0;  // CTA budget of the launch (0 = every SM); used to share the GPU between streams
  // FP32X3 fwd / dX (TMEM-A kernels): lo = x − trunc_tf32(x) of the activation operand,
  // already computed by its producer (same pitch as the operand); NULL: split here
  const float* act_lo = nullptr;
  SplitPlan* defer = nullptr;  // non-NULL: K-split partials are left for the consumer (see SplitPlan)
  // CTA-pair fwd / dX: launch as a programmatic dependent (the weights stream in while the
  // previous kernel — e.g. the LSTM cell producing this step's h — finishes)
  bool pdl = false;
};
int64_t gemm_workspace_bytes(int B, int max_in, int max_out);
st_status gemm_fwd(const GemmArgs& g, const float* X, const float* W, const float* bias, float* Z, int relu);
// Persistent LSTM recurrence (k_lstm_rec.cu): all T steps of one layer in one cooperative
// launch (FP32X3, B ≤ 128, H % 4 == 0). Forward: gates [T][B][4H] holds Gx_t (+ bias) and
// receives the activated gates, hbuf [(T+1)][B][H] (hbuf[0] = h_{−1}, not read), cbuf
// [T][B][H], hlo2 [2][B][H] scratch. Backward: dOut [T][B][H] → dG [T][B][4H], dc [B][H]
// scratch, dglo2 [2][B][4H] scratch. ST_ERR_UNSUPPORTED: shapes / device do not allow it.
st_status lstm_rec_fwd(const GemmArgs& g, int B, int H, int T, const float* Whh, float* gates, float* hbuf,
                       float* cbuf, float* hlo2);
st_status lstm_rec_bwd(const GemmArgs& g, int B, int H, int T, const float* Whh, const float* gates,
                       const float* cbuf, const float* dOut, float* dG, float* dglo2, float* dc);
st_status gemm_dx(const GemmArgs& g, const float* dZ, const float* W, const float* mask, float* D);
st_status gemm_dw(const GemmArgs& g, const float* X, const float* dZ, float* G, float* gb);
// dW fused with the K-B update (NEXT-3): g = Xᵀ·dZ never reaches HBM;
// the epilogue applies Eq. 1 + apply + predictions to the weight block `w` and the
// bias block `b` (b.W == NULL: no bias). G_scratch is used only by the fallback path.
st_status gemm_dw_update(const GemmArgs& g, const float* X, const float* dZ, const UpdateArgs& w,
                         const UpdateArgs& b, float* G_scratch);
// number of kernel launches the last gemm_* / tc_conv_* call issued on this thread
int gemm_last_launches();

// ---- 3×3 / pad-1 convolution as implicit tcgen05 GEMMs (a10; k_gemm_tc.cu) ----------
// NHWC activations [g.B images][H][W][C], HWIO weights [3][3][Cin][Cout]. The shifted
// windows are 4-D TMA boxes (zero-filled outside the image), so no im2col buffer exists.
// tc_conv_ok: Cin, Cout multiples of 32, tileable H × W, tensor-core mode, ST_CONV_IM2COL≠1.
bool tc_conv_ok(int mode, int H, int W, int Cin, int Cout);
st_status tc_conv_fwd(const GemmArgs& g, const float* X, int H, int W, int Cin, int Cout, const float* Wt,
                      const float* bias, float* Y, int relu);
st_status tc_conv_dx(const GemmArgs& g, const float* dZ, int H, int W, int Cin, int Cout, const float* Wt,
                     const float* mask, float* D);
st_status tc_conv_dw(const GemmArgs& g, const float* X, const float* dZ, int H, int W, int Cin, int Cout, float* G,
                     float* gb);
// first conv with 9·Cin ≤ 32 (RGB): col [P × 32] from launch_im2col_pad32, TMA GEMMs
bool tc_conv_small_ok(int mode, int Cin, int Cout);
st_status tc_conv_small_fwd(const GemmArgs& g, const float* col, int H, int W, int Cin, int Cout, const float* Wt,
                            const float* bias, float* Y, int relu);
st_status tc_conv_small_dw(const GemmArgs& g, const float* col, const float* dZ, int H, int W, int Cin, int Cout,
                           float* G, float* gb);
int tc_last_launches();

// ---- softmax cross-entropy, batch mean (D11) -----------------------------------
// loss_out[0] = mean_b −log softmax(Z_b)[y_b];  dZ = (softmax − onehot)/B.
// rowloss: device scratch [B] floats.
st_status launch_softmax_ce(const float* Z, const int32_t* y, int B, int C, float* rowloss, float* loss_out,
                            float* dZ, cudaStream_t s);

}  // namespace st
