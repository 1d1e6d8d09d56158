// GEMM dispatch for the stage path: tcgen05 tensor-core kernels (k_gemm_tc.cu)
// for ST_GEMM_FP32X3 / ST_GEMM_TF32, CUDA-core fp32 (k_gemm_simt.cu) for
// ST_GEMM_SIMT. Same contract for every mode (kernels.hpp).
#include <cstdlib>

#include "knobs.hpp"
#include "kernels.hpp"

namespace st {

st_status simt_fwd(const GemmArgs& g, const float* X, const float* W, const float* bias, float* Z, int relu);
st_status simt_dx(const GemmArgs& g, const float* dZ, const float* W, const float* mask, float* D);
st_status simt_dw(const GemmArgs& g, const float* X, const float* dZ, float* G, float* gb);

st_status tc_fwd(const GemmArgs& g, const float* X, const float* W, const float* bias, float* Z, int relu);
st_status tc_dx(const GemmArgs& g, const float* dZ, const float* W, const float* mask, float* D);
st_status tc_dw(const GemmArgs& g, const float* X, const float* dZ, float* G, float* gb);
int64_t tc_workspace_bytes(int B, int max_in, int max_out);
int tc_last_launches();
bool tc_dw_fusable(const GemmArgs& g, const float* X, const float* dZ);
bool tc_dw_update_aligned(const UpdateArgs& w);
st_status tc_dw_update(const GemmArgs& g, const float* X, const float* dZ, const UpdateArgs& w, const UpdateArgs& b);
int simt_last_launches();

static thread_local int g_last_launches = 0;

// per host thread (one stage context per thread): the engine sets it per task
static thread_local int tl_pdl = -1;
void set_thread_pdl(int on) { tl_pdl = on; }
bool pdl_enabled() {
  if (tl_pdl >= 0) return tl_pdl != 0;
  static int f = -1;
  if (f < 0) {
    f = dev_knob("ST_PDL_DENSE", 1) != 0 ? 1 : 0;
  }
  return f != 0;
}
int gemm_last_launches() { return g_last_launches; }

int64_t gemm_workspace_bytes(int B, int max_in, int max_out) { return tc_workspace_bytes(B, max_in, max_out); }

static st_status check(const GemmArgs& g) {
  if (g.B <= 0 || g.n_in <= 0 || g.n_out <= 0)
    return set_error(ST_ERR_INPUT, "gemm: bad shape B=%d in=%d out=%d", g.B, g.n_in, g.n_out);
  if (g.mode != ST_GEMM_SIMT && g.mode != ST_GEMM_FP32X3 && g.mode != ST_GEMM_TF32)
    return set_error(ST_ERR_INPUT, "gemm: unknown mode %d", g.mode);
  return ST_OK;
}

st_status gemm_fwd(const GemmArgs& g, const float* X, const float* W, const float* bias, float* Z, int relu) {
  ST_TRY(check(g));
  if (g.defer) g.defer->splits = 1;  // overridden when the TMEM-A kernel defers its reduce
  if (g.mode == ST_GEMM_SIMT) {
    st_status s = simt_fwd(g, X, W, bias, Z, relu);
    g_last_launches = simt_last_launches();
    return s;
  }
  st_status s = tc_fwd(g, X, W, bias, Z, relu);
  g_last_launches = tc_last_launches();
  return s;
}

st_status gemm_dx(const GemmArgs& g, const float* dZ, const float* W, const float* mask, float* D) {
  ST_TRY(check(g));
  if (g.defer) g.defer->splits = 1;  // overridden when the TMEM-A kernel defers its reduce
  if (g.mode == ST_GEMM_SIMT) {
    st_status s = simt_dx(g, dZ, W, mask, D);
    g_last_launches = simt_last_launches();
    return s;
  }
  st_status s = tc_dx(g, dZ, W, mask, D);
  g_last_launches = tc_last_launches();
  return s;
}

st_status gemm_dw(const GemmArgs& g, const float* X, const float* dZ, float* G, float* gb) {
  ST_TRY(check(g));
  if (g.mode == ST_GEMM_SIMT) {
    st_status s = simt_dw(g, X, dZ, G, gb);
    g_last_launches = simt_last_launches();
    return s;
  }
  st_status s = tc_dw(g, X, dZ, G, gb);
  g_last_launches = tc_last_launches();
  return s;
}

st_status gemm_dw_update(const GemmArgs& g, const float* X, const float* dZ, const UpdateArgs& w,
                         const UpdateArgs& b, float* G_scratch) {
  ST_TRY(check(g));
  if (tc_dw_fusable(g, X, dZ) && tc_dw_update_aligned(w)) {
    st_status s = tc_dw_update(g, X, dZ, w, b);
    g_last_launches = tc_last_launches();
    return s;
  }
  // fallback (pitch not 16-byte aligned, SIMT mode, B > 128): G through HBM + K-B over the block
  int launches = 0;
  ST_TRY(gemm_dw(g, X, dZ, G_scratch, b.W ? G_scratch + (size_t)g.n_in * g.n_out : nullptr));
  launches += g_last_launches;
  const size_t n = (size_t)g.n_in * g.n_out + (b.W ? (size_t)g.n_out : 0);
  // weight and bias blocks are contiguous in the arenas (S:106 layout)
  ST_TRY(launch_update_predict(w.W, w.V, G_scratch, w.WF, w.WB, n, w.c, g.stream));
  g_last_launches = launches + 1;
  return ST_OK;
}

}  // namespace st
