// extern "C" surface of libspectrain.so (include/spectrain.h). Argument
// checking, thread-local error strings and exception firewall; the work is in
// engine.cpp / schedule.cpp / the k_*.cu kernels.
#include <nccl.h>

#include <cstdarg>
#include <cstring>
#include <exception>
#include <string>

#include "engine.hpp"

namespace st {

static thread_local std::string g_last_error;

st_status set_error(st_status s, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}
void clear_error() { g_last_error.clear(); }

// engine.cpp
st_status query_sizes(const st_config* c, st_sizes* out);
st_status ctx_init(const st_config* cfg, const st_buffers* bufs, void* stream, void* comm_fwd, void* comm_bwd,
                   st_ctx** out);
st_status ctx_wait(st_ctx* c);
st_status ctx_mark_after_backward(st_ctx* c, int64_t mb, void* event);
st_status ctx_connect_local(st_ctx** ctxs, int n);
void ctx_destroy(st_ctx* c);
st_status ctx_set_params(st_ctx* c, const float* host, size_t n);
st_status ctx_get_params(st_ctx* c, float* W, float* V, size_t n, int64_t* version);
st_status ctx_forward(st_ctx* c, int64_t mb, const float* x_dev, const int32_t* y_dev, float* loss_host);
st_status ctx_backward(st_ctx* c, int64_t mb);
st_status ctx_predict_and_update(st_ctx* c);
st_status ctx_step(st_ctx* c, const float* x_dev, const int32_t* y_dev, st_step_info* info);
st_status ctx_run(st_ctx* c, int64_t M, const float* xs, const int32_t* ys, float* losses_host, bool host_io);
st_status ctx_run_group(st_ctx** ctxs, int n, int64_t M, const float* xs, const int32_t* ys, float* losses_host);
st_status ctx_get_trace(st_ctx* c, st_event* out, size_t cap, size_t* n);
st_status ctx_set_profiling(st_ctx* c, int on);
st_status ctx_get_profile(st_ctx* c, double* total_ms, int64_t* launches);
st_status ctx_get_layer_profile(st_ctx* c, double* ms, int64_t* counts, size_t n);

}  // namespace st

using namespace st;

static UpdateArgs block_args(float* W, float* V, float* WF, float* WB, size_t off, const UpdateConsts& c) {
  UpdateArgs u;
  u.W = W + off;
  u.V = V + off;
  u.WF = WF ? WF + off : nullptr;
  u.WB = WB ? WB + off : nullptr;
  u.c = c;
  return u;
}

#define GUARD(body)                                                           \
  try {                                                                       \
    body                                                                      \
  } catch (const std::exception& e) {                                         \
    return set_error(ST_ERR_STATE, "internal exception: %s", e.what());       \
  } catch (...) {                                                             \
    return set_error(ST_ERR_STATE, "internal exception");                     \
  }

#define NEED_CTX(c) \
  if (!(c)) return set_error(ST_ERR_INPUT, "context is NULL")

extern "C" {

const char* st_last_error(void) { return g_last_error.c_str(); }
const char* st_version(void) { return "spectrain-b200 0.1 (sm_100a)"; }

int st_version_difference(int k, int N, int dir) {
  if (dir != ST_FWD && dir != ST_BWD) return -1;
  return version_difference(k, N, dir);
}

st_status st_program(int N, int k, int64_t M, int pred, st_event* out, size_t cap, size_t* n) {
  GUARD({
    if (N < 1 || k < 0 || k >= N || M < 0 || !n) return set_error(ST_ERR_INPUT, "st_program: bad arguments");
    std::vector<st_event> ev = program_events(N, k, M, pred);
    *n = ev.size();
    if (!out) return ST_OK;
    if (cap < ev.size()) return set_error(ST_ERR_INPUT, "st_program: cap %zu < %zu", cap, ev.size());
    memcpy(out, ev.data(), ev.size() * sizeof(st_event));
    return ST_OK;
  })
}

st_status st_partition(const double* cost, int n_layers, int N, int32_t* cuts_out, double* max_cost_out) {
  GUARD({ return partition_layers(cost, n_layers, N, cuts_out, max_cost_out); })
}

st_status st_comm_plan(int N, int k, int64_t M, st_comm_group* out, size_t cap, size_t* n) {
  GUARD({
    if (N < 1 || k < 0 || k >= N || M < 0 || !n) return set_error(ST_ERR_INPUT, "st_comm_plan: bad arguments");
    std::vector<CommGroup> p = build_comm_plan(N, k, M);
    *n = p.size();
    if (!out) return ST_OK;
    if (cap < p.size()) return set_error(ST_ERR_INPUT, "st_comm_plan: cap %zu < %zu", cap, p.size());
    memcpy(out, p.data(), p.size() * sizeof(st_comm_group));
    return ST_OK;
  })
}

st_status st_query_sizes(const st_config* cfg, st_sizes* out) {
  GUARD({ return query_sizes(cfg, out); })
}

st_status st_get_nccl_id(uint8_t out[128]) {
  GUARD({
    if (!out) return set_error(ST_ERR_INPUT, "out is NULL");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return set_error(ST_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
    memcpy(out, id.internal, 128);
    return ST_OK;
  })
}

st_status st_init(const st_config* cfg, const st_buffers* bufs, void* stream, void* comm_fwd_stream,
                  void* comm_bwd_stream, st_ctx** out) {
  GUARD({ return ctx_init(cfg, bufs, stream, comm_fwd_stream, comm_bwd_stream, out); })
}

st_status st_connect_local(st_ctx** ctxs, int32_t n) {
  GUARD({ return ctx_connect_local(ctxs, n); })
}

void st_destroy(st_ctx* ctx) {
  try {
    ctx_destroy(ctx);
  } catch (...) {
  }
}

st_status st_set_params(st_ctx* ctx, const float* host, size_t n) {
  NEED_CTX(ctx);
  GUARD({ return ctx_set_params(ctx, host, n); })
}

st_status st_get_params(st_ctx* ctx, float* W, float* V, size_t n, int64_t* version) {
  NEED_CTX(ctx);
  GUARD({ return ctx_get_params(ctx, W, V, n, version); })
}

st_status st_stage_forward(st_ctx* ctx, int64_t mb, const float* x_dev, const int32_t* y_dev, float* loss_host) {
  NEED_CTX(ctx);
  GUARD({ return ctx_forward(ctx, mb, x_dev, y_dev, loss_host); })
}

st_status st_stage_backward(st_ctx* ctx, int64_t mb) {
  NEED_CTX(ctx);
  GUARD({ return ctx_backward(ctx, mb); })
}

st_status st_predict_and_update(st_ctx* ctx) {
  NEED_CTX(ctx);
  GUARD({ return ctx_predict_and_update(ctx); })
}

st_status st_step(st_ctx* ctx, const float* x_dev, const int32_t* y_dev, st_step_info* out) {
  NEED_CTX(ctx);
  GUARD({ return ctx_step(ctx, x_dev, y_dev, out); })
}

st_status st_run(st_ctx* ctx, int64_t M, const float* xs_dev, const int32_t* ys_dev, float* losses_host) {
  NEED_CTX(ctx);
  GUARD({ return ctx_run(ctx, M, xs_dev, ys_dev, losses_host, false); })
}

st_status st_run_host(st_ctx* ctx, int64_t M, const float* xs_host, const int32_t* ys_host, float* losses_host) {
  NEED_CTX(ctx);
  GUARD({ return ctx_run(ctx, M, xs_host, ys_host, losses_host, true); })
}

st_status st_run_group(st_ctx** ctxs, int32_t n, int64_t M, const float* xs_dev, const int32_t* ys_dev,
                       float* losses_host) {
  GUARD({ return ctx_run_group(ctxs, n, M, xs_dev, ys_dev, losses_host); })
}

st_status st_get_trace(st_ctx* ctx, st_event* out, size_t cap, size_t* n) {
  NEED_CTX(ctx);
  GUARD({ return ctx_get_trace(ctx, out, cap, n); })
}

const float* st_losses_device(st_ctx* ctx) { return (ctx && ctx->last_stage) ? ctx->losses_dev : nullptr; }

st_status st_sync(st_ctx* ctx) {
  NEED_CTX(ctx);
  GUARD({
    ST_CUDA_TRY(cudaSetDevice(ctx->device));
    return ctx_wait(ctx);
  })
}

st_status st_record_after_backward(st_ctx* ctx, int64_t mb, void* cuda_event) {
  NEED_CTX(ctx);
  GUARD({ return ctx_mark_after_backward(ctx, mb, cuda_event); })
}

st_status st_p2p_export(st_ctx* ctx, st_p2p_desc* out) {
  NEED_CTX(ctx);
  if (!out) return set_error(ST_ERR_INPUT, "p2p_export: out is NULL");
  GUARD({ return st::p2p_export(ctx, out); })
}

st_status st_p2p_connect(st_ctx* ctx, const st_p2p_desc* prev, const st_p2p_desc* next) {
  NEED_CTX(ctx);
  GUARD({ return st::p2p_connect(ctx, prev, next); })
}

st_status st_set_graph_mode(st_ctx* ctx, int on) {
  NEED_CTX(ctx);
  ctx->graph_mode = on != 0;
  return ST_OK;
}

st_status st_set_profiling(st_ctx* ctx, int on) {
  NEED_CTX(ctx);
  GUARD({ return ctx_set_profiling(ctx, on); })
}

st_status st_get_profile(st_ctx* ctx, double* total_ms, int64_t* launches) {
  NEED_CTX(ctx);
  GUARD({ return ctx_get_profile(ctx, total_ms, launches); })
}

st_status st_get_layer_profile(st_ctx* ctx, double* ms, int64_t* counts, size_t n) {
  NEED_CTX(ctx);
  GUARD({ return ctx_get_layer_profile(ctx, ms, counts, n); })
}

int64_t st_kernel_launches(st_ctx* ctx) { return ctx ? ctx->launches : -1; }

st_status st_update_predict_raw(float* W, float* V, const float* G, float* WF, float* WB, size_t n, float lr,
                                float gamma, int sF, int sB, int momentum, void* stream) {
  GUARD({
    if (n == 0) return ST_OK;
    if (!W || !V || !G) return set_error(ST_ERR_INPUT, "update_predict_raw: W, V, G required");
    auto bad = [](const void* p) { return p && ((uintptr_t)p & 15u); };
    if (bad(W) || bad(V) || bad(G) || bad(WF) || bad(WB))
      return set_error(ST_ERR_INPUT, "update_predict_raw: pointers must be 16-byte aligned");
    if (sF < 0 || sB < 0) return set_error(ST_ERR_INPUT, "update_predict_raw: s must be >= 0");
    if (momentum != ST_MOMENTUM_EMA && momentum != ST_MOMENTUM_HEAVY_BALL)
      return set_error(ST_ERR_INPUT, "update_predict_raw: bad momentum");
    const UpdateConsts c = make_update_consts(lr, gamma, sF, sB, momentum);
    return launch_update_predict(W, V, G, WF, WB, n, c, static_cast<cudaStream_t>(stream));
  })
}

int64_t st_prediction_error_work_bytes(void) { return prediction_error_work_bytes(); }

st_status st_prediction_error_raw(const float* W_old, const float* V_old, const float* W_now, size_t n, int s,
                                  float lr, double* out_host, void* work, void* stream) {
  GUARD({
    if (!out_host) return set_error(ST_ERR_INPUT, "prediction_error_raw: out_host required");
    out_host[0] = out_host[1] = 0.0;
    if (n == 0) return ST_OK;
    if (!W_old || !V_old || !W_now || !work) return set_error(ST_ERR_INPUT, "prediction_error_raw: NULL buffer");
    if (s < 0) return set_error(ST_ERR_INPUT, "prediction_error_raw: s must be >= 0");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    double* w = static_cast<double*>(work);
    ST_TRY(launch_prediction_error(W_old, V_old, W_now, n, (double)s * (double)lr, w, st));
    const int64_t off = prediction_error_work_bytes() / 8 - 2;
    ST_CUDA_TRY(cudaMemcpyAsync(out_host, w + off, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    ST_CUDA_TRY(cudaStreamSynchronize(st));
    return ST_OK;
  })
}

int64_t st_gemm_workspace_bytes(int B, int n_in, int n_out) { return gemm_workspace_bytes(B, n_in, n_out); }

st_status st_gemm_raw(int op, int gemm_mode, int B, int n_in, int n_out, const float* a, const float* b,
                      const float* aux, float* aux_out, float* out, int relu, void* work, void* stream) {
  GUARD({
    GemmArgs g;
    g.mode = gemm_mode;
    g.B = B;
    g.n_in = n_in;
    g.n_out = n_out;
    g.work = work;
    g.work_bytes = gemm_workspace_bytes(B, n_in, n_out);
    g.stream = static_cast<cudaStream_t>(stream);
    if (!a || !b || !out) return set_error(ST_ERR_INPUT, "gemm_raw: NULL operand");
    if (!work) return set_error(ST_ERR_INPUT, "gemm_raw: NULL workspace");
    // split-K tile counters live at the head of the workspace and must start at zero
    ST_CUDA_TRY(cudaMemsetAsync(work, 0, 64 * 1024, g.stream));
    switch (op) {
      case 0: return gemm_fwd(g, a, b, aux, out, relu);
      case 1: return gemm_dx(g, a, b, aux, out);
      case 2: return gemm_dw(g, a, b, out, aux_out);
      default: return set_error(ST_ERR_INPUT, "gemm_raw: op must be 0, 1 or 2");
    }
  })
}

st_status st_dw_update_raw(int gemm_mode, int B, int n_in, int n_out, const float* X, const float* dZ, float* W,
                           float* V, float* WF, float* WB, float lr, float gamma, int sF, int sB, int momentum,
                           float* G_scratch, void* work, void* stream) {
  GUARD({
    if (!X || !dZ || !W || !V || !G_scratch || !work) return set_error(ST_ERR_INPUT, "dw_update_raw: NULL argument");
    GemmArgs g;
    g.mode = gemm_mode;
    g.B = B;
    g.n_in = n_in;
    g.n_out = n_out;
    g.work = work;
    g.work_bytes = gemm_workspace_bytes(B, n_in, n_out);
    g.stream = static_cast<cudaStream_t>(stream);
    ST_CUDA_TRY(cudaMemsetAsync(work, 0, 64 * 1024, g.stream));
    const UpdateConsts c = make_update_consts(lr, gamma, sF, sB, momentum);
    const size_t nw = (size_t)n_in * n_out;
    return gemm_dw_update(g, X, dZ, block_args(W, V, WF, WB, 0, c), block_args(W, V, WF, WB, nw, c), G_scratch);
  })
}

st_status st_softmax_ce_raw(const float* logits, const int32_t* labels, int B, int C, float* loss_dev,
                            float* dlogits, void* work, void* stream) {
  GUARD({
    if (!logits || !labels || !loss_dev || !dlogits || !work) return set_error(ST_ERR_INPUT, "softmax_ce_raw: NULL");
    return launch_softmax_ce(logits, labels, B, C, static_cast<float*>(work), loss_dev, dlogits,
                             static_cast<cudaStream_t>(stream));
  })
}

}  // extern "C"
