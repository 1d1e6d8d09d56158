// The stage engine behind the C-ABI (include/spectrain.h).
//
// One context = one pipeline stage k of N. It owns no device memory:
// it carves the caller's arenas, runs the stage's 1F1B program (schedule.cpp),
// and for each task launches, on the borrowed compute stream:
//   F(i): [recv act] → per layer gemm_fwd with WF (+bias, ReLU) → [CE] → [send act]
//   B(j): [recv grad] → per layer (reverse) gemm_dx with WB (ReLU mask fused),
//         gemm_dw (+bias grad) → [send grad]
//   update: K-B (k_update.cu) — Eq. 1, D1 apply, WF/WB for the next tasks.
#include <nvtx3/nvToolsExt.h>
#include <chrono>
#include <cmath>
#include <cstring>
#include <thread>

#include "engine.hpp"
#include "knobs.hpp"

using st::set_error;

namespace st {

// ST_PRED_STASH slot pitch: P rounded up to 64 floats (256 B), so every slot keeps the
// alignment of the arena (the fused dW + update writes its WF block with float4 / TMA)
static int64_t stash_pitch(int64_t P) { return (P + 63) / 64 * 64; }

namespace {

int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
constexpr int64_t kAlignBytes = 256;
constexpr int64_t kAlignFloats = kAlignBytes / 4;

struct Layout {
  std::vector<LayerInfo> layers;
  int64_t P = 0;
  int64_t slot_elems = 0;
  int S = 1;
  int sF = 0, sB = 0;
  int in_first = 0, out_last = 0, max_in = 0, max_out = 0;
  int prev_act = ST_ACT_NONE;  // activation of the layer feeding this stage (k > 0)
  bool first = true, last = true;
  // work offsets (bytes)
  int64_t off_send_fwd = -1, off_recv_bwd = -1, off_send_bwd = -1, off_logits = -1, off_dlogits = -1;
  int64_t off_bufA = -1, off_bufB = -1, off_bufC = -1, off_losses = -1, off_rowloss = -1, off_ring_fwd = -1, off_ring_bwd = -1;
  int64_t off_ws = -1, off_ystage = -1;
  int64_t off_lrec = -1, off_ldh = -1, off_ldc = -1, off_ldG = -1, off_escr = -1, off_col = -1, off_dcol = -1;
  int64_t off_lhlo = -1, off_ldglo = -1;
  int64_t gemm_rows = 1;
  int64_t off_ws2 = -1;
  int gemm_in = 1, gemm_out = 1;  // largest GEMM operand widths (workspace sizing)
  int T = 1;
  int64_t R = 1;
  int rep_prev = 1, rep_self = 1, rep_next = 1;  // replicas of stages k−1, k, k+1 (NEXT-4)
  bool embed_first = false;
  size_t ring_fwd_elems = 0, ring_bwd_elems = 0;
  st_sizes sizes{};
};

int64_t layer_win(const st_layer& y) {
  return (y.kind == ST_LAYER_CONV || y.kind == ST_LAYER_POOL) ? (int64_t)y.hw * y.hw * y.n_in : y.n_in;
}
int64_t layer_wout(const st_layer& y) {
  if (y.kind == ST_LAYER_CONV) return (int64_t)y.hw * y.hw * y.n_out;
  if (y.kind == ST_LAYER_POOL) return (int64_t)(y.hw / 2) * (y.hw / 2) * y.n_out;
  return y.n_out;
}

st_status validate_and_layout(const st_config* c, Layout* L) {
  if (!c) return set_error(ST_ERR_INPUT, "config is NULL");
  if (c->num_stages < 1) return set_error(ST_ERR_INPUT, "num_stages must be >= 1 (got %d)", c->num_stages);
  if (c->stage < 0 || c->stage >= c->num_stages)
    return set_error(ST_ERR_INPUT, "stage %d outside [0, %d)", c->stage, c->num_stages);
  if (c->num_layers < c->num_stages || !c->layers)
    return set_error(ST_ERR_INPUT, "need at least one layer per stage (%d layers, %d stages)", c->num_layers,
                     c->num_stages);
  if (c->batch < 1) return set_error(ST_ERR_INPUT, "batch must be >= 1");
  if (!(c->lr > 0.f) || !std::isfinite(c->lr)) return set_error(ST_ERR_INPUT, "lr must be > 0");
  if (!(c->gamma > 0.f && c->gamma <= 1.f)) return set_error(ST_ERR_INPUT, "gamma must be in (0, 1]");
  if (c->pred != ST_PRED_SPECTRAIN && c->pred != ST_PRED_NONE && c->pred != ST_PRED_STASH &&
      c->pred != ST_PRED_STALENESS_FREE)
    return set_error(ST_ERR_INPUT, "bad pred");
  if (c->momentum != ST_MOMENTUM_EMA && c->momentum != ST_MOMENTUM_HEAVY_BALL)
    return set_error(ST_ERR_INPUT, "bad momentum");
  if (c->gemm != ST_GEMM_FP32X3 && c->gemm != ST_GEMM_TF32 && c->gemm != ST_GEMM_SIMT)
    return set_error(ST_ERR_INPUT, "bad gemm mode");
  if (c->loss != ST_LOSS_SOFTMAX_CE) return set_error(ST_ERR_INPUT, "bad loss");
  if (c->transport != ST_TRANSPORT_NCCL && c->transport != ST_TRANSPORT_LOCAL && c->transport != ST_TRANSPORT_P2P)
    return set_error(ST_ERR_INPUT, "bad transport");
  if (c->max_minibatches < 1) return set_error(ST_ERR_INPUT, "max_minibatches must be >= 1");
  const int N = c->num_stages, k = c->stage;
  if (N > 1 && !c->cuts) return set_error(ST_ERR_INPUT, "cuts is NULL");
  std::vector<int> bounds{0};
  for (int i = 0; i < N - 1; ++i) {
    if (c->cuts[i] <= bounds.back() || c->cuts[i] >= c->num_layers)
      return set_error(ST_ERR_INPUT, "cuts must be strictly increasing in (0, %d)", c->num_layers);
    bounds.push_back(c->cuts[i]);
  }
  bounds.push_back(c->num_layers);
  if (c->seq_len < 1) return set_error(ST_ERR_INPUT, "seq_len must be >= 1");
  for (int l = 0; l < c->num_layers; ++l) {
    const st_layer& y = c->layers[l];
    if (y.n_in < 1 || y.n_out < 1) return set_error(ST_ERR_SHAPE, "layer %d: bad dims", l);
    if (y.act != ST_ACT_NONE && y.act != ST_ACT_RELU) return set_error(ST_ERR_INPUT, "layer %d: bad act", l);
    if (y.kind < ST_LAYER_DENSE || y.kind > ST_LAYER_POOL)
      return set_error(ST_ERR_INPUT, "layer %d: bad kind %d", l, y.kind);
    if (y.kind == ST_LAYER_EMBED && l != 0) return set_error(ST_ERR_INPUT, "EMBED must be the network's layer 0");
    if ((y.kind == ST_LAYER_EMBED || y.kind == ST_LAYER_LSTM || y.kind == ST_LAYER_POOL) && y.act != ST_ACT_NONE)
      return set_error(ST_ERR_INPUT, "layer %d: EMBED / LSTM / POOL layers take act = NONE", l);
    if (y.kind == ST_LAYER_CONV || y.kind == ST_LAYER_POOL) {
      if (y.hw < 1 || (y.kind == ST_LAYER_POOL && (y.hw % 2 || y.n_in != y.n_out)))
        return set_error(ST_ERR_SHAPE, "layer %d: bad conv / pool geometry", l);
      if (c->seq_len != 1) return set_error(ST_ERR_INPUT, "conv / pool layers need seq_len = 1");
    }
    if (l > 0 && layer_wout(c->layers[l - 1]) != layer_win(y))
      return set_error(ST_ERR_SHAPE, "layer chain mismatch: layer %d out %lld != layer %d in %lld", l - 1,
                       (long long)layer_wout(c->layers[l - 1]), l, (long long)layer_win(y));
  }
  if (c->layers[c->num_layers - 1].kind != ST_LAYER_DENSE)
    return set_error(ST_ERR_INPUT, "the network's last layer must be DENSE (softmax CE)");
  const int l0 = bounds[k], l1 = bounds[k + 1];
  // hybrid DP × PP: replicas per stage (NEXT-4)
  auto rep = [&](int s) -> int { return (c->replicas && s >= 0 && s < N) ? c->replicas[s] : 1; };
  for (int s = 0; s < N; ++s) {
    if (rep(s) < 1) return set_error(ST_ERR_INPUT, "replicas[%d] = %d must be >= 1", s, rep(s));
    if (rep(s) == 1) continue;
    if (s == N - 1) return set_error(ST_ERR_INPUT, "the last stage cannot be replicated (it owns the batch-mean loss)");
    if ((s > 0 && rep(s - 1) > 1) || rep(s + 1) > 1)
      return set_error(ST_ERR_INPUT, "adjacent stages %d and %d cannot both be replicated", s, rep(s - 1) > 1 ? s - 1 : s + 1);
    if (c->seq_len != 1) return set_error(ST_ERR_INPUT, "replicated stages need seq_len = 1 (row slices per sample)");
    if (c->batch % rep(s)) return set_error(ST_ERR_INPUT, "batch %d not divisible by replicas[%d] = %d", c->batch, s, rep(s));
    if (c->transport == ST_TRANSPORT_P2P) return set_error(ST_ERR_INPUT, "replicated stages need NCCL or LOCAL transport");
  }
  if (c->replica < 0 || c->replica >= rep(k))
    return set_error(ST_ERR_INPUT, "replica %d outside [0, %d)", c->replica, rep(k));
  L->rep_prev = k > 0 ? rep(k - 1) : 1;
  L->rep_self = rep(k);
  L->rep_next = k + 1 < N ? rep(k + 1) : 1;
  const int64_t B = c->batch / L->rep_self;  // rows of this context (a replica: its slice)
  const int64_t T = c->seq_len;
  const int64_t R = B * T;
  L->T = (int)T;
  L->R = R;
  L->first = (k == 0);
  L->last = (k == N - 1);
  L->S = N - k;
  L->prev_act = (k > 0) ? c->layers[l0 - 1].act : ST_ACT_NONE;
  L->embed_first = c->layers[l0].kind == ST_LAYER_EMBED;
  int64_t off = 0, soff = 0;
  int max_h = 0, max_vocab = 0;
  int64_t max_col = 0, gemm_rows = R;
  for (int l = l0; l < l1; ++l) {
    const st_layer& y = c->layers[l];
    const bool has_bias = (y.kind == ST_LAYER_DENSE || y.kind == ST_LAYER_CONV) && y.bias;
    LayerInfo li{y.n_in, y.n_out, y.act, has_bias ? 1 : 0, y.kind, y.hw, layer_win(y), layer_wout(y), off, -1, -1, 0,
                 -1, -1, -1, -1};
    if (y.kind == ST_LAYER_POOL) {
      // no parameters
    } else if (y.kind == ST_LAYER_CONV) {
      off += (int64_t)9 * y.n_in * y.n_out;
      if (y.bias) {
        li.b_off = off;
        off += y.n_out;
      }
      const int64_t P = B * y.hw * y.hw;
      max_col = std::max(max_col, P * std::max<int64_t>(9 * y.n_in, 32));  // ≥ 32: padded first-conv im2col
      gemm_rows = std::max(gemm_rows, P);
    } else if (y.kind == ST_LAYER_EMBED) {
      off += (int64_t)y.n_in * y.n_out;
      max_vocab = std::max(max_vocab, y.n_in);
    } else if (y.kind == ST_LAYER_LSTM) {
      const int64_t H = y.n_out;
      off += (int64_t)y.n_in * 4 * H;
      li.whh_off = off;
      off += H * 4 * H;
      li.b_off = off;
      off += 4 * H;
      max_h = std::max(max_h, (int)H);
    } else {
      off += (int64_t)y.n_in * y.n_out;
      if (y.bias) {
        li.b_off = off;
        off += y.n_out;
      }
    }
    li.n_params = off - li.w_off;
    // layer input: aliases the previous LSTM's h buffer when that layer is in this stage
    const bool alias = (l > l0) && c->layers[l - 1].kind == ST_LAYER_LSTM;
    if (!alias) {
      li.stash_off = soff;
      soff += align_up(y.kind == ST_LAYER_EMBED ? R : R * li.win, kAlignFloats);
    }
    if (y.kind == ST_LAYER_LSTM) {
      const int64_t H = y.n_out;
      li.gates_off = soff;
      soff += align_up(R * 4 * H, kAlignFloats);
      li.c_off = soff;
      soff += align_up(R * H, kAlignFloats);
      li.h_off = soff;
      soff += align_up((R + B) * H, kAlignFloats);
    }
    // buffer widths (messages, ping-pong) and GEMM operand widths
    L->max_in = std::max<int>(L->max_in, y.kind == ST_LAYER_EMBED ? 1 : (int)li.win);
    L->max_out = std::max<int>(L->max_out, y.kind == ST_LAYER_LSTM ? 4 * y.n_out : (int)li.wout);
    if (y.kind == ST_LAYER_CONV) {
      L->gemm_in = std::max(L->gemm_in, 9 * y.n_in);
      L->gemm_out = std::max(L->gemm_out, y.n_out);
    } else if (y.kind == ST_LAYER_LSTM) {
      L->gemm_in = std::max(L->gemm_in, y.n_in);
      L->gemm_out = std::max(L->gemm_out, 4 * y.n_out);
    } else if (y.kind == ST_LAYER_DENSE) {
      L->gemm_in = std::max(L->gemm_in, y.n_in);
      L->gemm_out = std::max(L->gemm_out, y.n_out);
    }
    L->layers.push_back(li);
  }
  L->gemm_rows = gemm_rows;
  L->P = off;
  L->slot_elems = soff;
  L->in_first = (int)layer_win(c->layers[l0]);
  L->out_last = (int)layer_wout(c->layers[l1 - 1]);
  L->sF = stage_s(c->pred, k, N, ST_FWD);
  L->sB = stage_s(c->pred, k, N, ST_BWD);

  // work carve-up
  int64_t w = 0;
  auto take = [&](int64_t floats) {
    const int64_t o = w;
    w += align_up(floats * 4, kAlignBytes);
    return o;
  };
  const int64_t width = std::max(L->max_in, L->max_out);
  // message buffers: two slots each (mini-batch parity), so the transfer of one
  // mini-batch overlaps the compute of the next
  if (!L->last) {
    L->off_send_fwd = take(2 * align_up(R * L->out_last, kAlignFloats));
    L->off_recv_bwd = take(2 * align_up(R * L->out_last, kAlignFloats));
  }
  if (!L->first) L->off_send_bwd = take(2 * align_up(R * L->in_first, kAlignFloats));
  if (L->last) {
    L->off_logits = take(R * L->out_last);
    L->off_dlogits = take(R * L->out_last);
    L->off_rowloss = take(R);
    L->off_ystage = take(R);
  }
  L->off_bufA = take(R * width);
  L->off_bufB = take(R * width);
  L->off_bufC = take(R * width);
  L->off_losses = take(c->max_minibatches);
  if (max_h > 0) {
    L->off_lrec = take(B * 4 * max_h);
    L->off_ldh = take(B * max_h);
    L->off_ldc = take(B * max_h);
    L->off_ldG = take(R * 4 * max_h);
    L->off_lhlo = take(2 * B * max_h);       // two slots: the persistent recurrence reads h_{t−1}'s
    L->off_ldglo = take(2 * B * 4 * max_h);  // lo while step t writes h_t's (dG likewise)
  }
  if (max_vocab > 0) L->off_escr = take(embed_grad_scratch_bytes((int)R, max_vocab) / 4 + 1);
  if (max_col > 0) {
    L->off_col = take(max_col);
    L->off_dcol = take(max_col);
  }
  if (c->transport == ST_TRANSPORT_LOCAL) {
    if (!L->last) {
      L->ring_fwd_elems = (size_t)(R * L->out_last);
      L->off_ring_fwd = take((int64_t)L->ring_fwd_elems * (N + 1));
    }
    if (!L->first) {
      L->ring_bwd_elems = (size_t)(R * L->in_first);
      L->off_ring_bwd = take((int64_t)L->ring_bwd_elems * (N + 1));
    }
  }
  L->off_ws = w;
  w += align_up(gemm_workspace_bytes((int)gemm_rows, L->gemm_in, L->gemm_out), kAlignBytes);
  // the side stream (dW + update overlapped with the next dX) gets its own GEMM workspace
  L->off_ws2 = w;
  w += align_up(gemm_workspace_bytes((int)gemm_rows, L->gemm_in, L->gemm_out), kAlignBytes);

  st_sizes& z = L->sizes;
  z.params = L->P;
  z.w_bytes = z.v_bytes = z.g_bytes = align_up(L->P * 4, kAlignBytes);
  // ST_PRED_STASH: WF is the weight stash, one W copy per mini-batch in flight (N−k slots)
  z.wf_bytes = c->pred == ST_PRED_STASH ? stash_pitch(L->P) * 4 * L->S : (L->sF > 0 ? z.w_bytes : 0);
  z.wb_bytes = (L->sB > 0 && L->sB != L->sF) ? z.w_bytes : 0;
  z.stash_bytes = (int64_t)L->S * L->slot_elems * 4;
  z.work_bytes = w;
  z.s_fwd = L->sF;
  z.s_bwd = L->sB;
  return ST_OK;
}

// ---- profiling helpers ----------------------------------------------------------
// An event the caller or the profiler reads the time of: inside a graph capture it must be
// an external event record node (a plain record there only orders the graph's own nodes)
static cudaError_t record_timing_event(st_ctx* c, cudaEvent_t e, cudaStream_t s) {
  return cudaEventRecordWithFlags(e, s, c->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
}

// NVTX range for a timeline tool (nsys / ncu --nvtx); header-only NVTX v3, a no-op
// unless a tool is attached
struct NvtxRange {
  explicit NvtxRange(const char* fmt, int a, long long b) {
    char name[64];
    snprintf(name, sizeof name, fmt, a, b);
    nvtxRangePushA(name);
  }
  ~NvtxRange() { nvtxRangePop(); }
};

struct Timed {
  st_ctx* c;
  int cls;
  cudaStream_t s;
  cudaEvent_t b = nullptr;
  Timed(st_ctx* ctx, int k, cudaStream_t stream = nullptr) : c(ctx), cls(k), s(stream ? stream : ctx->stream) {
    if (!c->prof.on || !((c->prof.mask >> cls) & 1u)) return;
    cudaEvent_t a = get();
    b = get();
    record_timing_event(c, a, s);
    c->prof.pairs.push_back({cls, a, b});
  }
  ~Timed() {
    if (b) record_timing_event(c, b, s);
  }
  cudaEvent_t get() {
    if (!c->prof.pool.empty()) {
      cudaEvent_t e = c->prof.pool.back();
      c->prof.pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};

// Per-layer bracket (ST_PROF_LAYERS): one event pair around all of layer l's work of
// one pass (dir 0 forward, 1 backward) on stream s; backward brackets on the main and
// the side stream are both counted (the profiled backward runs serialised).
struct TimedLayer {
  st_ctx* c;
  cudaStream_t s;
  cudaEvent_t b = nullptr;
  TimedLayer(st_ctx* ctx, size_t l, int dir, cudaStream_t stream = nullptr)
      : c(ctx), s(stream ? stream : ctx->stream) {
    if (!c->prof.layers) return;
    cudaEvent_t a = take();
    b = take();
    record_timing_event(c, a, s);
    c->prof.lpairs.push_back({(int)(2 * l + dir), a, b});
  }
  ~TimedLayer() {
    if (b) record_timing_event(c, b, s);
  }
  cudaEvent_t take() {
    if (!c->prof.pool.empty()) {
      cudaEvent_t e = c->prof.pool.back();
      c->prof.pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};

}  // namespace

// ---- engine internals used by capi.cpp -------------------------------------------

st_status query_sizes(const st_config* c, st_sizes* out) {
  Layout L;
  ST_TRY(validate_and_layout(c, &L));
  if (out) *out = L.sizes;
  return ST_OK;
}

st_status ctx_wait(st_ctx* c);

static void begin_session(st_ctx* c, int64_t M) {
  p2p_begin_session(c);
  c->program = build_program(c->N, c->k, M);
  c->plan = build_comm_plan(c->N, c->k, M);
  c->pc = 0;
  c->plan_next = 0;
  c->session_M = M;
  c->pending_update = false;
  // message slots: nothing in flight at a session boundary (the previous session's comm
  // streams were joined into the compute stream)
  for (int b = 0; b < 2; ++b) c->sent_fwd_pending[b] = c->sent_bwd_pending[b] = c->bwd_ring_done[b] = false;
  std::fill(c->bwd_slot_done.begin(), c->bwd_slot_done.end(), 0);
}

st_status ctx_init(const st_config* cfg, const st_buffers* bufs, void* stream, void* comm_fwd, void* comm_bwd,
                   st_ctx** out) {
  if (!out) return set_error(ST_ERR_INPUT, "out is NULL");
  *out = nullptr;
  Layout L;
  ST_TRY(validate_and_layout(cfg, &L));
  if (!bufs || !bufs->W || !bufs->V || !bufs->G || !bufs->stash || !bufs->work)
    return set_error(ST_ERR_INPUT, "missing buffer (W, V, G, stash, work are required)");
  if (L.sizes.wf_bytes && !bufs->WF) return set_error(ST_ERR_INPUT, "WF buffer required (s_F = %d / stash)", L.sF);
  if (L.sizes.wb_bytes && !bufs->WB) return set_error(ST_ERR_INPUT, "WB buffer required (s_B = %d)", L.sB);
  auto misaligned = [](const void* p) { return p && ((uintptr_t)p % kAlignBytes) != 0; };
  if (misaligned(bufs->W) || misaligned(bufs->V) || misaligned(bufs->G) || misaligned(bufs->WF) ||
      misaligned(bufs->WB) || misaligned(bufs->stash) || misaligned(bufs->work))
    return set_error(ST_ERR_INPUT, "device buffers must be %lld-byte aligned", (long long)kAlignBytes);
  ST_CUDA_TRY(cudaSetDevice(cfg->device));

  std::unique_ptr<st_ctx> c(new st_ctx());
  c->N = cfg->num_stages;
  c->k = cfg->stage;
  c->B = (int)(L.R / L.T);  // rows of this context: the global batch, or a replica's slice
  c->B_global = cfg->batch;
  c->rep_prev = L.rep_prev;
  c->rep_self = L.rep_self;
  c->rep_next = L.rep_next;
  c->replica = cfg->replica;
  for (int s2 = 0; s2 < c->N; ++s2) c->reps.push_back(cfg->replicas ? cfg->replicas[s2] : 1);
  c->T = L.T;
  c->R = L.R;
  c->embed_first = L.embed_first;
  c->lr = cfg->lr;
  c->gamma = cfg->gamma;
  c->pred = cfg->pred;
  c->momentum = cfg->momentum;
  c->gemm = cfg->gemm;
  c->loss = cfg->loss;
  c->transport_kind = cfg->transport;
  c->device = cfg->device;
  c->max_mb = cfg->max_minibatches;
  c->layers = L.layers;
  c->P = L.P;
  c->sF = L.sF;
  c->sB = L.sB;
  c->max_width_in = L.max_in;
  c->max_width_out = L.max_out;
  c->first_stage = L.first;
  c->last_stage = L.last;
  c->prev_act = L.prev_act;
  c->in_first = L.in_first;
  c->out_last = L.out_last;
  c->W = bufs->W;
  c->V = bufs->V;
  c->G = bufs->G;
  c->WF_out = L.sF > 0 ? bufs->WF : nullptr;
  c->WB_out = (L.sB > 0 && L.sB != L.sF) ? bufs->WB : nullptr;
  c->WF = L.sF > 0 ? bufs->WF : bufs->W;
  c->WB = L.sB == 0 ? bufs->W : (L.sB == L.sF ? c->WF : bufs->WB);
  c->wstash = c->pred == ST_PRED_STASH ? bufs->WF : nullptr;
  c->stash_ver.assign((size_t)L.S, 0);
  c->stash = static_cast<float*>(bufs->stash);
  c->slot_elems = L.slot_elems;
  c->S = L.S;
  char* w = static_cast<char*>(bufs->work);
  auto at = [&](int64_t off) { return off < 0 ? nullptr : reinterpret_cast<float*>(w + off); };
  {
    const int64_t mf = align_up(L.R * L.out_last, kAlignFloats), mb = align_up(L.R * L.in_first, kAlignFloats);
    for (int b = 0; b < 2; ++b) {
      c->send_fwd2[b] = L.off_send_fwd < 0 ? nullptr : at(L.off_send_fwd) + b * mf;
      c->recv_bwd2[b] = L.off_recv_bwd < 0 ? nullptr : at(L.off_recv_bwd) + b * mf;
      c->send_bwd2[b] = L.off_send_bwd < 0 ? nullptr : at(L.off_send_bwd) + b * mb;
    }
    c->send_fwd = c->send_fwd2[0];
    c->recv_bwd = c->recv_bwd2[0];
    c->send_bwd = c->send_bwd2[0];
  }
  c->logits = at(L.off_logits);
  c->dlogits = at(L.off_dlogits);
  c->rowloss = at(L.off_rowloss);
  c->y_stage = reinterpret_cast<int32_t*>(at(L.off_ystage));
  c->lstm_rec = at(L.off_lrec);
  c->lstm_dh = at(L.off_ldh);
  c->lstm_dc = at(L.off_ldc);
  c->lstm_dG = at(L.off_ldG);
  c->lstm_hlo = at(L.off_lhlo);
  c->lstm_dglo = at(L.off_ldglo);
  c->embed_scratch = at(L.off_escr);
  c->conv_col = at(L.off_col);
  c->conv_dcol = at(L.off_dcol);
  c->gemm_rows_max = L.gemm_rows;
  c->gemm_in_max = L.gemm_in;
  c->gemm_out_max = L.gemm_out;
  c->bufA = at(L.off_bufA);
  c->bufB = at(L.off_bufB);
  c->bufC = at(L.off_bufC);
  c->losses_dev = at(L.off_losses);
  c->ring_fwd = at(L.off_ring_fwd);
  c->ring_bwd = at(L.off_ring_bwd);
  c->ring_fwd_elems = L.ring_fwd_elems;
  c->ring_bwd_elems = L.ring_bwd_elems;
  c->gemm_ws = w + L.off_ws;
  c->gemm_ws2 = w + L.off_ws2;
  c->stream = static_cast<cudaStream_t>(stream);
  {
    int sms = 0;
    ST_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg->device));
    c->sm_count = std::max(2, sms);
    c->dwu_sms = std::min(c->dwu_sms, c->sm_count - 2);
  }
  // comm streams: the caller's, or library-owned non-blocking streams (P2P: none — the
  // compute stream's kernels move the data; fewer streams also keeps its spin-waits off
  // hardware queues shared with a co-located peer, see st_p2p_connect)
  if (cfg->transport == ST_TRANSPORT_P2P) {
    c->comm_fwd = c->comm_bwd = c->stream;
  } else {
    if (comm_fwd) {
      c->comm_fwd = static_cast<cudaStream_t>(comm_fwd);
    } else {
      ST_CUDA_TRY(cudaStreamCreateWithFlags(&c->comm_fwd, cudaStreamNonBlocking));
      c->own_comm_fwd = true;
    }
    if (comm_bwd) {
      c->comm_bwd = static_cast<cudaStream_t>(comm_bwd);
    } else {
      ST_CUDA_TRY(cudaStreamCreateWithFlags(&c->comm_bwd, cudaStreamNonBlocking));
      c->own_comm_bwd = true;
    }
  }
  {
    auto mk = [](cudaEvent_t* e) { return cudaEventCreateWithFlags(e, cudaEventDisableTiming); };
    for (int b = 0; b < 2; ++b) {
      ST_CUDA_TRY(mk(&c->ev_sent_fwd[b]));
      ST_CUDA_TRY(mk(&c->ev_sent_bwd[b]));
      ST_CUDA_TRY(mk(&c->ev_recv_bwd[b]));
      ST_CUDA_TRY(mk(&c->ev_bwd_ring[b]));
      ST_CUDA_TRY(mk(&c->ev_join[b]));
    }
    c->ev_recv_fwd.assign((size_t)c->S, nullptr);
    c->ev_bwd_slot.assign((size_t)c->S, nullptr);
    c->bwd_slot_done.assign((size_t)c->S, 0);
    for (int i = 0; i < c->S; ++i) {
      ST_CUDA_TRY(mk(&c->ev_recv_fwd[(size_t)i]));
      ST_CUDA_TRY(mk(&c->ev_bwd_slot[(size_t)i]));
    }
    ST_CUDA_TRY(mk(&c->ev_fwd_done));
    ST_CUDA_TRY(mk(&c->ev_dx_ready));
  }
  if (const char* e = getenv("ST_COMM_TIMEOUT_S")) c->comm_timeout_s = std::max(1.0, atof(e));

  if (c->transport_kind == ST_TRANSPORT_NCCL) {
    st_status e;
    c->tp = make_nccl_transport(cfg->nccl_id, c->N, c->k, c->device, c->reps, c->replica, &e);
    if (e != ST_OK) return e;
  } else if (c->transport_kind == ST_TRANSPORT_P2P && c->N > 1) {
    const st_status e = p2p_alloc(c.get());
    if (e != ST_OK) {
      p2p_free(c.get());
      return e;
    }
  }
  ST_CUDA_TRY(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  c->side_events.resize(c->layers.size() + 1);
  for (auto& e : c->side_events) ST_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (const int v = dev_knob("ST_DWU_SMS", 0)) {  // one dW + update budget for every layer (sweeps)
    c->dwu_sms = std::min(std::max(1, v), c->sm_count - 2);
    c->dwu_env = true;
  }
  c->conv_overlap = dev_knob("ST_CONV_OVERLAP", 0) != 0;
  c->bwd_serial = dev_knob("ST_BWD_SERIAL", 1) != 0;
  c->pdl_serial = dev_knob("ST_PDL_SERIAL", 1) != 0;
  c->pdl = dev_knob("ST_PDL", 1) != 0;
  c->pdl_dense = dev_knob("ST_PDL_DENSE", 1) != 0;
  // several stage contexts sharing one GPU (LOCAL transport): their kernels interleave
  // across streams and waiting dependents would hold SMs the other stages need
  // (wide FCN at 2 co-located stages 45.8k → 41.8k samples/s with it)
  int co_located = 0;
  for (int r : c->reps) co_located += r;
  c->shares_gpu = c->transport_kind == ST_TRANSPORT_LOCAL && co_located > 1;
  if (c->transport_kind == ST_TRANSPORT_LOCAL && c->N > 1) {
    c->pdl_dense = false;
    c->pdl = false;
  }
  ST_CUDA_TRY(cudaMemsetAsync(c->V, 0, (size_t)c->P * 4, c->stream));
  ST_CUDA_TRY(cudaMemsetAsync(c->losses_dev, 0xff, (size_t)c->max_mb * 4, c->stream));  // NaN
  // GEMM workspace: split-K tile counters must start at zero (they self-reset afterwards)
  ST_CUDA_TRY(cudaMemsetAsync(c->gemm_ws, 0, 64 * 1024, c->stream));  // split-K counters
  ST_CUDA_TRY(cudaMemsetAsync(c->gemm_ws2, 0, 64 * 1024, c->stream));
  begin_session(c.get(), c->max_mb);
  *out = c.release();
  return ST_OK;
}

st_status ctx_connect_local(st_ctx** ctxs, int n) {
  if (!ctxs || n < 1 || !ctxs[0]) return set_error(ST_ERR_INPUT, "connect_local: need >= 1 context");
  const int N = ctxs[0]->N;
  const std::vector<int> reps = ctxs[0]->reps;
  int total = 0;
  for (int r : reps) total += r;
  if (n != total)
    return set_error(ST_ERR_INPUT, "connect_local: %d contexts for a %d-stage pipeline with %d stage contexts", n, N,
                     total);
  // stage-major, replica-minor order
  int i = 0;
  for (int k = 0; k < N; ++k)
    for (int r = 0; r < reps[k]; ++r, ++i) {
      st_ctx* c = ctxs[i];
      if (!c || c->k != k || c->N != N || c->replica != r || c->transport_kind != ST_TRANSPORT_LOCAL || c->reps != reps)
        return set_error(ST_ERR_INPUT, "connect_local: context %d is not stage %d replica %d of a LOCAL %d-stage "
                         "pipeline (same replicas table)", i, k, r, N);
      if (c->B_global != ctxs[0]->B_global) return set_error(ST_ERR_SHAPE, "connect_local: batch mismatch");
      if (k > 0 && ctxs[i - 1 - r]->out_last != c->in_first)
        return set_error(ST_ERR_SHAPE, "connect_local: cut width mismatch between stages %d and %d", k - 1, k);
    }
  auto link = make_local_link(N, reps);
  i = 0;
  for (int k = 0; k < N; ++k) {
    std::shared_ptr<ReplicaGroup> group = reps[k] > 1 ? make_replica_group(reps[k], link) : nullptr;
    for (int r = 0; r < reps[k]; ++r, ++i) {
      st_ctx* c = ctxs[i];
      ST_CUDA_TRY(cudaSetDevice(c->device));
      st_status e;
      c->tp = make_local_transport(link, k, c->ring_fwd, c->ring_bwd, c->ring_fwd_elems, c->ring_bwd_elems,
                                   c->replica, c->rep_prev, c->rep_self, c->rep_next, &e);
      if (e != ST_OK) return e;
      c->link = link;
      c->rgroup = group;
    }
  }
  return ST_OK;
}

void ctx_destroy(st_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& p : c->prof.pairs) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : c->prof.pool) cudaEventDestroy(e);
  if (c->side) {
    cudaStreamSynchronize(c->side);
    cudaStreamDestroy(c->side);
  }
  for (auto e : c->side_events) cudaEventDestroy(e);
  if (c->comm_fwd) cudaStreamSynchronize(c->comm_fwd);
  if (c->comm_bwd) cudaStreamSynchronize(c->comm_bwd);
  c->tp.reset();  // communicators before the streams they used
  p2p_free(c);
  for (int b = 0; b < 2; ++b)
    for (cudaEvent_t e : {c->ev_sent_fwd[b], c->ev_sent_bwd[b], c->ev_recv_bwd[b], c->ev_bwd_ring[b], c->ev_join[b]})
      if (e) cudaEventDestroy(e);
  for (auto e : c->ev_recv_fwd)
    if (e) cudaEventDestroy(e);
  for (auto e : c->ev_bwd_slot)
    if (e) cudaEventDestroy(e);
  if (c->ev_fwd_done) cudaEventDestroy(c->ev_fwd_done);
  if (c->ev_dx_ready) cudaEventDestroy(c->ev_dx_ready);
  if (c->own_comm_fwd) cudaStreamDestroy(c->comm_fwd);
  if (c->own_comm_bwd) cudaStreamDestroy(c->comm_bwd);
  delete c;
}

st_status ctx_set_params(st_ctx* c, const float* host, size_t n) {
  if (!c || (!host && n)) return set_error(ST_ERR_INPUT, "NULL argument");
  if ((int64_t)n != c->P) return set_error(ST_ERR_SHAPE, "set_params: n = %zu but stage has %lld", n, (long long)c->P);
  ST_CUDA_TRY(cudaSetDevice(c->device));
  // host or device memory (UVA): a model too large to stage on the host is uploaded layer by layer
  if (n) ST_CUDA_TRY(cudaMemcpyAsync(c->W, host, n * 4, cudaMemcpyDefault, c->stream));
  ST_CUDA_TRY(cudaMemsetAsync(c->V, 0, n * 4, c->stream));
  if (c->WF_out) ST_CUDA_TRY(cudaMemcpyAsync(c->WF_out, c->W, n * 4, cudaMemcpyDeviceToDevice, c->stream));
  for (int slot = 0; c->wstash && slot < c->S; ++slot)  // every in-flight forward before the first update sees W0
    ST_CUDA_TRY(cudaMemcpyAsync(c->wstash + (size_t)slot * stash_pitch(c->P), c->W, n * 4, cudaMemcpyDeviceToDevice, c->stream));
  if (c->WB_out) ST_CUDA_TRY(cudaMemcpyAsync(c->WB_out, c->W, n * 4, cudaMemcpyDeviceToDevice, c->stream));
  ST_CUDA_TRY(cudaMemsetAsync(c->losses_dev, 0xff, (size_t)c->max_mb * 4, c->stream));
  ST_CUDA_TRY(cudaStreamSynchronize(c->stream));
  c->version = 0;
  c->trace.clear();
  begin_session(c, c->max_mb);
  return ST_OK;
}

st_status ctx_get_params(st_ctx* c, float* W, float* V, size_t n, int64_t* version) {
  if (!c) return set_error(ST_ERR_INPUT, "NULL context");
  if ((W || V) && (int64_t)n != c->P)
    return set_error(ST_ERR_SHAPE, "get_params: n = %zu but stage has %lld", n, (long long)c->P);
  ST_CUDA_TRY(cudaSetDevice(c->device));
  ST_TRY(ctx_wait(c));
  if (W) ST_CUDA_TRY(cudaMemcpy(W, c->W, n * 4, cudaMemcpyDeviceToHost));
  if (V) ST_CUDA_TRY(cudaMemcpy(V, c->V, n * 4, cudaMemcpyDeviceToHost));
  if (version) *version = c->version;
  return ST_OK;
}

// ---- communication --------------------------------------------------------------
//
// Every message is one op on the comm stream of its direction (comm_fwd: activations,
// comm_bwd: gradients), issued in comm-plan order (schedule.cpp build_comm_plan) and
// ordered against the compute stream by events:
//   send_fwd(i): waits for F(i) (ev_fwd_done), sends send_fwd2[i % 2]; F(i + 2) waits
//                for it before overwriting that slot;
//   send_bwd(j): waits for B(j)'s layer-0 dX only (ev_dx_ready), so the transfer
//                overlaps that layer's dW + update; B(j + 2) waits before overwriting;
//   recv_fwd(i): into stash slot i % S once B(i − S), its previous reader, finished;
//                F(i) waits for it;
//   recv_bwd(j): into recv_bwd2[j % 2] once B(j − 2) finished; B(j) waits for it.
// NCCL receives are posted eagerly (after the previous task), so data arrives while
// the current task computes; LOCAL receives block the host until the peer's send is
// enqueued and are therefore issued right before the task that needs them.

// one message: device buffer + element count
struct CommOp {
  int kind;
  int64_t mb;
  float* buf;
  size_t count;
};

static CommOp comm_op(st_ctx* c, int kind, int64_t mb) {
  const size_t nin = (size_t)c->R * c->in_first, nout = (size_t)c->R * c->out_last;
  switch (kind) {
    case CK_SEND_FWD: return {kind, mb, c->send_fwd2[mb % 2], nout};
    case CK_RECV_FWD:
      return {kind, mb, c->stash + (size_t)(mb % c->S) * c->slot_elems + c->layers[0].stash_off, nin};
    case CK_SEND_BWD: return {kind, mb, c->send_bwd2[mb % 2], nin};
    default: return {kind, mb, c->recv_bwd2[mb % 2], nout};
  }
}

// one message to / from a neighbour — split into row slices, one per replica, when that
// neighbour is a replicated stage (hybrid DP × PP); chan = the replica of the
// replicated side of the channel
static st_status move(st_ctx* c, const CommOp& o, cudaStream_t cs) {
  const bool to_next = o.kind == CK_SEND_FWD || o.kind == CK_RECV_BWD;
  const int nrep = to_next ? c->rep_next : c->rep_prev;
  const bool send = o.kind == CK_SEND_FWD || o.kind == CK_SEND_BWD;
  if (nrep <= 1) {
    const int chan = c->rep_self > 1 ? c->replica : 0;
    return send ? c->tp->send(o.kind, o.mb, o.buf, o.count, cs, chan) : c->tp->recv(o.kind, o.mb, o.buf, o.count, cs, chan);
  }
  const size_t part = o.count / (size_t)nrep;  // rows split evenly (B divisible by the replica count)
  ST_TRY(c->tp->group_begin());
  for (int r = 0; r < nrep; ++r) {
    const st_status e = send ? c->tp->send(o.kind, o.mb, o.buf + r * part, part, cs, r)
                             : c->tp->recv(o.kind, o.mb, o.buf + r * part, part, cs, r);
    if (e != ST_OK) {
      c->tp->group_end();
      return e;
    }
  }
  return c->tp->group_end();
}

static st_status issue_op(st_ctx* c, const CommGroup& g) {
  if (!c->tp) return set_error(ST_ERR_STATE, "stage %d: transport not connected", c->k);
  for (int i = 0; i < g.n_ops; ++i) {
    const CommOp o = comm_op(c, g.kind[i], g.mb[i]);
    const bool fwd = o.kind == CK_SEND_FWD || o.kind == CK_RECV_FWD;
    cudaStream_t cs = fwd ? c->comm_fwd : c->comm_bwd;
    const int b = (int)(o.mb % 2);
    const size_t slot = (size_t)(o.mb % c->S);
    switch (o.kind) {
      case CK_SEND_FWD: ST_CUDA_TRY(cudaStreamWaitEvent(cs, c->ev_fwd_done, 0)); break;
      case CK_SEND_BWD: ST_CUDA_TRY(cudaStreamWaitEvent(cs, c->ev_dx_ready, 0)); break;
      case CK_RECV_FWD:
        if (c->bwd_slot_done[slot]) ST_CUDA_TRY(cudaStreamWaitEvent(cs, c->ev_bwd_slot[slot], 0));
        break;
      default:
        if (c->bwd_ring_done[b]) ST_CUDA_TRY(cudaStreamWaitEvent(cs, c->ev_bwd_ring[b], 0));
    }
    {
      Timed t(c, KC_COMM, cs);
      static const char* names[4] = {"stage %d send_fwd(%lld)", "stage %d recv_fwd(%lld)", "stage %d send_bwd(%lld)",
                                     "stage %d recv_bwd(%lld)"};
      NvtxRange range(names[o.kind & 3], c->k, (long long)o.mb);
      ST_TRY(move(c, o, cs));
    }
    switch (o.kind) {
      case CK_SEND_FWD:
        ST_CUDA_TRY(cudaEventRecord(c->ev_sent_fwd[b], cs));
        c->sent_fwd_pending[b] = true;
        break;
      case CK_SEND_BWD:
        ST_CUDA_TRY(cudaEventRecord(c->ev_sent_bwd[b], cs));
        c->sent_bwd_pending[b] = true;
        break;
      case CK_RECV_FWD: ST_CUDA_TRY(cudaEventRecord(c->ev_recv_fwd[slot], cs)); break;
      default: ST_CUDA_TRY(cudaEventRecord(c->ev_recv_bwd[b], cs));
    }
  }
  return ST_OK;
}

static bool eager_recvs(st_ctx* c) { return c->transport_kind == ST_TRANSPORT_NCCL; }

// Before task n: every op the plan places before it (its receive, and — LOCAL — the
// previous task's send).
static st_status comm_before_task(st_ctx* c, size_t n) {
  while (c->plan_next < c->plan.size() && (size_t)c->plan[c->plan_next].before_op <= n)
    ST_TRY(issue_op(c, c->plan[c->plan_next++]));
  return ST_OK;
}

// After task n: its send; NCCL also posts the next task's receive right away.
static st_status comm_after_task(st_ctx* c, size_t n) {
  while (c->plan_next < c->plan.size()) {
    const CommGroup& g = c->plan[c->plan_next];
    if ((size_t)g.before_op > n + 1) break;
    const bool is_recv = g.kind[0] == CK_RECV_FWD || g.kind[0] == CK_RECV_BWD;
    if ((size_t)g.before_op == n + 1 && is_recv && !eager_recvs(c)) break;
    ST_TRY(issue_op(c, g));
    c->plan_next++;
  }
  return ST_OK;
}

// The comm streams' work so far becomes part of the compute stream (session end, sync).
static st_status join_comm(st_ctx* c) {
  if (!c->tp) return ST_OK;
  ST_CUDA_TRY(cudaEventRecord(c->ev_join[0], c->comm_fwd));
  ST_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_join[0], 0));
  ST_CUDA_TRY(cudaEventRecord(c->ev_join[1], c->comm_bwd));
  ST_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_join[1], 0));
  return ST_OK;
}

// Host wait for the compute stream that cannot hang on a dead peer: polls the stream and
// the transport's asynchronous error state; a failure or no completion within
// comm_timeout_s aborts the transport (NCCL: ncclCommAbort on both communicators) and
// returns ST_ERR_NCCL (ST_ERR_STATE for a failed LOCAL peer).
st_status ctx_wait(st_ctx* c) {
  ST_TRY(join_comm(c));
  if (!c->tp) {
    ST_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return ST_OK;
  }
  const auto t0 = std::chrono::steady_clock::now();
  int sleep_us = 2;
  for (;;) {
    const cudaError_t q = cudaStreamQuery(c->stream);
    if (q == cudaSuccess) return c->p2p ? p2p_check(c) : ST_OK;
    if (q != cudaErrorNotReady) return set_error(ST_ERR_CUDA, "stage %d: %s", c->k, cudaGetErrorString(q));
    const st_status e = c->tp->poll();
    if (e != ST_OK) {
      const std::string msg = st_last_error();
      c->tp->abort();
      return set_error(e, "%s", msg.c_str());
    }
    const double waited = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (waited > c->comm_timeout_s) {
      const bool trace = getenv("ST_P2P_TRACE") != nullptr;
      if (trace) fprintf(stderr, "[st] stage %d: wait timed out after %.1f s, aborting\n", c->k, waited);
      c->tp->abort();
      if (trace) fprintf(stderr, "[st] stage %d: aborted, reading flags\n", c->k);
      const std::string flags = c->p2p ? p2p_describe(c) : std::string();
      if (trace) fprintf(stderr, "[st] stage %d: flags%s\n", c->k, flags.c_str());
      return set_error(c->transport_kind == ST_TRANSPORT_NCCL ? ST_ERR_NCCL : ST_ERR_STATE,
                       "stage %d: no completion after %.0f s (ST_COMM_TIMEOUT_S): a peer stage is hung or gone; "
                       "transport aborted (program op %zu of %zu)%s",
                       c->k, waited, c->pc, c->program.size(), flags.c_str());
    }
    std::this_thread::sleep_for(std::chrono::microseconds(sleep_us));
    sleep_us = std::min(sleep_us * 2, 1000);
  }
}

// ---- tasks -----------------------------------------------------------------------

static GemmArgs gargs(st_ctx* c, const LayerInfo& L) {
  GemmArgs g;
  g.mode = c->gemm;
  g.B = (int)c->R;  // GEMM rows: batch · sequence length
  g.n_in = L.n_in;
  g.n_out = L.n_out;
  g.work = c->gemm_ws;
  g.work_bytes = gemm_workspace_bytes((int)c->gemm_rows_max, c->gemm_in_max, c->gemm_out_max);
  g.stream = c->stream;
  g.pdl = c->pdl_now;  // programmatic dependent launches for this task (see run_task)
  return g;
}

// layer input pointer inside a stash slot (aliases the previous LSTM layer's h_t rows)
static float* layer_in(st_ctx* c, float* slot, size_t l) {
  const LayerInfo& L = c->layers[l];
  if (L.stash_off >= 0) return slot + L.stash_off;
  const LayerInfo& P = c->layers[l - 1];
  return slot + P.h_off + (size_t)c->B * P.n_out;
}

static GemmArgs gargs_rows(st_ctx* c, int rows, int n_in, int n_out) {
  GemmArgs g;
  g.mode = c->gemm;
  g.B = rows;
  g.n_in = n_in;
  g.n_out = n_out;
  g.work = c->gemm_ws;
  g.work_bytes = gemm_workspace_bytes((int)c->gemm_rows_max, c->gemm_in_max, c->gemm_out_max);
  g.stream = c->stream;
  g.pdl = c->pdl_now;
  return g;
}

// LSTM forward over T steps (a8): Gx = X·W_ih + b for all steps in one GEMM, then per
// step the recurrent GEMM h_{t−1}·W_hh and the fused cell kernel.
static st_status lstm_forward(st_ctx* c, const LayerInfo& L, const float* Wh, const float* X, float* slot) {
  const int B = c->B, H = L.n_out, T = c->T;
  float* gates = slot + L.gates_off;
  float* cbuf = slot + L.c_off;
  float* hbuf = slot + L.h_off;
  {
    Timed t(c, KC_GEMM_FWD);
    ST_TRY(gemm_fwd(gargs_rows(c, (int)c->R, L.n_in, 4 * H), X, Wh + L.w_off, Wh + L.b_off, gates, 0));
    c->launches += gemm_last_launches();
  }
  ST_CUDA_TRY(cudaMemsetAsync(hbuf, 0, (size_t)B * H * 4, c->stream));          // h_{-1} = 0
  if (!c->shares_gpu) {
    // all T steps in one persistent launch (k_lstm_rec.cu); the per-step path below when the
    // shapes do not allow it. Not with co-located contexts: two cooperative grids filling
    // the GPU at once could each wait for SMs the other holds.
    Timed tt(c, KC_GEMM_FWD);
    const st_status r = lstm_rec_fwd(gargs_rows(c, B, H, 4 * H), B, H, T, Wh + L.whh_off, gates, hbuf, cbuf,
                                     c->lstm_hlo);
    if (r == ST_OK) {
      c->launches += 1;
      return ST_OK;
    }
    if (r != ST_ERR_UNSUPPORTED) return r;
  }
  ST_CUDA_TRY(cudaMemsetAsync(c->lstm_hlo, 0, (size_t)B * H * 4, c->stream));  // its tf32 lo
  for (int t = 0; t < T; ++t) {
    float* h_prev = hbuf + (size_t)t * B * H;
    // G_t = Gx_t + h_{t−1}·W_hh: the GEMM takes h_{t−1}'s lo from the previous cell step and
    // leaves its K-split partials to the cell kernel (two launches per step fewer)
    SplitPlan plan;
    {
      Timed tt(c, KC_GEMM_FWD);
      GemmArgs g = gargs_rows(c, B, H, 4 * H);
      g.act_lo = c->lstm_hlo;
      g.defer = &plan;
      g.pdl = c->pdl;
      ST_TRY(gemm_fwd(g, h_prev, Wh + L.whh_off, nullptr, c->lstm_rec, 0));
      c->launches += gemm_last_launches();
    }
    Timed tt(c, KC_LOSS);
    ST_TRY(launch_lstm_cell_fwd(gates + (size_t)t * B * 4 * H, c->lstm_rec, &plan,
                                t ? cbuf + (size_t)(t - 1) * B * H : nullptr, cbuf + (size_t)t * B * H,
                                hbuf + (size_t)(t + 1) * B * H, c->lstm_hlo, B, H, c->stream));
    c->launches += 1;
  }
  return ST_OK;
}

static st_status forward_compute(st_ctx* c, int64_t mb, const float* x_dev, const int32_t* y_dev, bool host_io,
                                 float* loss_host) {
  float* slot = c->stash + (size_t)(mb % c->S) * c->slot_elems;
  // Eq. 4 with s_F (aliases W when s_F = 0); weight stashing: this mini-batch's stash slot,
  // written with the current W by the update that preceded this forward (or W0)
  const float* Wh = c->wstash ? c->wstash + (size_t)(mb % c->S) * stash_pitch(c->P) : c->WF;
  if (c->first_stage) {
    if (!x_dev) return set_error(ST_ERR_INPUT, "stage 0 forward needs x");
    const size_t bytes = c->embed_first ? (size_t)c->R * 4 : (size_t)c->R * c->in_first * 4;
    ST_CUDA_TRY(cudaMemcpyAsync(slot + c->layers[0].stash_off, x_dev, bytes,
                                host_io ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, c->stream));
  }
  if (c->last_stage && host_io && y_dev) {
    ST_CUDA_TRY(cudaMemcpyAsync(c->y_stage, y_dev, (size_t)c->R * 4, cudaMemcpyHostToDevice, c->stream));
    y_dev = c->y_stage;
  }
  const size_t nl = c->layers.size();
  for (size_t l = 0; l < nl; ++l) {
    const LayerInfo& L = c->layers[l];
    TimedLayer tl(c, l, 0);
    const float* in = layer_in(c, slot, l);
    // where this layer's output goes: the next layer's input stash, or the stage output
    float* out = nullptr;
    const bool next_aliases = (l + 1 < nl) && c->layers[l + 1].stash_off < 0;
    if (l + 1 < nl && !next_aliases)
      out = slot + c->layers[l + 1].stash_off;
    else if (l + 1 == nl)
      out = c->last_stage ? c->logits : c->send_fwd;
    if (L.kind == ST_LAYER_CONV && tc_conv_ok(c->gemm, L.hw, L.hw, L.n_in, L.n_out)) {
      Timed t(c, KC_GEMM_FWD);  // implicit GEMM: the shifted windows come straight from `in`
      ST_TRY(tc_conv_fwd(gargs_rows(c, c->B, 9 * L.n_in, L.n_out), in, L.hw, L.hw, L.n_in, L.n_out, Wh + L.w_off,
                         L.bias ? Wh + L.b_off : nullptr, out, L.act == ST_ACT_RELU));
      c->launches += tc_last_launches();
    } else if (L.kind == ST_LAYER_CONV && tc_conv_small_ok(c->gemm, L.n_in, L.n_out)) {
      {
        Timed t(c, KC_LOSS);
        ST_TRY(launch_im2col_pad32(in, c->B, L.hw, L.hw, L.n_in, c->conv_col, c->stream));
        c->launches += 1;
      }
      Timed t(c, KC_GEMM_FWD);
      ST_TRY(tc_conv_small_fwd(gargs_rows(c, c->B, 9 * L.n_in, L.n_out), c->conv_col, L.hw, L.hw, L.n_in, L.n_out,
                               Wh + L.w_off, L.bias ? Wh + L.b_off : nullptr, out, L.act == ST_ACT_RELU));
      c->launches += tc_last_launches();
    } else if (L.kind == ST_LAYER_CONV) {
      const int P = c->B * L.hw * L.hw;
      {
        Timed t(c, KC_LOSS);
        ST_TRY(launch_im2col(in, c->B, L.hw, L.hw, L.n_in, c->conv_col, c->stream));
        c->launches += 1;
      }
      Timed t(c, KC_GEMM_FWD);
      ST_TRY(gemm_fwd(gargs_rows(c, P, 9 * L.n_in, L.n_out), c->conv_col, Wh + L.w_off,
                      L.bias ? Wh + L.b_off : nullptr, out, L.act == ST_ACT_RELU));
      c->launches += gemm_last_launches();
    } else if (L.kind == ST_LAYER_POOL) {
      Timed t(c, KC_LOSS);
      ST_TRY(launch_maxpool_fwd(in, c->B, L.hw, L.hw, L.n_in, out, c->stream));
      c->launches += 1;
    } else if (L.kind == ST_LAYER_EMBED) {
      Timed t(c, KC_LOSS);
      ST_TRY(launch_embed_gather(Wh + L.w_off, reinterpret_cast<const int32_t*>(in), (int)c->R, L.n_out, out,
                                 c->stream));
      c->launches += 1;
    } else if (L.kind == ST_LAYER_LSTM) {
      ST_TRY(lstm_forward(c, L, Wh, in, slot));
      if (out)  // stage output / a non-aliasing consumer: copy h_0..h_{T−1}
        ST_CUDA_TRY(cudaMemcpyAsync(out, slot + L.h_off + (size_t)c->B * L.n_out, (size_t)c->R * L.n_out * 4,
                                    cudaMemcpyDeviceToDevice, c->stream));
    } else {
      Timed t(c, KC_GEMM_FWD);
      ST_TRY(gemm_fwd(gargs(c, L), in, Wh + L.w_off, L.bias ? Wh + L.b_off : nullptr, out, L.act == ST_ACT_RELU));
      c->launches += gemm_last_launches();
    }
  }
  if (c->last_stage) {
    if (!y_dev) return set_error(ST_ERR_INPUT, "last stage forward needs y_dev");
    Timed t(c, KC_LOSS);
    ST_TRY(launch_softmax_ce(c->logits, y_dev, (int)c->R, c->out_last, c->rowloss, c->losses_dev + (mb % c->max_mb),
                             c->dlogits, c->stream));
    c->launches += 2;
    if (loss_host)
      ST_CUDA_TRY(cudaMemcpyAsync(loss_host, c->losses_dev + (mb % c->max_mb), 4, cudaMemcpyDeviceToHost, c->stream));
  }
  return ST_OK;
}

static UpdateArgs block_update(st_ctx* c, int64_t off, const UpdateConsts& k) {
  UpdateArgs u;
  u.W = c->W + off;
  u.V = c->V + off;
  u.WF = c->WF_out ? c->WF_out + off : nullptr;
  u.WB = c->WB_out ? c->WB_out + off : nullptr;
  u.c = k;
  return u;
}

// fused = true: each layer's dW GEMM applies the K-B update to its own weight and bias
// blocks in its epilogue (G never reaches HBM); the caller then only bumps the version.
// Safe per layer: dX_l (which reads WB_l) is issued before dW_l on the same stream and
// no later task of this backward touches layer l again.
// LSTM backward through time (a8). dOut [R × H]: gradient w.r.t. the layer output.
// Writes the layer's gradient block into G and, if D != NULL, dX = dG·W_ihᵀ into D.
static st_status lstm_backward(st_ctx* c, const LayerInfo& L, const float* Wh, const float* X, float* slot,
                               const float* dOut, float* D) {
  const int B = c->B, H = L.n_out, T = c->T;
  const float* gates = slot + L.gates_off;
  const float* cbuf = slot + L.c_off;
  const float* hbuf = slot + L.h_off;
  bool rec_done = false;
  if (!c->shares_gpu) {  // all T steps in one persistent launch (see lstm_forward)
    Timed tt(c, KC_GEMM_DX);
    const st_status r = lstm_rec_bwd(gargs_rows(c, B, H, 4 * H), B, H, T, Wh + L.whh_off, gates, cbuf, dOut,
                                     c->lstm_dG, c->lstm_dglo, c->lstm_dc);
    if (r == ST_OK) {
      c->launches += 1;
      rec_done = true;
    } else if (r != ST_ERR_UNSUPPORTED) {
      return r;
    }
  }
  SplitPlan plan;  // dh_next of the step after t (splits = 0: none at t = T−1)
  for (int t = rec_done ? -1 : T - 1; t >= 0; --t) {
    {
      Timed tt(c, KC_LOSS);
      ST_TRY(launch_lstm_cell_bwd(gates + (size_t)t * B * 4 * H, cbuf + (size_t)t * B * H,
                                  t ? cbuf + (size_t)(t - 1) * B * H : nullptr, dOut + (size_t)t * B * H,
                                  t < T - 1 ? c->lstm_dh : nullptr, &plan, c->lstm_dc, t == T - 1,
                                  c->lstm_dG + (size_t)t * B * 4 * H, t > 0 ? c->lstm_dglo : nullptr, B, H,
                                  c->stream));
      c->launches += 1;
    }
    if (t > 0) {  // dh_{t−1} = dG_t · W_hhᵀ (dG_t's lo from the cell, partials left to the next cell)
      Timed tt(c, KC_GEMM_DX);
      GemmArgs g = gargs_rows(c, B, H, 4 * H);
      g.act_lo = c->lstm_dglo;
      g.defer = &plan;
      g.pdl = c->pdl;
      ST_TRY(gemm_dx(g, c->lstm_dG + (size_t)t * B * 4 * H, Wh + L.whh_off, nullptr, c->lstm_dh));
      c->launches += gemm_last_launches();
    }
  }
  {
    Timed tt(c, KC_GEMM_DW);
    // g_W_ih = Xᵀ·dG (+ g_b = Σ dG); g_W_hh = H_prevᵀ·dG with H_prev = [0, h_0 .. h_{T−2}]
    ST_TRY(gemm_dw(gargs_rows(c, (int)c->R, L.n_in, 4 * H), X, c->lstm_dG, c->G + L.w_off, c->G + L.b_off));
    c->launches += gemm_last_launches();
    ST_TRY(gemm_dw(gargs_rows(c, (int)c->R, H, 4 * H), hbuf, c->lstm_dG, c->G + L.whh_off, nullptr));
    c->launches += gemm_last_launches();
  }
  if (D) {
    Timed tt(c, KC_GEMM_DX);
    ST_TRY(gemm_dx(gargs_rows(c, (int)c->R, L.n_in, 4 * H), c->lstm_dG, Wh + L.w_off, nullptr, D));
    c->launches += gemm_last_launches();
  }
  return ST_OK;
}

// fused = true: each layer's parameters are updated right after its gradient is
// known — inside the dW GEMM epilogue for TMA-friendly dense layers (G never reaches
// HBM), otherwise by a K-B launch over the layer block. Safe per layer: the layer's
// dX (which reads WB) is issued before its update on the same stream and no later
// task of this backward touches the layer again.
static st_status backward_compute(st_ctx* c, int64_t mb, bool fused = false) {
  const UpdateConsts kc = make_update_consts(c->lr, c->gamma, c->sF, c->sB, c->momentum);
  float* slot = c->stash + (size_t)(mb % c->S) * c->slot_elems;
  // Eq. 4 with s_B (D5: re-predicted from the current state); weight stashing: the
  // forward's copy. The update after this backward refills the same slot with W' for the
  // next forward, F(mb + N − k), which is the slot's next user.
  const float* Wh = c->wstash ? c->wstash + (size_t)(mb % c->S) * stash_pitch(c->P) : c->WB;
  if (c->wstash) c->WF_out = c->wstash + (size_t)(mb % c->S) * stash_pitch(c->P);
  const float* dZ = c->last_stage ? c->dlogits : c->recv_bwd;
  const int nl = (int)c->layers.size();
  // Gradient buffers rotate over 3 so that the dW + update of layer l (side stream,
  // reading dZ_l) can overlap the dX of layer l−1 (main stream, writing dZ_{l−2}).
  float* pp[3] = {c->bufA, c->bufB, c->bufC};
  int reader[3] = {-1, -1, -1};  // layer whose side-stream dW last read pp[i] (event index)
  int next = 0;
  bool side_busy = false;
  int64_t side_params = 0;  // parameters of the dW + update last issued on the side stream
  int side_dwu = c->dwu_sms;  // its SM budget
  auto join_side = [&]() -> st_status {
    if (!side_busy) return ST_OK;
    ST_CUDA_TRY(cudaEventRecord(c->side_events[nl], c->side));
    ST_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->side_events[nl], 0));
    side_busy = false;
    reader[0] = reader[1] = reader[2] = -1;
    return ST_OK;
  };
  for (int l = nl - 1; l >= 0; --l) {
    const LayerInfo& L = c->layers[l];
    TimedLayer tl(c, (size_t)l, 1);  // ST_PROF_LAYERS: the side stream is joined below, so
                                     // this bracket covers the layer's dW + update too
    // Programmatic dependent launches pay off on one in-order stream; for a large dense
    // layer the main-stream dX overlaps the side-stream dW + update, and early-launched
    // CTAs waiting on their predecessor hold SMs the other stream needs (large FCN −5%),
    // so those layers launch normally
    // — unless the layer's dW + update is serialised after its dX (≥ 2^27 parameters): then
    // one stream has the GPU again and the launches chain programmatically (ST_PDL_SERIAL)
    const bool serial_layer = fused && c->bwd_serial && c->pdl_serial && L.n_params >= ((int64_t)1 << 27);
    c->pdl_now = c->pdl_dense &&
                 (serial_layer || !(fused && L.kind == ST_LAYER_DENSE && L.n_params >= ((int64_t)1 << 22)));
    set_thread_pdl(c->pdl_now ? 1 : 0);
    float* Ain = layer_in(c, slot, (size_t)l);
    const bool need_dx = !(c->first_stage && l == 0) && L.kind != ST_LAYER_EMBED;
    // implicit convs and pools also overlap: a conv's dW + update runs on the side stream
    // while the next layers' dX / max-pool backward run on the main stream
    const bool conv_ov = c->conv_overlap && (L.kind == ST_LAYER_POOL ||
                                             (L.kind == ST_LAYER_CONV && tc_conv_ok(c->gemm, L.hw, L.hw, L.n_in, L.n_out)));
    const bool overlap = fused && (L.kind == ST_LAYER_DENSE || conv_ov);
    if (!overlap) ST_TRY(join_side());
    float* D = nullptr;
    int dslot = -1;
    if (need_dx) {
      if (l == 0) {
        D = c->send_bwd;
      } else {
        dslot = next;
        next = (next + 1) % 3;
        D = pp[dslot];
        if (reader[dslot] >= 0) {  // a side-stream dW still reads this buffer
          ST_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->side_events[reader[dslot]], 0));
          reader[dslot] = -1;
        }
      }
    }
    const int producer_act = (l > 0) ? c->layers[l - 1].act : c->prev_act;
    if (L.kind == ST_LAYER_POOL) {
      if (D) {
        Timed t(c, KC_LOSS);
        ST_TRY(launch_maxpool_bwd(Ain, dZ, c->B, L.hw, L.hw, L.n_in, producer_act == ST_ACT_RELU, D, c->stream));
        c->launches += 1;
      }
    } else if (L.kind == ST_LAYER_CONV && tc_conv_ok(c->gemm, L.hw, L.hw, L.n_in, L.n_out)) {
      // implicit GEMMs: dX = conv with the flipped kernel (ReLU mask of the producer of
      // Ain fused), then dW = Σ_p window(Ain)ᵀ dZ (+ bias gradient) into G
      if (D) {
        GemmArgs gx = gargs_rows(c, c->B, 9 * L.n_in, L.n_out);
        if (side_busy) gx.max_ctas = std::max(2, (c->sm_count - c->dwu_sms) & ~1);  // a conv dW is running on the side
        Timed t(c, KC_GEMM_DX);
        ST_TRY(tc_conv_dx(gx, dZ, L.hw, L.hw, L.n_in, L.n_out, Wh + L.w_off, producer_act == ST_ACT_RELU ? Ain : nullptr,
                          D));
        c->launches += tc_last_launches();
      }
      if (overlap) {
        // dW + bias gradient + K-B update on the side stream, after this layer's dX (which
        // reads WB_l); its own GEMM workspace; a CTA budget while more conv dX follow
        ST_CUDA_TRY(cudaEventRecord(c->side_events[l], c->stream));
        ST_CUDA_TRY(cudaStreamWaitEvent(c->side, c->side_events[l], 0));
        GemmArgs gw = gargs_rows(c, c->B, 9 * L.n_in, L.n_out);
        gw.stream = c->side;
        gw.work = c->gemm_ws2;
        bool more_dx = false;
        for (int q = l - 1; q >= 0 && !more_dx; --q)
          more_dx = c->layers[q].kind == ST_LAYER_CONV && !(c->first_stage && q == 0);
        if (more_dx) gw.max_ctas = c->dwu_sms;
        {
          Timed t(c, KC_GEMM_DW, c->side);
          ST_TRY(tc_conv_dw(gw, Ain, dZ, L.hw, L.hw, L.n_in, L.n_out, c->G + L.w_off, L.bias ? c->G + L.b_off : nullptr));
          c->launches += tc_last_launches();
          const UpdateArgs u = block_update(c, L.w_off, kc);
          ST_TRY(launch_update_predict(u.W, u.V, c->G + L.w_off, u.WF, u.WB, (size_t)L.n_params, kc, c->side));
          c->launches += 1;
        }
        ST_CUDA_TRY(cudaEventRecord(c->side_events[l], c->side));
        side_busy = true;
        side_params = L.n_params;
        for (int i = 0; i < 3; ++i)
          if (dZ == pp[i]) reader[i] = l;
      } else {
        Timed t(c, KC_GEMM_DW);
        ST_TRY(tc_conv_dw(gargs_rows(c, c->B, 9 * L.n_in, L.n_out), Ain, dZ, L.hw, L.hw, L.n_in, L.n_out,
                          c->G + L.w_off, L.bias ? c->G + L.b_off : nullptr));
        c->launches += tc_last_launches();
        if (fused) {  // K-B over the layer's weight + bias block (contiguous, S:106 layout)
          const UpdateArgs u = block_update(c, L.w_off, kc);
          ST_TRY(launch_update_predict(u.W, u.V, c->G + L.w_off, u.WF, u.WB, (size_t)L.n_params, kc, c->stream));
          c->launches += 1;
        }
      }
    } else if (L.kind == ST_LAYER_CONV && tc_conv_small_ok(c->gemm, L.n_in, L.n_out)) {
      const int P = c->B * L.hw * L.hw;
      if (D) {  // dcol = dZ·Wᵀ [P × 9·Cin], dX = col2im(dcol) ⊙ mask (9·Cin < 32: CUDA-core GEMM)
        Timed t(c, KC_GEMM_DX);
        ST_TRY(gemm_dx(gargs_rows(c, P, 9 * L.n_in, L.n_out), dZ, Wh + L.w_off, nullptr, c->conv_dcol));
        c->launches += gemm_last_launches();
        ST_TRY(launch_col2im(c->conv_dcol, c->B, L.hw, L.hw, L.n_in, producer_act == ST_ACT_RELU ? Ain : nullptr, D,
                             c->stream));
        c->launches += 1;
      }
      {
        Timed t(c, KC_LOSS);
        ST_TRY(launch_im2col_pad32(Ain, c->B, L.hw, L.hw, L.n_in, c->conv_col, c->stream));
        c->launches += 1;
      }
      Timed t(c, KC_GEMM_DW);
      ST_TRY(tc_conv_small_dw(gargs_rows(c, c->B, 9 * L.n_in, L.n_out), c->conv_col, dZ, L.hw, L.hw, L.n_in,
                              L.n_out, c->G + L.w_off, L.bias ? c->G + L.b_off : nullptr));
      c->launches += tc_last_launches();
      if (fused) {
        const UpdateArgs u = block_update(c, L.w_off, kc);
        ST_TRY(launch_update_predict(u.W, u.V, c->G + L.w_off, u.WF, u.WB, (size_t)L.n_params, kc, c->stream));
        c->launches += 1;
      }
    } else if (L.kind == ST_LAYER_CONV) {
      const int P = c->B * L.hw * L.hw;
      {
        Timed t(c, KC_LOSS);
        ST_TRY(launch_im2col(Ain, c->B, L.hw, L.hw, L.n_in, c->conv_col, c->stream));
        c->launches += 1;
      }
      if (D) {  // dcol = dZ·Wᵀ, dX = col2im(dcol) ⊙ ReLU mask of the producer of Ain
        Timed t(c, KC_GEMM_DX);
        ST_TRY(gemm_dx(gargs_rows(c, P, 9 * L.n_in, L.n_out), dZ, Wh + L.w_off, nullptr, c->conv_dcol));
        c->launches += gemm_last_launches();
        ST_TRY(launch_col2im(c->conv_dcol, c->B, L.hw, L.hw, L.n_in, producer_act == ST_ACT_RELU ? Ain : nullptr, D,
                             c->stream));
        c->launches += 1;
      }
      Timed t(c, KC_GEMM_DW);
      const GemmArgs gw = gargs_rows(c, P, 9 * L.n_in, L.n_out);
      if (fused) {
        UpdateArgs bu{};
        if (L.bias) bu = block_update(c, L.b_off, kc);
        ST_TRY(gemm_dw_update(gw, c->conv_col, dZ, block_update(c, L.w_off, kc), bu, c->G + L.w_off));
      } else {
        ST_TRY(gemm_dw(gw, c->conv_col, dZ, c->G + L.w_off, L.bias ? c->G + L.b_off : nullptr));
      }
      c->launches += gemm_last_launches();
    } else if (L.kind == ST_LAYER_EMBED) {
      Timed t(c, KC_GEMM_DW);
      ST_TRY(launch_embed_grad(dZ, reinterpret_cast<const int32_t*>(Ain), (int)c->R, L.n_in, L.n_out, c->G + L.w_off,
                               c->embed_scratch, c->stream));
      c->launches += 5;
    } else if (L.kind == ST_LAYER_LSTM) {
      ST_TRY(lstm_backward(c, L, Wh, Ain, slot, dZ, D));
    } else {
      if (D) {
        // ReLU mask of the layer that produced Ain (D12: ReLU'(0) = 0): 1[Z>0] == 1[ReLU(Z)>0]
        GemmArgs gx = gargs(c, L);
        // share the GPU with the running dW + update — unless that one is small (e.g. the
        // 10-wide output layer's), when this dX would otherwise run alone on part of the GPU
        if (side_busy && side_params >= (int64_t)1 << 22) gx.max_ctas = std::max(2, (c->sm_count - side_dwu) & ~1);
        Timed t(c, KC_GEMM_DX);
        ST_TRY(gemm_dx(gx, dZ, Wh + L.w_off, producer_act == ST_ACT_RELU ? Ain : nullptr, D));
        c->launches += gemm_last_launches();
      }
      if (fused && c->bwd_serial && L.n_params >= ((int64_t)1 << 27)) {
        // serialised: the dW + update of a very large layer (16384²: 268M parameters) takes
        // the whole GPU after its dX — alone it streams W / V at 0.95 of the HBM peak, so
        // running the next dX beside it cannot win (measured: large FCN 6264 overlapped vs
        // 6222 samples/s serialised, within clock noise; the update at 0.90 instead of 0.75
        // of the peak in the step); smaller layers stay overlapped (wide FCN: −2% serialised)
        ST_TRY(join_side());
        GemmArgs gw = gargs(c, L);
        UpdateArgs bu{};
        if (L.bias) bu = block_update(c, L.b_off, kc);
        Timed t(c, KC_GEMM_DW);
        ST_TRY(gemm_dw_update(gw, Ain, dZ, block_update(c, L.w_off, kc), bu, c->G + L.w_off));
        c->launches += gemm_last_launches();
      } else if (fused) {
        // dW + update on the side stream, after this layer's dX (which reads WB_l)
        ST_CUDA_TRY(cudaEventRecord(c->side_events[l], c->stream));
        ST_CUDA_TRY(cudaStreamWaitEvent(c->side, c->side_events[l], 0));
        GemmArgs gw = gargs(c, L);
        gw.stream = c->side;
        gw.work = c->gemm_ws2;
        // a dX of layer l−1 will run concurrently only if that layer is DENSE and needs one
        const bool more_dx = l > 0 && c->layers[l - 1].kind == ST_LAYER_DENSE && !(c->first_stage && l == 1);
        // SM budget of the overlapped dW + update: 80 (swept on 8192-wide layers); a layer
        // with 100–140 output tiles gets one CTA per tile, so every CTA owns a whole m-tile
        // column (no dZ re-staging, adjacent W / V rows streamed together): 16384-wide
        // layers 80 → 128 CTAs, large FCN 5.2k → 5.9k samples/s. ST_DWU_SMS overrides.
        const int m_tiles = (L.n_out + 127) / 128;
        side_dwu = c->dwu_env ? c->dwu_sms : ((m_tiles >= 100 && m_tiles <= c->sm_count - 8) ? m_tiles : c->dwu_sms);
        if (more_dx) gw.max_ctas = side_dwu;
        UpdateArgs bu{};
        if (L.bias) bu = block_update(c, L.b_off, kc);
        {
          Timed t(c, KC_GEMM_DW, c->side);
          ST_TRY(gemm_dw_update(gw, Ain, dZ, block_update(c, L.w_off, kc), bu, c->G + L.w_off));
        }
        c->launches += gemm_last_launches();
        ST_CUDA_TRY(cudaEventRecord(c->side_events[l], c->side));
        side_busy = true;
        side_params = L.n_params;
        for (int i = 0; i < 3; ++i)
          if (dZ == pp[i]) reader[i] = l;
      } else {
        Timed t(c, KC_GEMM_DW);
        ST_TRY(gemm_dw(gargs(c, L), Ain, dZ, c->G + L.w_off, L.bias ? c->G + L.b_off : nullptr));
        c->launches += gemm_last_launches();
      }
    }
    if (fused && (L.kind == ST_LAYER_EMBED || L.kind == ST_LAYER_LSTM)) {
      Timed t(c, KC_UPDATE);
      UpdateArgs u = block_update(c, L.w_off, kc);
      ST_TRY(launch_update_predict(u.W, u.V, c->G + L.w_off, u.WF, u.WB, (size_t)L.n_params, kc, c->stream));
      c->launches += 1;
    }
    // the layer-0 dX is the message to stage k−1: its send may start now, overlapping
    // this layer's dW + update on the side stream
    if (l == 0 && D && !c->first_stage) {
      if (c->p2p)
        ST_TRY(p2p_after_dx(c, mb));  // the gradient is in stage k−1's ring slot
      else
        ST_CUDA_TRY(cudaEventRecord(c->ev_dx_ready, c->stream));
    }
    if (D) dZ = D;
    if (c->prof.layers) ST_TRY(join_side());  // per-layer profile: no cross-layer overlap
  }
  ST_TRY(join_side());
  return ST_OK;
}

static st_status run_task(st_ctx* c, const float* x_dev, const int32_t* y_dev, bool host_io = false,
                          float* loss_host = nullptr, bool fused_update = false) {
  if (c->pc >= c->program.size()) return set_error(ST_ERR_STATE, "stage %d: program finished", c->k);
  if (c->pending_update)
    return set_error(ST_ERR_STATE, "stage %d: predict_and_update must follow every backward", c->k);
  const Task t = c->program[c->pc];
  NvtxRange range(t.dir == ST_FWD ? "stage %d F(%lld)" : "stage %d B(%lld)", c->k, (long long)t.mb);
  // programmatic dependent launches for this task (the backward refines it per layer)
  c->pdl_now = c->pdl_dense;
  set_thread_pdl(c->pdl_now ? 1 : 0);
  const bool p2p = c->p2p != nullptr;  // no comm plan: the GEMMs write the peer buffers
  if (!p2p) ST_TRY(comm_before_task(c, c->pc));
  st_event e{};
  e.stage = c->k;
  e.op_idx = (int32_t)c->trace.size();
  e.dir = t.dir;
  e.mb = t.mb;
  e.base_version = c->version;
  if (c->wstash) {  // the backward records the version its forward used (the stashed copy)
    if (t.dir == ST_FWD) c->stash_ver[(size_t)(t.mb % c->S)] = c->version;
    else e.base_version = c->stash_ver[(size_t)(t.mb % c->S)];
  }
  e.s = t.dir == ST_FWD ? c->sF : c->sB;
  e.target = e.base_version + e.s;
  c->trace.push_back(e);
  const int b = (int)(t.mb % 2);
  const size_t slot = (size_t)(t.mb % c->S);
  if (t.dir == ST_FWD) {
    if (p2p) {
      ST_TRY(p2p_before_forward(c, t.mb));  // input landed; output = the peer's stash slot
    } else {
      if (!c->first_stage) ST_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_recv_fwd[slot], 0));  // input arrived
      if (!c->last_stage) {  // the output slot's previous send (mb − 2) has left
        if (c->sent_fwd_pending[b]) ST_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_sent_fwd[b], 0));
        c->send_fwd = c->send_fwd2[b];
      }
    }
    ST_TRY(forward_compute(c, t.mb, x_dev, y_dev, host_io, loss_host));
    if (p2p)
      ST_TRY(p2p_after_forward(c, t.mb));
    else if (!c->last_stage)
      ST_CUDA_TRY(cudaEventRecord(c->ev_fwd_done, c->stream));
  } else {
    if (p2p) {
      ST_TRY(p2p_before_backward(c, t.mb));  // gradient landed; layer-0 dX = the peer's ring slot
    } else {
      if (!c->last_stage) {  // the gradient from k+1 arrived
        ST_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_recv_bwd[b], 0));
        c->recv_bwd = c->recv_bwd2[b];
      }
      if (!c->first_stage) {
        if (c->sent_bwd_pending[b]) ST_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_sent_bwd[b], 0));
        c->send_bwd = c->send_bwd2[b];
      }
    }
    // a replicated stage (hybrid DP × PP): G of this replica's rows, summed over the
    // replicas, then the same K-B update on every replica
    const bool replicated = c->rep_self > 1;
    ST_TRY(backward_compute(c, t.mb, fused_update && !replicated));
    if (replicated) {
      Timed tc(c, KC_COMM);
      if (c->rgroup)
        ST_TRY(replica_reduce_local(c->rgroup.get(), c->replica, c->G, (size_t)c->P, c->stream));
      else if (c->tp)
        ST_TRY(c->tp->allreduce_sum(c->G, (size_t)c->P, c->stream));
      else
        return set_error(ST_ERR_STATE, "stage %d replica %d: transport not connected", c->k, c->replica);
    }
    if (p2p) ST_TRY(p2p_after_backward(c, t.mb));
    // this backward's readers are done with its stash slot and its gradient slot
    ST_CUDA_TRY(cudaEventRecord(c->ev_bwd_slot[slot], c->stream));
    c->bwd_slot_done[slot] = 1;
    ST_CUDA_TRY(cudaEventRecord(c->ev_bwd_ring[b], c->stream));
    c->bwd_ring_done[b] = true;
    for (size_t i = 0; i < c->marks.size();) {  // st_record_after_backward
      if (c->marks[i].first == t.mb) {
        ST_CUDA_TRY(record_timing_event(c, c->marks[i].second, c->stream));
        c->marks.erase(c->marks.begin() + (long)i);
      } else {
        ++i;
      }
    }
    if (fused_update && replicated) {
      const UpdateConsts kc = make_update_consts(c->lr, c->gamma, c->sF, c->sB, c->momentum);
      Timed tu(c, KC_UPDATE);
      ST_TRY(launch_update_predict(c->W, c->V, c->G, c->WF_out, c->WB_out, (size_t)c->P, kc, c->stream));
      c->launches += 1;
      c->version += 1;
    } else if (fused_update) {
      c->version += 1;  // the update already ran inside the dW epilogues
    } else {
      c->pending_update = true;
    }
  }
  if (!p2p) ST_TRY(comm_after_task(c, c->pc));
  c->pc++;
  return ST_OK;
}

st_status ctx_update(st_ctx* c) {
  NvtxRange range("stage %d update(v%lld)", c->k, (long long)c->version);
  if (!c->pending_update) return set_error(ST_ERR_STATE, "stage %d: no backward pending", c->k);
  const UpdateConsts k = make_update_consts(c->lr, c->gamma, c->sF, c->sB, c->momentum);
  {
    Timed t(c, KC_UPDATE);
    ST_TRY(launch_update_predict(c->W, c->V, c->G, c->WF_out, c->WB_out, (size_t)c->P, k, c->stream));
  }
  c->launches += 1;
  c->version += 1;
  c->pending_update = false;
  return ST_OK;
}

static st_status expect(st_ctx* c, int dir, int64_t mb) {
  if (c->pc >= c->program.size())
    return set_error(ST_ERR_STATE, "stage %d: program of %lld mini-batches finished", c->k, (long long)c->session_M);
  const Task& t = c->program[c->pc];
  if (t.dir != dir || t.mb != mb)
    return set_error(ST_ERR_STATE, "stage %d: next op is %c(%lld), not %c(%lld)", c->k, t.dir == ST_FWD ? 'F' : 'B',
                     (long long)t.mb, dir == ST_FWD ? 'F' : 'B', (long long)mb);
  return ST_OK;
}

st_status ctx_forward(st_ctx* c, int64_t mb, const float* x_dev, const int32_t* y_dev, float* loss_host) {
  ST_CUDA_TRY(cudaSetDevice(c->device));
  ST_TRY(expect(c, ST_FWD, mb));
  ST_TRY(run_task(c, x_dev, y_dev));
  if (loss_host && c->last_stage) {
    ST_CUDA_TRY(cudaMemcpyAsync(loss_host, c->losses_dev + (mb % c->max_mb), 4, cudaMemcpyDeviceToHost, c->stream));
    ST_TRY(ctx_wait(c));
    if (!std::isfinite(*loss_host))
      return set_error(ST_ERR_DIVERGED, "non-finite loss at mini-batch %lld", (long long)mb);
  }
  return ST_OK;
}

st_status ctx_backward(st_ctx* c, int64_t mb) {
  ST_CUDA_TRY(cudaSetDevice(c->device));
  ST_TRY(expect(c, ST_BWD, mb));
  return run_task(c, nullptr, nullptr);
}

st_status ctx_predict_and_update(st_ctx* c) {
  ST_CUDA_TRY(cudaSetDevice(c->device));
  return ctx_update(c);
}

static const float* x_of(st_ctx* c, const float* xs, int64_t mb) {
  // a replica of a replicated first stage reads its row slice of each mini-batch
  const size_t w = c->embed_first ? 1 : (size_t)c->in_first;
  return (c->first_stage && xs) ? xs + ((size_t)mb * c->B_global * c->T + (size_t)c->replica * c->R) * w : nullptr;
}
static const int32_t* y_of(st_ctx* c, const int32_t* ys, int64_t mb) {
  return (c->last_stage && ys) ? ys + (size_t)mb * c->R : nullptr;
}

st_status ctx_step(st_ctx* c, const float* x_dev, const int32_t* y_dev, st_step_info* info) {
  ST_CUDA_TRY(cudaSetDevice(c->device));
  st_step_info z{0, -1, -1, 0, NAN};
  if (c->pending_update) return set_error(ST_ERR_STATE, "stage %d: pending update", c->k);
  if (c->pc >= c->program.size()) {
    z.done = 1;
    if (info) *info = z;
    return ST_OK;
  }
  const Task t = c->program[c->pc];
  if (t.dir == ST_FWD) {
    ST_TRY(run_task(c, x_dev, y_dev));
    z.ops_run++;
    z.ran_forward = (int32_t)t.mb;
    if (c->last_stage) {
      ST_CUDA_TRY(cudaMemcpyAsync(&z.loss, c->losses_dev + (t.mb % c->max_mb), 4, cudaMemcpyDeviceToHost, c->stream));
      ST_TRY(ctx_wait(c));
    }
  }
  // a warm-up F is followed by another F; a steady F by its paired B; cooldown is B alone
  if (c->pc < c->program.size() && c->program[c->pc].dir == ST_BWD) {
    const Task b = c->program[c->pc];
    ST_TRY(run_task(c, nullptr, nullptr, false, nullptr, true));
    z.ops_run += 2;
    z.ran_backward = (int32_t)b.mb;
  }
  z.done = c->pc >= c->program.size();
  if (info) *info = z;
  return ST_OK;
}

st_status ctx_run(st_ctx* c, int64_t M, const float* xs, const int32_t* ys, float* losses_host, bool host_io) {
  ST_CUDA_TRY(cudaSetDevice(c->device));
  if (M < 0 || M > c->max_mb)
    return set_error(ST_ERR_INPUT, "run: M = %lld outside [0, max_minibatches = %lld]", (long long)M,
                     (long long)c->max_mb);
  if (c->pc != 0 && c->pc != c->program.size())
    return set_error(ST_ERR_STATE, "run: stage %d is in the middle of a program (op %zu of %zu)", c->k, c->pc,
                     c->program.size());
  if (c->pending_update) return set_error(ST_ERR_STATE, "run: pending update");
  if (c->first_stage && M > 0 && !xs) return set_error(ST_ERR_INPUT, "run: stage 0 needs xs_dev");
  if (c->last_stage && M > 0 && !ys) return set_error(ST_ERR_INPUT, "run: last stage needs ys_dev");
  begin_session(c, M);
  // graph mode (st_set_graph_mode): the whole session is captured into one CUDA graph and
  // launched once — every kernel, copy, event and NCCL call of the session becomes a node,
  // so the GPU runs them back to back without a host launch per kernel (latency-bound
  // configs). The host bookkeeping (program, trace, versions) runs during the capture.
  const bool graph = c->graph_mode && !c->link;  // LOCAL groups block on host channels: eager
  if (graph) {
    ST_CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    c->capturing = true;
    // fork the auxiliary streams into the capture before any of them is used
    ST_CUDA_TRY(cudaEventRecord(c->ev_join[0], c->stream));
    for (cudaStream_t s2 : {c->side, c->comm_fwd, c->comm_bwd})
      if (s2 != c->stream) ST_CUDA_TRY(cudaStreamWaitEvent(s2, c->ev_join[0], 0));
  }
  st_status run_err = ST_OK;
  while (run_err == ST_OK && c->pc < c->program.size()) {
    const Task t = c->program[c->pc];
    float* lh = (host_io && losses_host && c->last_stage && t.dir == ST_FWD) ? losses_host + t.mb : nullptr;
    run_err = run_task(c, x_of(c, xs, t.mb), y_of(c, ys, t.mb), host_io, lh, true);
  }
  // the session's last transfers become part of the compute stream
  if (run_err == ST_OK) run_err = join_comm(c);
  if (graph) {
    if (run_err == ST_OK) {  // the side stream's last work joins too (every layer's update)
      ST_CUDA_TRY(cudaEventRecord(c->ev_join[1], c->side));
      ST_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_join[1], 0));
    }
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    c->capturing = false;
    if (run_err != ST_OK) {
      if (g) cudaGraphDestroy(g);
      return run_err;
    }
    if (e != cudaSuccess) return set_error(ST_ERR_CUDA, "stage %d: graph capture: %s", c->k, cudaGetErrorString(e));
    cudaGraphExec_t x = nullptr;
    const cudaError_t ei = cudaGraphInstantiate(&x, g, 0);
    cudaGraphDestroy(g);
    if (ei != cudaSuccess) return set_error(ST_ERR_CUDA, "stage %d: graph instantiate: %s", c->k, cudaGetErrorString(ei));
    const cudaError_t el = cudaGraphLaunch(x, c->stream);
    cudaGraphExecDestroy(x);  // released once the launch completes
    if (el != cudaSuccess) return set_error(ST_ERR_CUDA, "stage %d: graph launch: %s", c->k, cudaGetErrorString(el));
    c->graph_sessions += 1;
  }
  ST_TRY(run_err);
  const bool want_losses = losses_host && c->last_stage && M > 0;
  // host buffers (st_run_host) are read by asynchronous copies: never return before they
  // finish; the wait polls the transport (a hung peer surfaces as an error after
  // ST_COMM_TIMEOUT_S), so the losses are copied only once the stream is idle
  if (want_losses || host_io) ST_TRY(ctx_wait(c));
  if (want_losses && !host_io)
    ST_CUDA_TRY(cudaMemcpy(losses_host, c->losses_dev, (size_t)M * 4, cudaMemcpyDeviceToHost));
  if (want_losses)
    for (int64_t i = 0; i < M; ++i)
      if (!std::isfinite(losses_host[i]))
        return set_error(ST_ERR_DIVERGED, "non-finite loss at mini-batch %lld", (long long)i);
  return ST_OK;
}

st_status ctx_mark_after_backward(st_ctx* c, int64_t mb, void* event) {
  if (!event) return set_error(ST_ERR_INPUT, "record_after_backward: event is NULL");
  if (mb < 0) return set_error(ST_ERR_INPUT, "record_after_backward: mb must be >= 0");
  if (c->marks.size() >= 64) return set_error(ST_ERR_INPUT, "record_after_backward: more than 64 pending marks");
  c->marks.push_back({mb, static_cast<cudaEvent_t>(event)});
  return ST_OK;
}

st_status ctx_run_group(st_ctx** ctxs, int n, int64_t M, const float* xs, const int32_t* ys, float* losses_host) {
  if (!ctxs || n < 1) return set_error(ST_ERR_INPUT, "run_group: no contexts");
  std::vector<st_status> res(n, ST_OK);
  std::vector<std::string> msg(n);
  std::vector<std::thread> th;
  for (int k = 0; k < n; ++k) {
    th.emplace_back([&, k] {
      st_ctx* c = ctxs[k];
      try {
        cudaSetDevice(c->device);
        res[k] = ctx_run(c, M, c->first_stage ? xs : nullptr, c->last_stage ? ys : nullptr,
                         c->last_stage ? losses_host : nullptr, false);
        if (res[k] != ST_OK) msg[k] = st_last_error();
      } catch (const std::exception& e) {
        res[k] = ST_ERR_STATE;
        msg[k] = std::string("internal exception: ") + e.what();
      } catch (...) {
        res[k] = ST_ERR_STATE;
        msg[k] = "internal exception";
      }
      // a failed stage releases its peers at once instead of leaving them to time out
      if (res[k] != ST_OK && c->tp) c->tp->abort();
    });
  }
  for (auto& t : th) t.join();
  // report the root cause: a stage that failed on its own, not one released by the abort
  for (int k = 0; k < n; ++k)
    if (res[k] != ST_OK && msg[k].find("a peer stage failed") == std::string::npos)
      return set_error(res[k], "stage %d: %s", k, msg[k].c_str());
  for (int k = 0; k < n; ++k)
    if (res[k] != ST_OK) return set_error(res[k], "stage %d: %s", k, msg[k].c_str());
  return ST_OK;
}

st_status ctx_get_trace(st_ctx* c, st_event* out, size_t cap, size_t* n) {
  if (!c || !n) return set_error(ST_ERR_INPUT, "NULL argument");
  *n = c->trace.size();
  if (!out) return ST_OK;
  if (cap < c->trace.size()) return set_error(ST_ERR_INPUT, "trace: cap %zu < %zu events", cap, c->trace.size());
  memcpy(out, c->trace.data(), c->trace.size() * sizeof(st_event));
  return ST_OK;
}

st_status ctx_set_profiling(st_ctx* c, int on) {
  ST_CUDA_TRY(cudaSetDevice(c->device));
  ST_CUDA_TRY(cudaStreamSynchronize(c->stream));
  for (auto& p : c->prof.pairs) {
    c->prof.pool.push_back(p.a);
    c->prof.pool.push_back(p.b);
  }
  c->prof.pairs.clear();
  for (int i = 0; i < KC_COUNT; ++i) {
    c->prof.total_ms[i] = 0;
    c->prof.launches[i] = 0;
  }
  // on: bitmask of kernel classes (1 << KC_*); nonzero enables. Events are created
  // here, outside any timed region, so bracketing costs only the two records.
  for (auto& p : c->prof.lpairs) {
    c->prof.pool.push_back(p.a);
    c->prof.pool.push_back(p.b);
  }
  c->prof.lpairs.clear();
  c->prof.layer_ms.assign(2 * c->layers.size(), 0.0);
  c->prof.layer_n.assign(2 * c->layers.size(), 0);
  c->prof.layers = (on & ST_PROF_LAYERS) != 0;
  on &= ~ST_PROF_LAYERS;
  c->prof.mask = (unsigned)on;
  c->prof.on = on != 0;
  if (c->prof.on || c->prof.layers) {
    while (c->prof.pool.size() < 8192) {
      cudaEvent_t e;
      ST_CUDA_TRY(cudaEventCreate(&e));
      c->prof.pool.push_back(e);
    }
  }
  return ST_OK;
}

st_status ctx_get_layer_profile(st_ctx* c, double* ms, int64_t* counts, size_t n) {
  if (n < 2 * c->layers.size()) return set_error(ST_ERR_INPUT, "layer profile needs 2 x %zu entries", c->layers.size());
  ST_CUDA_TRY(cudaSetDevice(c->device));
  ST_CUDA_TRY(cudaStreamSynchronize(c->stream));
  ST_CUDA_TRY(cudaStreamSynchronize(c->side));
  for (auto& p : c->prof.lpairs) {
    float t = 0.f;
    ST_CUDA_TRY(cudaEventElapsedTime(&t, p.a, p.b));
    c->prof.layer_ms[p.cls] += t;
    c->prof.layer_n[p.cls] += 1;
    c->prof.pool.push_back(p.a);
    c->prof.pool.push_back(p.b);
  }
  c->prof.lpairs.clear();
  for (size_t i = 0; i < 2 * c->layers.size(); ++i) {
    if (ms) ms[i] = c->prof.layer_ms[i];
    if (counts) counts[i] = c->prof.layer_n[i];
  }
  return ST_OK;
}

st_status ctx_get_profile(st_ctx* c, double* total_ms, int64_t* launches) {
  ST_CUDA_TRY(cudaSetDevice(c->device));
  ST_CUDA_TRY(cudaStreamSynchronize(c->stream));
  for (auto& p : c->prof.pairs) {
    float ms = 0.f;
    ST_CUDA_TRY(cudaEventElapsedTime(&ms, p.a, p.b));
    c->prof.total_ms[p.cls] += ms;
    c->prof.launches[p.cls] += 1;
    c->prof.pool.push_back(p.a);
    c->prof.pool.push_back(p.b);
  }
  c->prof.pairs.clear();
  for (int i = 0; i < KC_COUNT; ++i) {
    if (total_ms) total_ms[i] = c->prof.total_ms[i];
    if (launches) launches[i] = c->prof.launches[i];
  }
  return ST_OK;
}

}  // namespace st
