// Stage engine: one SpecTrain pipeline stage bound to caller-owned arenas.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "common.hpp"
#include "kernels.hpp"

namespace st {

struct Task {
  int dir;  // ST_FWD / ST_BWD
  int64_t mb;
};

enum CommKind { CK_SEND_FWD = 0, CK_RECV_FWD = 1, CK_SEND_BWD = 2, CK_RECV_BWD = 3 };
using CommGroup = st_comm_group;

int version_difference(int k, int N, int dir);
// the version difference stage k uses for its forward / backward under a pred mode:
// Eq. 5 / Eq. 6 (SPECTRAIN), 0 (NONE, STASH), N−k−1 / 0 (STALENESS_FREE)
int stage_s(int pred, int k, int N, int dir);
std::vector<Task> build_program(int N, int k, int64_t M);
std::vector<st_event> program_events(int N, int k, int64_t M, int pred);
std::vector<CommGroup> build_comm_plan(int N, int k, int64_t M);
st_status partition_layers(const double* cost, int L, int N, int32_t* cuts, double* max_cost);

// Stage-to-stage transport. The engine issues every
// message as ONE op on the comm stream of its direction (kind CK_SEND_FWD /
// CK_RECV_FWD: activations, the k→k+1 channel; CK_SEND_BWD / CK_RECV_BWD:
// gradients, the k+1→k channel), ordered against the compute stream with events
// (engine.cpp issue_op). A transport only moves bytes on the stream it is given.
class Transport {
 public:
  virtual ~Transport() = default;
  // chan: the replica index of the replicated side of this channel (hybrid DP × PP,
  // NEXT-4; 0 when neither neighbour is replicated)
  virtual st_status send(int kind, int64_t mb, const float* buf, size_t count, cudaStream_t s, int chan = 0) = 0;
  virtual st_status recv(int kind, int64_t mb, float* buf, size_t count, cudaStream_t s, int chan = 0) = 0;
  // the ops to / from several replicas of a neighbour form one group (NCCL: ncclGroupStart / End)
  virtual st_status group_begin() { return ST_OK; }
  virtual st_status group_end() { return ST_OK; }
  // sum `buf` over the replicas of this stage (NCCL: ncclAllReduce on the replica communicator)
  virtual st_status allreduce_sum(float* buf, size_t n, cudaStream_t s) {
    (void)buf; (void)n; (void)s;
    return set_error(ST_ERR_STATE, "transport: no replica all-reduce");
  }
  // asynchronous failure of the transport (NCCL: ncclCommGetAsyncError on both
  // communicators); ST_OK while healthy
  virtual st_status poll() { return ST_OK; }
  // tear the transport down after a failure so that no peer or stream waits forever
  // (NCCL: ncclCommAbort; LOCAL: wake and fail every blocked peer)
  virtual void abort() {}
};

// reps: replicas per stage (NCCL ranks are stage-major: rank(s, r) = Σ_{j<s} reps[j] + r)
std::unique_ptr<Transport> make_nccl_transport(const uint8_t id[128], int N, int k, int device,
                                               const std::vector<int>& reps, int replica, st_status* err);

struct LocalLink;  // shared channels of a LOCAL pipeline (transport.cpp)
std::unique_ptr<Transport> make_local_transport(std::shared_ptr<LocalLink> link, int k, float* ring_fwd,
                                                float* ring_bwd, size_t fwd_elems, size_t bwd_elems, int replica,
                                                int rep_prev, int rep_self, int rep_next, st_status* err);
std::shared_ptr<LocalLink> make_local_link(int N, const std::vector<int>& reps);
void abort_local_link(LocalLink* link);

// co-located replicas of one stage (LOCAL transport): in-place sum of their gradient
// arenas, each replica reducing one slice of every arena (transport.cpp)
struct ReplicaGroup;
std::shared_ptr<ReplicaGroup> make_replica_group(int R, std::shared_ptr<LocalLink> link);
st_status replica_reduce_local(ReplicaGroup* g, int replica, float* G, size_t n, cudaStream_t s);

// P2P transport (p2p.cu): the producing kernels write into the peer's buffers, flags
// in the waiter's memory hand them over (NEXT-3)
struct P2pState;

struct LayerInfo {
  int n_in, n_out, act, bias, kind;
  int hw;             // conv / pool: input spatial side
  int64_t win, wout;  // per-sample activation width in / out
  int64_t w_off;      // offset of W_l (dense), E (embed), W_ih (lstm) in the stage arena
  int64_t whh_off;    // lstm: offset of W_hh (−1 otherwise)
  int64_t b_off;      // offset of b_l (−1 if none)
  int64_t n_params;   // parameters of the layer (a contiguous block from w_off)
  int64_t stash_off;  // offset of the layer input inside one stash slot (−1: aliases the
                      // previous LSTM layer's h buffer); embed: int32 tokens [R]
  int64_t gates_off, c_off, h_off;  // lstm: gates [R×4H], c [R×H], h [(R+B)×H] per slot
};

// LSTM / embedding kernels (k_lstm.cu)
// rec / dh_next: the recurrent GEMM output, or (plan with splits > 1) its deferred
// split-K partials; h_lo / dG_lo (nullable): tf32 lo halves for the next recurrent GEMM
st_status launch_lstm_cell_fwd(float* gates, const float* rec, const SplitPlan* rp, const float* c_prev, float* c_out,
                               float* h_out, float* h_lo, int B, int H, cudaStream_t s);
st_status launch_lstm_cell_bwd(const float* gates, const float* c_t, const float* c_prev, const float* dOut,
                               const float* dh_next, const SplitPlan* hp, float* dc, int first, float* dG,
                               float* dG_lo, int B, int H, cudaStream_t s);
st_status launch_embed_gather(const float* E, const int32_t* tok, int rows, int D, float* out, cudaStream_t s);
int64_t embed_grad_scratch_bytes(int rows, int V);
st_status launch_embed_grad(const float* dA, const int32_t* tok, int rows, int V, int D, float* gE, void* scratch,
                            cudaStream_t s);
// conv / pool kernels (k_conv.cu)
st_status launch_im2col(const float* X, int B, int H, int W, int C, float* col, cudaStream_t s);
// rows padded to 32 columns (9·C ≤ 32), zeros after the window: the first conv's TMA path
st_status launch_im2col_pad32(const float* X, int B, int H, int W, int C, float* col, cudaStream_t s);
st_status launch_col2im(const float* dcol, int B, int H, int W, int C, const float* mask, float* dX, cudaStream_t s);
st_status launch_maxpool_fwd(const float* X, int B, int H, int W, int C, float* Y, cudaStream_t s);
st_status launch_maxpool_bwd(const float* X, const float* dY, int B, int H, int W, int C, int relu_mask, float* dX,
                             cudaStream_t s);

struct Profiler {
  bool on = false;
  unsigned mask = 0;  // bit i: bracket kernel class i
  struct Pair {
    int cls;
    cudaEvent_t a, b;
  };
  std::vector<Pair> pairs;
  std::vector<cudaEvent_t> pool;
  double total_ms[KC_COUNT] = {};
  int64_t launches[KC_COUNT] = {};
  // ST_PROF_LAYERS: per-layer brackets (cls = 2·layer + dir) of the whole forward /
  // backward work of each layer; the backward runs serialised (no side-stream overlap)
  bool layers = false;
  std::vector<Pair> lpairs;
  std::vector<double> layer_ms;  // [2·L]: fwd, bwd per layer
  std::vector<int64_t> layer_n;
};

}  // namespace st

struct st_ctx {
  // configuration
  int N = 1, k = 0, B = 1;
  int T = 1;           // sequence length
  int64_t R = 1;       // activation rows = B·T
  bool embed_first = false;
  float lr = 0.f, gamma = 0.f;
  int pred = ST_PRED_SPECTRAIN, momentum = ST_MOMENTUM_EMA, gemm = ST_GEMM_FP32X3, loss = ST_LOSS_SOFTMAX_CE;
  int transport_kind = ST_TRANSPORT_NCCL;
  int device = 0;
  int64_t max_mb = 0;
  std::vector<st::LayerInfo> layers;
  int64_t P = 0;
  int sF = 0, sB = 0;
  int max_width_in = 0, max_width_out = 0;
  bool first_stage = true, last_stage = true;

  // arenas (borrowed)
  float *W = nullptr, *V = nullptr, *G = nullptr;
  const float *WF = nullptr, *WB = nullptr;  // weights the next F / B read (may alias W)
  float *WF_out = nullptr, *WB_out = nullptr;  // K-B outputs (NULL when aliased)
  int prev_act = ST_ACT_NONE;                  // activation of the layer feeding stage k > 0
  int in_first = 0, out_last = 0;
  float* stash = nullptr;
  int64_t slot_elems = 0;
  int S = 1;  // stash slots = N − k
  // work carve-up
  // messages of the current task (engine.cpp run_task picks one of two slots per
  // mini-batch parity, so a transfer of mb can overlap the compute of mb + 1)
  float* send_fwd = nullptr;  // [R × out_last]  (non-last stage)
  float* recv_bwd = nullptr;  // [R × out_last]  (non-last stage)
  float* send_bwd = nullptr;  // [R × in_first]  (k > 0)
  float* send_fwd2[2] = {nullptr, nullptr};
  float* recv_bwd2[2] = {nullptr, nullptr};
  float* send_bwd2[2] = {nullptr, nullptr};
  // comm streams (activations k→k+1 / from k−1 on comm_fwd; gradients on comm_bwd) and
  // the events ordering them against the compute stream (engine.cpp issue_op)
  cudaStream_t comm_fwd = nullptr, comm_bwd = nullptr;
  bool own_comm_fwd = false, own_comm_bwd = false;
  cudaEvent_t ev_sent_fwd[2] = {}, ev_sent_bwd[2] = {};  // send of slot b finished (comm stream)
  bool sent_fwd_pending[2] = {false, false}, sent_bwd_pending[2] = {false, false};
  cudaEvent_t ev_recv_bwd[2] = {};                       // gradient of slot b arrived (comm_bwd)
  cudaEvent_t ev_bwd_ring[2] = {};                       // the backward reading recv_bwd2[b] finished (compute)
  bool bwd_ring_done[2] = {false, false};
  std::vector<cudaEvent_t> ev_recv_fwd;                  // per stash slot: activation arrived (comm_fwd)
  std::vector<cudaEvent_t> ev_bwd_slot;                  // per stash slot: its last backward finished (compute)
  std::vector<char> bwd_slot_done;
  cudaEvent_t ev_fwd_done = nullptr;    // the forward whose output is sent next
  cudaEvent_t ev_dx_ready = nullptr;    // layer-0 dX of the current backward written (compute)
  cudaEvent_t ev_join[2] = {};          // comm streams joined into compute at session end
  double comm_timeout_s = 600.0;        // ST_COMM_TIMEOUT_S: a wait longer than this is a hung peer
  std::vector<std::pair<int64_t, cudaEvent_t>> marks;  // st_record_after_backward
  float* logits = nullptr;    // [B × C]         (last stage)
  float* dlogits = nullptr;   // [B × C]
  float* bufA = nullptr;      // [R × max width] backward gradient buffers (3-way rotation)
  float* bufB = nullptr;
  float* bufC = nullptr;
  cudaStream_t side = nullptr;          // library-owned: dW + update overlapped with the next dX
  std::vector<cudaEvent_t> side_events; // one per layer (dW done) + join
  bool dwu_env = false;                 // ST_DWU_SMS given: one budget for every layer
  int dwu_sms = 80;                     // SM budget of an overlapped dW + update (measured best)
  float* losses_dev = nullptr;  // [max_mb]
  float* rowloss = nullptr;     // [B]
  int32_t* y_stage = nullptr;   // [R] labels staged from host (st_run_host)
  float* lstm_rec = nullptr;    // [B × 4H] h_{t−1}·W_hh
  float* lstm_dh = nullptr;     // [B × H] dh_next
  bool pdl_now = false;         // this task's launches (run_task)
  bool pdl_dense = true;        // dense fwd / dX kernels as programmatic dependent launches (ST_PDL_DENSE=0: off)
  bool pdl = true;              // LSTM recurrence: GEMM ↔ cell as programmatic dependent launches (ST_PDL=0: off)
  bool graph_mode = false;      // st_set_graph_mode: st_run sessions captured into one CUDA graph
  int64_t graph_sessions = 0;   // sessions launched as graphs
  bool capturing = false;       // inside the capture of a graph session
  bool bwd_serial = true;       // dense layers with ≥ 2^27 parameters: dW + update after the dX on the
                                // compute stream (whole GPU each) instead of overlapped on the side stream
  bool conv_overlap = false;    // implicit-conv dW + update on the side stream (ST_CONV_OVERLAP=1; measured
                                // slower: VGG-16 58.9k -> 53.0k samples/s with an 80 / 68 SM split)
  float* wstash = nullptr;      // ST_PRED_STASH: S slots of P floats (the WF buffer)
  std::vector<int64_t> stash_ver;  // ST_PRED_STASH: version each slot's forward used
  float* lstm_hlo = nullptr;    // [B × H] tf32 lo of h_{t−1} (3xTF32 operand of the recurrent GEMM)
  float* lstm_dglo = nullptr;   // [B × 4H] tf32 lo of dG_t (operand of the dh GEMM)
  float* lstm_dc = nullptr;     // [B × H] dc_next
  float* lstm_dG = nullptr;     // [R × 4H] gate gradients of all steps
  void* embed_scratch = nullptr;
  float* conv_col = nullptr;    // [P × 9·C_in] im2col of the current conv layer
  float* conv_dcol = nullptr;   // [P × 9·C_in] its gradient
  int64_t gemm_rows_max = 1;    // largest GEMM row count (R or conv pixel rows)
  int gemm_in_max = 1, gemm_out_max = 1;
  float* ring_fwd = nullptr;    // LOCAL transport rings
  float* ring_bwd = nullptr;
  size_t ring_fwd_elems = 0, ring_bwd_elems = 0;
  void* gemm_ws = nullptr;
  void* gemm_ws2 = nullptr;  // workspace of the side stream
  cudaStream_t stream = nullptr;
  int sm_count = 148;  // SMs of this device (cudaDevAttrMultiProcessorCount)

  // program state
  std::vector<st::Task> program;
  std::vector<st::CommGroup> plan;
  size_t pc = 0;
  size_t plan_next = 0;  // next comm-plan op to issue
  int64_t session_M = 0;
  int64_t version = 0;
  bool pending_update = false;
  std::vector<st_event> trace;
  std::unique_ptr<st::Transport> tp;
  std::shared_ptr<st::LocalLink> link;
  st::P2pState* p2p = nullptr;  // ST_TRANSPORT_P2P
  // hybrid DP × PP (NEXT-4): replicas of stages k−1, k, k+1, this context's replica index
  int rep_prev = 1, rep_self = 1, rep_next = 1, replica = 0;
  int B_global = 1;
  std::vector<int> reps;                         // replicas per stage (all N)
  bool shares_gpu = false;
  bool pdl_serial = true;  // programmatic launches for the serialised backward of ≥ 2^27-parameter layers  // LOCAL transport with other stage / replica contexts in this process
  std::shared_ptr<st::ReplicaGroup> rgroup;      // LOCAL: the stage's co-located replicas

  st::Profiler prof;
  int64_t launches = 0;
};

namespace st {
st_status p2p_alloc(st_ctx* c);
void p2p_free(st_ctx* c);
st_status p2p_export(st_ctx* c, st_p2p_desc* out);
st_status p2p_connect(st_ctx* c, const st_p2p_desc* prev, const st_p2p_desc* next);
void p2p_begin_session(st_ctx* c);
st_status p2p_before_forward(st_ctx* c, int64_t mb);
st_status p2p_after_forward(st_ctx* c, int64_t mb);
st_status p2p_before_backward(st_ctx* c, int64_t mb);
st_status p2p_after_dx(st_ctx* c, int64_t mb);
st_status p2p_after_backward(st_ctx* c, int64_t mb);
st_status p2p_check(st_ctx* c);
std::string p2p_describe(st_ctx* c);  // the flag block (diagnostics of a hang)
st_status launch_replica_sum(float* const* Gs, int R, size_t begin, size_t end, cudaStream_t s);
}  // namespace st
