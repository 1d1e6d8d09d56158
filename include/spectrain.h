/*
 * spectrain.h — C-ABI of libspectrain.so: one SpecTrain pipeline stage per
 * context (Chen, Yang, Cheng, arXiv 1809.02839).
 *
 * Citation key: P:n = PAPER.md line n, S:n = SPEC.md line n (the reference text
 * the method comes from); DESIGN.md §3 lists every reading (D1..D20) taken where
 * the paper is silent.
 *
 * What a context computes (per pipeline stage k of N):
 *   - PipeDream 1F1B task order over M mini-batches: min(N-k-1, M) warm-up
 *     forwards, then (F, B) pairs, then cooldown backwards ("round-robin").
 *   - Before every task, the predicted weights  Ŵ = W − s·η·v  (Eq. 4)
 *     with the version difference s of Eq. 5 (forward) or Eq. 6
 *     (backward); pred = ST_PRED_NONE forces s = 0 (vanilla).
 *   - Forward per dense layer: Z = A·Ŵ_W + Ŵ_b, A' = ReLU(Z) (identity on the
 *     network's last layer); softmax cross-entropy (batch mean) on the last stage
 *     (D11).
 *   - Backward: dZ = dA ⊙ 1[Z>0]; g_W = Aᵀ·dZ; g_b = Σ_b dZ; dA_prev = dZ·Ŵ_Wᵀ
 *     (D5: the backward re-predicts with s_B from the current state).
 *   - After each backward: v ← γ·v + (1−γ)·g (Eq. 1; ST_MOMENTUM_HEAVY_BALL:
 *     v ← γ·v + g, D2), W ← W − η·v (D1, Momentum SGD P:373), version += 1.
 *
 * Memory and ownership. All device memory is allocated by the CALLER (PyTorch in
 * the shipped binding) with the byte counts st_query_sizes reports, and is
 * BORROWED by the context until st_destroy. Device pointers must be 256-byte
 * aligned. Host pointers are read or written only during the call that receives
 * them. Streams are borrowed as well: the compute stream carries every kernel;
 * messages to / from the neighbouring stages run on two comm streams (one per
 * direction), ordered against the compute stream with CUDA events so that
 * transfers overlap compute. At the end of st_run / st_run_host and in st_sync
 * the comm streams are joined into the compute stream, so after those calls the
 * compute stream orders everything the context did. Calls return before the GPU
 * work finishes unless stated (st_sync blocks).
 *
 * Errors. Every function that can fail returns st_status; the message of the last
 * failure on the calling thread is available from st_last_error(). No C++
 * exception crosses this boundary. A failed call leaves the context usable only
 * for st_last_error/st_destroy unless the status is ST_ERR_INPUT/ST_ERR_SHAPE
 * (argument rejected before any state changed).
 *
 * Parameter layout (identical on host and device): stage-local flat fp32
 * array, layer-major; for each DENSE layer W_l [n_in × n_out] row-major, then b_l
 * [n_out] if the layer has a bias; EMBED: E [vocab × dim]; LSTM: W_ih, W_hh, b.
 *
 * Rows. Every activation, message and label vector has R = batch·seq_len rows
 * (seq_len = 1 for the FC models). Inputs of a stage whose first layer is EMBED are
 * int32 token ids [R] passed through the float* x arguments (same byte size).
 */
#ifndef SPECTRAIN_H_
#define SPECTRAIN_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define ST_API __attribute__((visibility("default")))
#else
#define ST_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ST_OK = 0,
  ST_ERR_INPUT = 1,     /* invalid argument / configuration */
  ST_ERR_SHAPE = 2,     /* layer chain or buffer size mismatch */
  ST_ERR_STATE = 3,     /* op out of program order: fatal invariant */
  ST_ERR_CUDA = 4,      /* CUDA runtime/driver failure */
  ST_ERR_NCCL = 5,      /* NCCL failure */
  ST_ERR_OOM = 6,       /* caller-provided buffer too small */
  ST_ERR_DIVERGED = 7,  /* non-finite loss; message names the mini-batch */
  ST_ERR_UNSUPPORTED = 8
} st_status;

enum { ST_FWD = 0, ST_BWD = 1 };
enum { ST_ACT_NONE = 0, ST_ACT_RELU = 1 };
/* Layer kinds. DENSE: Z = A·W + b, act. EMBED (network
 * layer 0 only): n_in = vocabulary, n_out = dimension, params E [n_in × n_out]; the
 * stage-0 input is int32 token ids. LSTM: n_in inputs, n_out = hidden H; params
 * W_ih [n_in × 4H], W_hh [H × 4H], b [4H], gate order i, f, g, o (reading D18),
 * h_{-1} = c_{-1} = 0 per mini-batch. */
enum { ST_LAYER_DENSE = 0, ST_LAYER_EMBED = 1, ST_LAYER_LSTM = 2, ST_LAYER_CONV = 3, ST_LAYER_POOL = 4 };
/* CONV: 3×3, stride 1, zero padding 1 on NHWC [hw × hw × n_in] → [hw × hw × n_out],
 * params W [3·3·n_in × n_out] (HWIO, rows (kh, kw, c)), then b; act RELU or NONE.
 * POOL: 2×2 max-pool stride 2, n_in = n_out = channels, hw even; no params. The
 * per-sample activation width entering a CONV / POOL layer is hw·hw·n_in; a DENSE layer
 * after the last POOL sees the flattened NHWC vector. (SURVEY §8(a) a10, D19, D21.) */
/* ST_PRED_STASH: PipeDream weight stashing (Fig. 6c) — no
 * prediction (s = 0); the forward of a mini-batch uses the stage's current W and its
 * backward the same stashed copy. The WF buffer then holds the stash: N−k slots of P
 * floats at a pitch of P rounded up to 64 (wf_bytes says how much); the update after
 * B(mb) writes W' into B(mb)'s slot, whose next user is F(mb + N − k). Trace: a
 * backward's base_version is the version its forward used. */
/* ST_PRED_STALENESS_FREE: the staleness-free target the paper
 * sets for SpecTrain — the whole round trip of a mini-batch on a stage adopts the version
 * that exists once the previous mini-batch has updated — per stage:
 * s_F = N−k−1 (the updates between F(i) and B(i) on stage k), s_B = 0. Both passes of
 * mini-batch i then target stage version i; Eq. 5/6 (SPECTRAIN) add ⌊k/2⌋ to both
 * (reading D6). */
enum { ST_PRED_SPECTRAIN = 0, ST_PRED_NONE = 1, ST_PRED_STASH = 2, ST_PRED_STALENESS_FREE = 3 };
enum { ST_MOMENTUM_EMA = 0, ST_MOMENTUM_HEAVY_BALL = 1 };
/* GEMM arithmetic. FP32X3 = 3xTF32 split (hi·hi + hi·lo + lo·hi) on tcgen05
 * tensor cores, fp32 accumulate in TMEM — the parity mode.
 * TF32 = single-pass tcgen05 kind::tf32 (fast mode, NOT parity-grade).
 * SIMT = CUDA-core fp32 FMA (bring-up / diagnostic mode). */
enum { ST_GEMM_FP32X3 = 0, ST_GEMM_TF32 = 1, ST_GEMM_SIMT = 2 };
enum { ST_LOSS_SOFTMAX_CE = 0 };
/* Stage-to-stage transport. NCCL: one process
 * per GPU; two communicators over the N stage ranks, one per direction (activations
 * k → k+1, gradients k+1 → k), ncclSend / ncclRecv per message on the comm stream of
 * that direction; asynchronous NCCL errors are polled while the library waits, and a
 * wait longer than ST_COMM_TIMEOUT_S seconds (default 600) aborts both communicators
 * (ST_ERR_NCCL). LOCAL: several stage contexts in ONE process (same GPU) linked with
 * st_connect_local; messages are device copies on the same comm streams, handed over
 * through host channels; a failing stage releases its blocked peers (ST_ERR_STATE).
 * P2P (transfer fused into compute over peer memory): no copy and
 * no send — stage k's last forward GEMM writes its output straight into stage k+1's
 * stash slot, stage k+1's layer-0 dX GEMM writes the gradient straight into stage k's
 * gradient ring; peer buffers are mapped with CUDA IPC (one process per GPU over
 * NVLink / NVSwitch, or processes sharing a GPU) or used directly (contexts of one
 * process); completion is handed over by flags in the waiter's memory (system-scope
 * release / acquire, one-thread kernels on the compute stream). Connect with
 * st_p2p_export + st_p2p_connect before the first task. A wait longer than
 * ST_COMM_TIMEOUT_S releases the spinning kernels and returns ST_ERR_STATE. Stages of one
 * process on one GPU are refused (their streams share hardware queues); with CUDA's
 * lazy module loading, a peer that dies during the FIRST session can block a kernel's
 * first launch behind a spinning wait (CUDA_MODULE_LOADING=EAGER rules that out). */
enum { ST_TRANSPORT_NCCL = 0, ST_TRANSPORT_LOCAL = 1, ST_TRANSPORT_P2P = 2 };

/* Opaque, trivially copyable descriptor of one P2P stage's exported buffers (its stash,
 * gradient ring and flag block: CUDA IPC handles + offsets, geometry, owner pid).
 * Exchange it between processes as 1024 raw bytes (e.g. torch.distributed). */
typedef struct {
  uint8_t bytes[1024];
} st_p2p_desc;

typedef struct {
  int32_t n_in;
  int32_t n_out;
  int32_t act;   /* ST_ACT_RELU for hidden layers, ST_ACT_NONE for the network's last layer */
  int32_t bias;  /* 1: the layer has a bias vector b_l [n_out] (DENSE) */
  int32_t kind;  /* ST_LAYER_* */
  int32_t hw;    /* CONV / POOL: input spatial side (square images); ignored otherwise */
} st_layer;

typedef struct {
  int32_t num_layers;       /* layers of the WHOLE network */
  const st_layer* layers;   /* [num_layers]; read during st_query_sizes / st_init only */
  int32_t num_stages;       /* N ≥ 1 */
  const int32_t* cuts;      /* [N-1] strictly increasing; stage k owns layers [cuts[k-1], cuts[k]) */
  int32_t stage;            /* k, 0 ≤ k < N */
  int32_t batch;            /* B ≥ 1 (mini-batch size) */
  int32_t seq_len;          /* T ≥ 1: activations are [T·B × width], time-major rows t·B + b */
  float lr;                 /* η > 0 */
  float gamma;              /* γ, 0 < γ ≤ 1 */
  int32_t pred;             /* ST_PRED_* */
  int32_t momentum;         /* ST_MOMENTUM_* */
  int32_t gemm;             /* ST_GEMM_* */
  int32_t loss;             /* ST_LOSS_SOFTMAX_CE */
  int32_t transport;        /* ST_TRANSPORT_* */
  int32_t device;           /* CUDA device ordinal of this stage */
  int64_t max_minibatches;  /* capacity of the on-device loss vector (≥ the M of st_run) */
  uint8_t nccl_id[128];     /* ST_TRANSPORT_NCCL: ncclUniqueId from st_get_nccl_id on stage 0 */
  /* Hybrid data × pipeline parallelism: replicas[s] ≥ 1
   * contexts share stage s (NULL = one each). A replicated stage splits the mini-batch
   * by rows — replica r computes rows [r·B/R, (r+1)·B/R) with batch B/R (`batch` stays
   * the GLOBAL B on every context) — and its replicas sum their gradients before the
   * identical K-B update (NCCL all-reduce over the stage's replicas, or an in-place
   * reduce across co-located replica contexts), so the pipeline computes exactly what
   * the unreplicated one does. The neighbours exchange row slices with each replica.
   * Limits (ST_ERR_INPUT): the last stage and adjacent stages cannot both / at all be
   * replicated, seq_len = 1, B divisible by R, not with ST_TRANSPORT_P2P. NCCL ranks
   * are stage-major: rank(s, r) = Σ_{j<s} replicas[j] + r. */
  const int32_t* replicas;  /* [N] or NULL */
  int32_t replica;          /* this context's index within its stage, 0 ≤ replica < replicas[stage] */
} st_config;

/* Byte counts the caller must allocate (0 = not needed: the buffer aliases W). */
typedef struct {
  int64_t params;       /* P_k: parameters of this stage (elements) */
  int64_t w_bytes;      /* W  — current weights */
  int64_t v_bytes;      /* V  — smoothed gradient, Eq. 1 */
  int64_t g_bytes;      /* G  — gradient of the last backward */
  int64_t wf_bytes;     /* WF — Ŵ for the next forward (0 if s_F = 0); ST_PRED_STASH: the weight stash */
  int64_t wb_bytes;     /* WB — Ŵ for the next backward (0 if s_B = 0 or s_B = s_F) */
  int64_t stash_bytes;  /* activation stash: N−k slots × Σ_l B·n_in_l fp32 */
  int64_t work_bytes;   /* messages, logits, split-K workspace, counters, losses */
  int32_t s_fwd;        /* Eq. 5 value used by this stage (0 under ST_PRED_NONE) */
  int32_t s_bwd;        /* Eq. 6 value */
} st_sizes;

typedef struct {
  float* W;
  float* V;
  float* G;
  float* WF;    /* NULL when wf_bytes == 0 */
  float* WB;    /* NULL when wb_bytes == 0 */
  void* stash;
  void* work;
} st_buffers;

/* One trace record per executed task. base_version = updates
 * already applied on this stage; s = version difference; target = base + s. */
typedef struct {
  int32_t stage;
  int32_t op_idx;
  int32_t dir;      /* ST_FWD / ST_BWD */
  int32_t pad_;
  int64_t mb;
  int64_t base_version;
  int64_t s;
  int64_t target;
} st_event;

/* One communication op of a stage program (host-side plan, no device work), in
 * issue order. kind: 0 send_fwd (to k+1, activation of mb), 1 recv_fwd (from k−1),
 * 2 send_bwd (to k−1, gradient), 3 recv_bwd (from k+1); kinds 0/1 run on the
 * activation communicator + comm_fwd stream, 2/3 on the gradient one + comm_bwd.
 * before_op = index of the program op it sits in front of (2M = after the last op);
 * n_ops = 1 (kind[1] = −1, mb[1] = −1 are unused). */
typedef struct {
  int32_t before_op;
  int32_t n_ops;
  int32_t kind[2];
  int64_t mb[2];
} st_comm_group;

typedef struct {
  int32_t ops_run;      /* tasks executed by this st_step call (0..3) */
  int32_t ran_forward;  /* mini-batch index of the forward run, −1 if none */
  int32_t ran_backward; /* mini-batch index of the backward run, −1 if none */
  int32_t done;         /* 1 when the stage program is complete */
  float loss;           /* loss of ran_forward on the last stage (synchronises), else NaN */
} st_step_info;

typedef struct st_ctx st_ctx;

/* ---- pure / host-only ------------------------------------------------------ */

/* Eq. 5 (dir = ST_FWD): ⌊k/2⌋ + N − k − 1; Eq. 6 (ST_BWD):
 * ⌊k/2⌋. Returns −1 unless 0 ≤ k < N (and N ≥ 1). */
ST_API int st_version_difference(int k, int N, int dir);

/* The event list stage k WILL produce for M mini-batches (program of SURVEY §8(c)
 * step 2 with the Eq. 5/6 values and base versions of §8(a) a1). Host only, no
 * GPU. out may be NULL to query the count (*n = 2M). ST_ERR_INPUT if cap < 2M. */
ST_API st_status st_program(int N, int k, int64_t M, int pred, st_event* out, size_t cap, size_t* n);

/* Layer-to-stage partition (stage imbalance bounds a pipeline,
 * P:146): contiguous cuts of n_layers layers with per-layer costs
 * cost[0..n_layers) (≥ 0, e.g. measured or roofline times) into N non-empty stages that
 * minimise the maximum stage cost; among optimal partitions the lexicographically
 * smallest cut vector. cuts_out[0..N−1) receives the first layer of stages 1..N−1 (the
 * st_config.cuts convention); *max_cost_out (may be NULL) the optimum. Host only.
 * Errors: ST_ERR_INPUT (N < 1, N > n_layers, negative / non-finite cost, NULL). */
ST_API st_status st_partition(const double* cost, int n_layers, int N, int32_t* cuts_out, double* max_cost_out);

/* The communication plan of stage k (order of grouped sends/receives the engine
 * issues). Host only. out may be NULL to query the count. */
ST_API st_status st_comm_plan(int N, int k, int64_t M, st_comm_group* out, size_t cap, size_t* n);

/* Byte counts for cfg (validates the whole config; no device work). */
ST_API st_status st_query_sizes(const st_config* cfg, st_sizes* out);

/* 128-byte ncclUniqueId; call on stage 0 and broadcast (torch.distributed). */
ST_API st_status st_get_nccl_id(uint8_t out[128]);

/* ---- context lifecycle ----------------------------------------------------- */

/* Binds buffers and streams (cudaStream_t cast to void*): `stream` = the compute
 * stream (NULL = legacy default stream); comm_fwd_stream / comm_bwd_stream = the
 * streams of the activation / gradient transfers (NULL: the library creates its own
 * non-blocking streams). Builds the 1F1B program, initialises NCCL for
 * ST_TRANSPORT_NCCL (collective across the N stage processes: every stage must call
 * st_init; two communicators), sets V = 0, WF = WB = W, version = 0. W is NOT
 * initialised: call st_set_params before the first task.
 * Errors: ST_ERR_INPUT (config, NULL / misaligned buffer), ST_ERR_SHAPE, ST_ERR_CUDA,
 * ST_ERR_NCCL (communicator setup). */
ST_API st_status st_init(const st_config* cfg, const st_buffers* bufs, void* stream, void* comm_fwd_stream,
                         void* comm_bwd_stream, st_ctx** out);

/* P2P transport: describe this context's peer-writable buffers (the stash and work
 * arenas must be cudaMalloc-backed allocations: CUDA IPC cannot export expandable /
 * VMM segments — ST_ERR_INPUT). The flag block is a small library-owned cudaMalloc
 * (freed by st_destroy). Errors: ST_ERR_STATE (not a P2P context), ST_ERR_INPUT. */
ST_API st_status st_p2p_export(st_ctx* ctx, st_p2p_desc* out);
/* P2P transport: map the neighbours' buffers (prev = stage k−1's descriptor, NULL for
 * k = 0; next = stage k+1's, NULL for k = N−1). Same-process descriptors are used as
 * plain pointers, others are opened with cudaIpcOpenMemHandle (closed by st_destroy).
 * Errors: ST_ERR_INPUT (missing / bad descriptor), ST_ERR_SHAPE (the descriptors do not
 * describe the adjacent stages of this pipeline), ST_ERR_CUDA (IPC open failed). */
ST_API st_status st_p2p_connect(st_ctx* ctx, const st_p2p_desc* prev, const st_p2p_desc* next);

/* LOCAL transport: link ctxs[0..n) as consecutive stages 0..n−1 of one pipeline
 * in this process. Required before any task of a LOCAL context. */
ST_API st_status st_connect_local(st_ctx** ctxs, int32_t n);

ST_API void st_destroy(st_ctx* ctx);

/* W ← host[0..n) (n must equal P_k; host or device memory of this GPU — UVA), V ← 0,
 * WF = WB = W, version ← 0, program restarted. Synchronous. ST_ERR_SHAPE on n mismatch. */
ST_API st_status st_set_params(st_ctx* ctx, const float* host, size_t n);

/* Copies W and V (either may be NULL) to host and the version counter. Synchronous. */
ST_API st_status st_get_params(st_ctx* ctx, float* W, float* V, size_t n, int64_t* version);

/* ---- the verbs of one pipeline task ---------------------------------------- */

/* F(mb) with WF. Stage 0 reads x_dev [R × n_in] (device, copied into the
 * stash; int32 tokens [R] for an EMBED layer); other stages receive the activation
 * from stage k−1. The last stage reads labels y_dev [R] int32 and writes the loss to its on-device loss vector
 * at index mb; if loss_host ≠ NULL it synchronises and copies the loss out
 * (ST_ERR_DIVERGED if non-finite). Non-last stages send their output to k+1.
 * ST_ERR_STATE if F(mb) is not the next op of the program. */
ST_API st_status st_stage_forward(st_ctx* ctx, int64_t mb, const float* x_dev, const int32_t* y_dev, float* loss_host);

/* B(mb) with WB: receives dA from k+1 (last stage: its stored CE gradient),
 * computes dX (sent to k−1 unless k = 0) and G. Does NOT update: the engine
 * requires st_predict_and_update before the next task. ST_ERR_STATE otherwise. */
ST_API st_status st_stage_backward(st_ctx* ctx, int64_t mb);

/* The fused K-B kernel on the whole stage arena: Eq. 1, the D1 apply, WF (s_F > 0)
 * and WB (s_B > 0, s_B ≠ s_F) for the next tasks; version += 1.
 * ST_ERR_STATE if no backward is pending. */
ST_API st_status st_predict_and_update(st_ctx* ctx);

/* Runs this stage's next program slot: warm-up F; steady F + B + update;
 * cooldown B + update. x_dev/y_dev are the inputs of the forward mini-batch
 * (stage 0 / last stage; others may pass NULL). */
ST_API st_status st_step(st_ctx* ctx, const float* x_dev, const int32_t* y_dev, st_step_info* out);

/* Whole M-mini-batch program from the current position. xs_dev [M × R × n_in]
 * (stage 0; [M × R] int32 tokens for EMBED), ys_dev [M × R] (last stage); losses_host [M] (last stage, may be
 * NULL) — when non-NULL the call synchronises and checks finiteness. */
ST_API st_status st_run(st_ctx* ctx, int64_t M, const float* xs_dev, const int32_t* ys_dev, float* losses_host);

/* st_run with HOST buffers (the end-to-end entry point): xs_host [M × B × n_in]
 * (stage 0) and ys_host [M × B] (last stage) are copied to the device per
 * mini-batch right before its forward (stream-ordered; pinned memory makes the
 * copies asynchronous), and each mini-batch's loss is copied back to
 * losses_host[mb] (last stage) as soon as it is computed. Synchronises at the end. */
ST_API st_status st_run_host(st_ctx* ctx, int64_t M, const float* xs_host, const int32_t* ys_host,
                             float* losses_host);

/* LOCAL transport: runs st_run on every context of a connected group, one host
 * thread per stage; returns the first failure. */
ST_API st_status st_run_group(st_ctx** ctxs, int32_t n, int64_t M, const float* xs_dev, const int32_t* ys_dev,
                       float* losses_host);

/* Trace of all tasks executed since st_set_params. out may be NULL (count query). */
ST_API st_status st_get_trace(st_ctx* ctx, st_event* out, size_t cap, size_t* n);

/* Device pointer of the on-device loss vector (last stage; NULL otherwise). */
ST_API const float* st_losses_device(st_ctx* ctx);

/* Joins the comm streams into the compute stream and waits for it. With a transport it
 * polls instead of blocking: an asynchronous NCCL error, or no completion within
 * ST_COMM_TIMEOUT_S seconds (a hung or dead peer), aborts the transport and returns
 * ST_ERR_NCCL (LOCAL: ST_ERR_STATE); the context is then only good for st_destroy. */
ST_API st_status st_sync(st_ctx* ctx);

/* Measurement hook (samples/s between stage-0 events after B(49) and
 * B(249), the paper's iteration window P:415): once the backward of mini-batch mb is
 * issued (in this or a later session, st_run or the verbs), `cuda_event` (a cudaEvent_t
 * cast to void*, created by the caller) is recorded on the compute stream after all the
 * work of that backward (its side-stream dW + update joined). One-shot; at most 64
 * pending. Errors: ST_ERR_INPUT (NULL event, mb < 0, too many pending). */
ST_API st_status st_record_after_backward(st_ctx* ctx, int64_t mb, void* cuda_event);

/* CUDA-graph sessions: with `on`, st_run / st_run_host capture the
 * whole session — every kernel, copy, event record and NCCL call the engine issues on
 * its compute, side and comm streams — into one CUDA graph (stream capture) and launch
 * it once, so latency-bound configurations stop paying a host launch per kernel. The
 * host bookkeeping (program counter, trace, versions) is done during the capture.
 * Requires: host buffers passed to st_run_host pinned (capturable copies); not for
 * contexts linked with st_connect_local (their host channels block), which keep running
 * eagerly. Errors: ST_ERR_CUDA (capture / instantiate / launch failed). */
ST_API st_status st_set_graph_mode(st_ctx* ctx, int on);

/* ---- measurement hooks ----------------------------------------------------- */

/* Profiling: `on` is a bitmask of kernel classes (bit i = class i; 0 = off). The
 * engine brackets every launch of a selected class with CUDA events on the stream
 * it is launched on (events are pre-created by this call, so a timed region pays
 * only the two records). Classes: 0 update (K-B), 1 gemm_fwd, 2 gemm_dx,
 * 3 gemm_dw, 4 loss (CE + bias-grad), 5 comm. Resets the totals. */
ST_API st_status st_set_profiling(st_ctx* ctx, int on);
/* Bit of `on` (st_set_profiling) that brackets each layer's whole forward and
 * backward work instead (PipeDream-style per-layer profile; SURVEY §8(f)
 * NEXT-4): while set, the backward runs serialised (each layer's dW + update is joined
 * before the next layer starts), so a bracket is that layer's cost alone. */
#define ST_PROF_LAYERS (1 << 30)
/* Per layer l of the stage: ms[2l] / ms[2l+1] = total milliseconds of its forward /
 * backward work since profiling was switched on, counts[...] = passes bracketed
 * (either may be NULL). n ≥ 2·(layers of the stage), else ST_ERR_INPUT. Synchronises. */
ST_API st_status st_get_layer_profile(st_ctx* ctx, double* ms, int64_t* counts, size_t n);
/* Per class: total milliseconds and launch count since profiling was switched on
 * (synchronises). arrays of length 6. */
ST_API st_status st_get_profile(st_ctx* ctx, double* total_ms, int64_t* launches);
/* Kernel launches issued by this context since creation (all classes). */
ST_API int64_t st_kernel_launches(st_ctx* ctx);

/* ---- raw kernels (test and bench hooks on caller arenas) --------------------- */

/* Prediction accuracy of Fig. 7. W_old / V_old: a
 * stage's weights and stored smoothed gradient s updates before W_now (device fp32,
 * n elements each). out_host[0] = Σ (W_old − s·lr·V_old − W_now)² (the Eq. 4
 * prediction's error), out_host[1] = Σ (W_old − W_now)² (the stale weights' error), both
 * accumulated in fp64 in a fixed order (RMSE = sqrt(sum / n)). work: device scratch of
 * st_prediction_error_work_bytes() bytes, 8-byte aligned. Stream-ordered, then syncs the
 * stream to return the sums. Errors: ST_ERR_INPUT (NULL buffer, s < 0), ST_ERR_CUDA. */
ST_API int64_t st_prediction_error_work_bytes(void);
ST_API st_status st_prediction_error_raw(const float* W_old, const float* V_old, const float* W_now, size_t n, int s,
                                         float lr, double* out_host, void* work, void* stream);

/* K-B on caller arenas of n fp32: v' = γv + (1−γ)g (HEAVY_BALL: γv + g),
 * w' = w − η v', WF = w' − s_F η v' (if WF ≠ NULL), WB = w' − s_B η v' (if WB ≠ NULL).
 * All pointers 16-byte aligned device pointers; n = 0 is a no-op.
 * ST_ERR_INPUT on misalignment. Stream-ordered. */
ST_API st_status st_update_predict_raw(float* W, float* V, const float* G, float* WF, float* WB, size_t n, float lr,
                                float gamma, int sF, int sB, int momentum, void* stream);

/* GEMM kernels of the stage path, on caller buffers (device, row-major fp32).
 *   op 0 (fwd): Z[B×out] = X[B×in]·W[in×out] + b[out]; relu → ReLU applied.
 *   op 1 (dX):  D[B×in]  = dZ[B×out]·W[in×out]ᵀ, then ⊙ 1[mask[B×in] > 0] if mask.
 *   op 2 (dW):  G[in×out] = X[B×in]ᵀ·dZ[B×out]; gb[out] = Σ_b dZ[b,:] if gb ≠ NULL.
 * Buffer roles: a = X (op 0, 2) or dZ (op 1); b = W (op 0, 1) or dZ (op 2);
 * bias/mask = b (op 0) or mask (op 1) or gb (op 2); out = Z / D / G.
 * work: device scratch of st_gemm_workspace_bytes() bytes. */
ST_API st_status st_gemm_raw(int op, int gemm_mode, int B, int n_in, int n_out, const float* a, const float* b,
                      const float* aux, float* aux_out, float* out, int relu, void* work, void* stream);
ST_API int64_t st_gemm_workspace_bytes(int B, int n_in, int n_out);

/* dW fused with the K-B update on one layer block (the path st_run takes): with
 * g = [X[B×in]ᵀ·dZ[B×out] ; Σ_b dZ] never written to HBM, applies Eq. 1, the D1
 * apply and the Eq. 4 predictions to W / V / WF / WB, each a block of in·out + out
 * fp32 (weights [in×out] row-major, then the bias). WF / WB may be NULL. G_scratch
 * (same size) is used only when the fused kernel cannot run (16-byte pitch rule,
 * SIMT mode). work: st_gemm_workspace_bytes(B, in, out). Stream-ordered. */
ST_API st_status st_dw_update_raw(int gemm_mode, int B, int n_in, int n_out, const float* X, const float* dZ, float* W,
                                  float* V, float* WF, float* WB, float lr, float gamma, int sF, int sB, int momentum,
                                  float* G_scratch, void* work, void* stream);

/* Softmax-CE on caller buffers: logits [B×C], labels [B] → loss_dev[0] (batch
 * mean) and dlogits [B×C] = (softmax − onehot)/B. */
ST_API st_status st_softmax_ce_raw(const float* logits, const int32_t* labels, int B, int C, float* loss_dev,
                            float* dlogits, void* work, void* stream);

ST_API const char* st_last_error(void);
ST_API const char* st_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SPECTRAIN_H_ */
