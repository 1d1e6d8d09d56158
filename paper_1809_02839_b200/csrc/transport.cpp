// Stage-to-stage transports ("activations and
// gradients are transferred between GPUs", "sent to the next GPU ... to hide
// the latency").
//
// The engine (engine.cpp issue_op) issues every message as one op on the comm
// stream of its direction — activations k→k+1 on comm_fwd, gradients k+1→k on
// comm_bwd — ordered against the compute stream with CUDA events, so transfers
// overlap compute. A transport only moves the bytes on the stream it is handed.
//
// NCCL: one process per GPU; two communicators over the same ranks (one per
// direction), ncclSend / ncclRecv per message; asynchronous errors
// polled by the engine while it waits (ST_ERR_NCCL), ncclCommAbort on failure.
//
// LOCAL: several stage contexts in one process (tests run an N-stage pipeline on
// one GPU; bench can oversubscribe). Each directed channel k→k+1 / k+1→k is a
// host queue of (mini-batch, ring slot) records plus a device ring owned by the
// sender: send = stream-ordered copy into the ring slot + CUDA event; receive =
// blocking pop, wait on the event, copy out, record a "consumed" event the sender
// waits on before reusing the slot. A failing stage aborts the link: every peer
// blocked on it returns ST_ERR_STATE at once instead of waiting for the timeout.
#include <nccl.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>

#include "engine.hpp"

namespace st {

// ------------------------------------------------------------------ NCCL
namespace {

// Two communicators over the same N ranks, one per direction of the pipeline (SURVEY
// §7.2 H5: forward- and backward-direction traffic must progress independently, so
// they do not share a communicator): `fwd_` carries the activations k → k+1, `bwd_`
// the gradients k+1 → k. The engine issues each communicator's ops from one host
// thread on one comm stream, in the same order on every rank (the comm plan).
class NcclTransport final : public Transport {
 public:
  NcclTransport(ncclComm_t f, ncclComm_t b, ncclComm_t rep, int N, int k, std::vector<int> reps)
      : fwd_(f), bwd_(b), rep_(rep), N_(N), k_(k), reps_(std::move(reps)) {
    base_.assign(N_ + 1, 0);
    for (int s = 0; s < N_; ++s) base_[s + 1] = base_[s] + reps_[s];
  }
  ~NcclTransport() override {
    if (aborted_) return;
    if (fwd_) ncclCommDestroy(fwd_);
    if (bwd_) ncclCommDestroy(bwd_);
    if (rep_) ncclCommDestroy(rep_);
  }
  // rank of the peer stage's context on this channel: its replica `chan` if it is the
  // replicated side, else its only context
  int rank_of(int stage, int chan) const { return base_[stage] + (reps_[stage] > 1 ? chan : 0); }
  st_status group_begin() override {
    ncclResult_t r = ncclGroupStart();
    return r == ncclSuccess ? ST_OK : set_error(ST_ERR_NCCL, "ncclGroupStart: %s", ncclGetErrorString(r));
  }
  st_status group_end() override {
    ncclResult_t r = ncclGroupEnd();
    return r == ncclSuccess ? ST_OK : set_error(ST_ERR_NCCL, "ncclGroupEnd: %s", ncclGetErrorString(r));
  }
  st_status allreduce_sum(float* buf, size_t n, cudaStream_t s) override {
    if (!rep_) return set_error(ST_ERR_STATE, "stage %d: not replicated", k_);
    ncclResult_t r = ncclAllReduce(buf, buf, n, ncclFloat32, ncclSum, rep_, s);
    if (r != ncclSuccess)
      return set_error(ST_ERR_NCCL, "stage %d: ncclAllReduce (replica gradients): %s", k_, ncclGetErrorString(r));
    return ST_OK;
  }
  st_status send(int kind, int64_t mb, const float* buf, size_t count, cudaStream_t s, int chan) override {
    const bool f = kind == CK_SEND_FWD;
    if (!f && kind != CK_SEND_BWD) return set_error(ST_ERR_INPUT, "nccl send: bad kind %d", kind);
    const int ps = f ? k_ + 1 : k_ - 1;
    if (ps < 0 || ps >= N_) return set_error(ST_ERR_STATE, "stage %d: no peer %d", k_, ps);
    const int peer = rank_of(ps, chan);
    ncclResult_t r = ncclSend(buf, count, ncclFloat32, peer, f ? fwd_ : bwd_, s);
    if (r != ncclSuccess)
      return set_error(ST_ERR_NCCL, "stage %d: ncclSend(mb %lld -> %d): %s", k_, (long long)mb, peer,
                       ncclGetErrorString(r));
    return ST_OK;
  }
  st_status recv(int kind, int64_t mb, float* buf, size_t count, cudaStream_t s, int chan) override {
    const bool f = kind == CK_RECV_FWD;
    if (!f && kind != CK_RECV_BWD) return set_error(ST_ERR_INPUT, "nccl recv: bad kind %d", kind);
    const int ps = f ? k_ - 1 : k_ + 1;
    if (ps < 0 || ps >= N_) return set_error(ST_ERR_STATE, "stage %d: no peer %d", k_, ps);
    const int peer = rank_of(ps, chan);
    ncclResult_t r = ncclRecv(buf, count, ncclFloat32, peer, f ? fwd_ : bwd_, s);
    if (r != ncclSuccess)
      return set_error(ST_ERR_NCCL, "stage %d: ncclRecv(mb %lld <- %d): %s", k_, (long long)mb, peer,
                       ncclGetErrorString(r));
    return ST_OK;
  }
  st_status poll() override {
    if (aborted_) return set_error(ST_ERR_NCCL, "stage %d: communicators were aborted", k_);
    for (ncclComm_t c : {fwd_, bwd_, rep_}) {
      if (!c) continue;
      ncclResult_t a = ncclSuccess;
      ncclResult_t r = ncclCommGetAsyncError(c, &a);
      if (r != ncclSuccess)
        return set_error(ST_ERR_NCCL, "stage %d: ncclCommGetAsyncError: %s", k_, ncclGetErrorString(r));
      if (a != ncclSuccess && a != ncclInProgress)
        return set_error(ST_ERR_NCCL, "stage %d: asynchronous NCCL error on the %s communicator: %s", k_,
                         c == fwd_ ? "activation" : "gradient", ncclGetErrorString(a));
    }
    return ST_OK;
  }
  // ncclCommAbort of one communicator waits for the device work in flight, and a kernel of
  // the other communicator may be what that work waits on (the compute stream waits on
  // both comm streams): abort both concurrently so both abort flags are raised at once.
  void abort() override {
    if (aborted_) return;
    aborted_ = true;
    int dev = 0;
    cudaGetDevice(&dev);
    std::thread t([this, dev] {
      cudaSetDevice(dev);
      ncclCommAbort(bwd_);
    });
    std::thread t2([this, dev] {
      cudaSetDevice(dev);
      if (rep_) ncclCommAbort(rep_);
    });
    ncclCommAbort(fwd_);
    t.join();
    t2.join();
  }

 private:
  ncclComm_t fwd_, bwd_, rep_;
  int N_, k_;
  std::vector<int> reps_, base_;
  bool aborted_ = false;
};

}  // namespace

std::unique_ptr<Transport> make_nccl_transport(const uint8_t id[128], int N, int k, int device,
                                               const std::vector<int>& reps, int replica, st_status* err) {
  *err = ST_OK;
  int world = 0, rank = 0;
  for (int s = 0; s < N; ++s) {
    if (s == k) rank = world + replica;
    world += reps[s];
  }
  if (world == 1) return nullptr;  // a 1-stage, unreplicated pipeline never communicates
  ncclUniqueId uid;
  static_assert(sizeof(uid.internal) == 128, "ncclUniqueId size");
  memcpy(uid.internal, id, 128);
  if (cudaSetDevice(device) != cudaSuccess) {
    *err = set_error(ST_ERR_CUDA, "cudaSetDevice(%d)", device);
    return nullptr;
  }
  ncclComm_t f = nullptr, b = nullptr, rc = nullptr;
  ncclResult_t r = ncclCommInitRank(&f, world, uid, rank);
  if (r != ncclSuccess) {
    *err = set_error(ST_ERR_NCCL, "ncclCommInitRank(world=%d, rank=%d): %s", world, rank, ncclGetErrorString(r));
    return nullptr;
  }
  // the gradient-direction communicator: same ranks, same order (collective over all stages)
  r = ncclCommSplit(f, 0, rank, &b, nullptr);
  if (r != ncclSuccess || !b) {
    *err = set_error(ST_ERR_NCCL, "ncclCommSplit (gradient communicator, rank %d): %s", rank, ncclGetErrorString(r));
    ncclCommDestroy(f);
    return nullptr;
  }
  // the replicas of each replicated stage (collective over all ranks; others get none)
  bool any_rep = false;
  for (int s = 0; s < N; ++s) any_rep |= reps[s] > 1;
  if (any_rep) {
    r = ncclCommSplit(f, reps[k] > 1 ? k : NCCL_SPLIT_NOCOLOR, replica, &rc, nullptr);
    if (r != ncclSuccess) {
      *err = set_error(ST_ERR_NCCL, "ncclCommSplit (replica communicator, rank %d): %s", rank, ncclGetErrorString(r));
      ncclCommDestroy(f);
      ncclCommDestroy(b);
      return nullptr;
    }
  }
  return std::unique_ptr<Transport>(new NcclTransport(f, b, rc, N, k, reps));
}

// ------------------------------------------------------------------ LOCAL
struct Channel {
  std::mutex mu;
  std::condition_variable cv;
  struct Msg {
    int64_t mb;
    int slot;
    size_t count;
  };
  std::deque<Msg> q;
  float* ring = nullptr;  // sender-owned, R slots of `elems`
  size_t elems = 0;
  int R = 0;
  int64_t sent = 0, received = 0;
  std::vector<cudaEvent_t> ready, consumed;
  std::vector<bool> consumed_recorded;
};

struct LocalLink {
  int N = 0;
  std::atomic<bool> aborted{false};
  // fwd[k][c]: k→k+1, bwd[k][c]: k+1→k; c = replica of the replicated side of the
  // boundary (one channel per replica; one channel when neither side is replicated)
  std::vector<std::vector<std::unique_ptr<Channel>>> fwd, bwd;
  std::vector<std::condition_variable*> extra_cvs;  // replica-group barriers woken by an abort
  std::mutex extra_mu;
};

std::shared_ptr<LocalLink> make_local_link(int N, const std::vector<int>& reps) {
  auto l = std::make_shared<LocalLink>();
  l->N = N;
  for (int k = 0; k + 1 < N; ++k) {
    const int nc = std::max(reps[k], reps[k + 1]);
    l->fwd.emplace_back();
    l->bwd.emplace_back();
    for (int c = 0; c < nc; ++c) {
      l->fwd.back().emplace_back(new Channel());
      l->bwd.back().emplace_back(new Channel());
    }
  }
  return l;
}

void abort_local_link(LocalLink* l) {
  if (!l) return;
  l->aborted = true;
  for (auto* v : {&l->fwd, &l->bwd})
    for (auto& row : *v)
      for (auto& ch : row) {
        { std::lock_guard<std::mutex> g(ch->mu); }
        ch->cv.notify_all();
      }
  std::lock_guard<std::mutex> g(l->extra_mu);
  for (auto* cv : l->extra_cvs) cv->notify_all();
}

namespace {

constexpr int kRingSlots(int N) { return N + 1; }
constexpr double kTimeoutS = 600.0;

class LocalTransport final : public Transport {
 public:
  LocalTransport(std::shared_ptr<LocalLink> l, int k) : link_(std::move(l)), k_(k) {}
  ~LocalTransport() override {
    for (auto& e : owned_) cudaEventDestroy(e);
  }

  // replica: this context's index within its stage; rep_prev / rep_self / rep_next:
  // replicas of stages k−1, k, k+1. A replicated context owns channel `replica` of its
  // boundaries; an unreplicated one next to a replicated stage owns all of them. The
  // ring of a sender with several outgoing channels is split between them.
  st_status setup(float* ring_fwd, float* ring_bwd, size_t fwd_elems, size_t bwd_elems, int replica, int rep_prev,
                  int rep_self, int rep_next) {
    const int N = link_->N;
    const int R = kRingSlots(N);
    auto chans = [&](int rep_other) {
      std::vector<int> v;
      if (rep_self > 1) v.push_back(replica);
      else for (int c = 0; c < rep_other; ++c) v.push_back(c);
      return v;
    };
    // As sender: own the ring + ready events of my outgoing channels.
    if (k_ + 1 < N) {
      auto cs = chans(rep_next);
      const size_t e = fwd_elems / cs.size();
      for (size_t i = 0; i < cs.size(); ++i) ST_TRY(init_sender(*link_->fwd[k_][cs[i]], ring_fwd + i * e * R, e, R));
    }
    if (k_ > 0) {
      auto cs = chans(rep_prev);
      const size_t e = bwd_elems / cs.size();
      for (size_t i = 0; i < cs.size(); ++i) ST_TRY(init_sender(*link_->bwd[k_ - 1][cs[i]], ring_bwd + i * e * R, e, R));
    }
    // As receiver: consumed events of my incoming channels.
    if (k_ > 0)
      for (int c : chans(rep_prev)) ST_TRY(init_receiver(*link_->fwd[k_ - 1][c], R));
    if (k_ + 1 < N)
      for (int c : chans(rep_next)) ST_TRY(init_receiver(*link_->bwd[k_][c], R));
    return ST_OK;
  }

  st_status send(int kind, int64_t mb, const float* buf, size_t count, cudaStream_t s, int chan) override {
    switch (kind) {
      case CK_SEND_FWD: return do_send(*link_->fwd[k_][chan], mb, buf, count, s);
      case CK_SEND_BWD: return do_send(*link_->bwd[k_ - 1][chan], mb, buf, count, s);
      default: return set_error(ST_ERR_INPUT, "local transport: bad send kind %d", kind);
    }
  }
  st_status recv(int kind, int64_t mb, float* buf, size_t count, cudaStream_t s, int chan) override {
    switch (kind) {
      case CK_RECV_FWD: return do_recv(*link_->fwd[k_ - 1][chan], mb, buf, count, s);
      case CK_RECV_BWD: return do_recv(*link_->bwd[k_][chan], mb, buf, count, s);
      default: return set_error(ST_ERR_INPUT, "local transport: bad recv kind %d", kind);
    }
  }
  st_status poll() override {
    if (link_->aborted) return set_error(ST_ERR_STATE, "local transport: a peer stage failed (stage %d)", k_);
    return ST_OK;
  }
  void abort() override { abort_local_link(link_.get()); }

 private:
  st_status init_sender(Channel& ch, float* ring, size_t elems, int R) {
    if (!ring) return set_error(ST_ERR_INPUT, "local transport: missing ring buffer");
    std::lock_guard<std::mutex> g(ch.mu);
    ch.ring = ring;
    ch.elems = elems;
    ch.R = R;
    ch.ready.resize(R);
    for (int s = 0; s < R; ++s) {
      ST_CUDA_TRY(cudaEventCreateWithFlags(&ch.ready[s], cudaEventDisableTiming));
      owned_.push_back(ch.ready[s]);
    }
    return ST_OK;
  }
  st_status init_receiver(Channel& ch, int R) {
    std::lock_guard<std::mutex> g(ch.mu);
    ch.consumed.resize(R);
    ch.consumed_recorded.assign(R, false);
    for (int s = 0; s < R; ++s) {
      ST_CUDA_TRY(cudaEventCreateWithFlags(&ch.consumed[s], cudaEventDisableTiming));
      owned_.push_back(ch.consumed[s]);
    }
    return ST_OK;
  }

  st_status do_send(Channel& ch, int64_t mb, const float* buf, size_t count, cudaStream_t stream) {
    std::unique_lock<std::mutex> lk(ch.mu);
    if (count > ch.elems) return set_error(ST_ERR_SHAPE, "local send: %zu > ring slot %zu", count, ch.elems);
    // never reuse a slot whose previous message has not been taken by the receiver
    if (!ch.cv.wait_for(lk, std::chrono::duration<double>(kTimeoutS),
                        [&] { return link_->aborted || ch.sent - ch.received < ch.R; }))
      return set_error(ST_ERR_STATE, "local transport: send timeout (stage %d, mb %lld)", k_, (long long)mb);
    if (link_->aborted)
      return set_error(ST_ERR_STATE, "local transport: a peer stage failed (stage %d, send mb %lld)", k_, (long long)mb);
    const int slot = (int)(ch.sent % ch.R);
    if (ch.consumed_recorded.size() == (size_t)ch.R && ch.consumed_recorded[slot])
      ST_CUDA_TRY(cudaStreamWaitEvent(stream, ch.consumed[slot], 0));
    float* dst = ch.ring + (size_t)slot * ch.elems;
    ST_CUDA_TRY(cudaMemcpyAsync(dst, buf, count * sizeof(float), cudaMemcpyDefault, stream));
    ST_CUDA_TRY(cudaEventRecord(ch.ready[slot], stream));
    ch.q.push_back({mb, slot, count});
    ch.sent++;
    lk.unlock();
    ch.cv.notify_all();
    return ST_OK;
  }

  st_status do_recv(Channel& ch, int64_t mb, float* buf, size_t count, cudaStream_t stream) {
    std::unique_lock<std::mutex> lk(ch.mu);
    if (!ch.cv.wait_for(lk, std::chrono::duration<double>(kTimeoutS),
                        [&] { return link_->aborted || !ch.q.empty(); }))
      return set_error(ST_ERR_STATE, "local transport: receive timeout (stage %d, mb %lld)", k_, (long long)mb);
    if (link_->aborted)
      return set_error(ST_ERR_STATE, "local transport: a peer stage failed (stage %d, recv mb %lld)", k_, (long long)mb);
    Channel::Msg m = ch.q.front();
    ch.q.pop_front();
    if (m.mb != mb || m.count != count)
      return set_error(ST_ERR_STATE, "local transport: expected mb %lld (%zu floats), got mb %lld (%zu)",
                       (long long)mb, count, (long long)m.mb, m.count);
    ST_CUDA_TRY(cudaStreamWaitEvent(stream, ch.ready[m.slot], 0));
    ST_CUDA_TRY(cudaMemcpyAsync(buf, ch.ring + (size_t)m.slot * ch.elems, count * sizeof(float), cudaMemcpyDefault,
                                stream));
    ST_CUDA_TRY(cudaEventRecord(ch.consumed[m.slot], stream));
    ch.consumed_recorded[m.slot] = true;
    ch.received++;
    lk.unlock();
    ch.cv.notify_all();
    return ST_OK;
  }

  std::shared_ptr<LocalLink> link_;
  int k_;
  std::vector<cudaEvent_t> owned_;
};

}  // namespace

std::unique_ptr<Transport> make_local_transport(std::shared_ptr<LocalLink> link, int k, float* ring_fwd,
                                                float* ring_bwd, size_t fwd_elems, size_t bwd_elems, int replica,
                                                int rep_prev, int rep_self, int rep_next, st_status* err) {
  auto t = std::unique_ptr<LocalTransport>(new LocalTransport(std::move(link), k));
  *err = t->setup(ring_fwd, ring_bwd, fwd_elems, bwd_elems, replica, rep_prev, rep_self, rep_next);
  if (*err != ST_OK) return nullptr;
  return std::unique_ptr<Transport>(t.release());
}

// ------------------------------------------------------------------ LOCAL replica group
// In-place all-reduce of the R co-located replicas' gradient arenas (hybrid DP × PP):
// (1) every replica's backward finished (event + host barrier), (2) replica r sums
// slice r of all R arenas into all of them (disjoint memory per launch, fixed order),
// (3) every slice is summed (event + host barrier) before any replica's update reads
// its arena. A replica's next backward, which overwrites its arena, follows its own
// wait in (3), and the others' next reads of it follow the next (1).
struct ReplicaGroup {
  int R = 0;
  std::shared_ptr<LocalLink> link;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t gen = 0;
  std::vector<float*> G;
  std::vector<cudaEvent_t> ev_bwd, ev_sum;
  ~ReplicaGroup() {
    for (auto e : ev_bwd) cudaEventDestroy(e);
    for (auto e : ev_sum) cudaEventDestroy(e);
  }
  st_status barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t my = gen;
    if (++arrived == R) {
      arrived = 0;
      ++gen;
      lk.unlock();
      cv.notify_all();
      return ST_OK;
    }
    if (!cv.wait_for(lk, std::chrono::duration<double>(kTimeoutS), [&] { return gen != my || link->aborted; }))
      return set_error(ST_ERR_STATE, "replica group: barrier timeout");
    if (gen == my) return set_error(ST_ERR_STATE, "local transport: a peer stage failed (replica barrier)");
    return ST_OK;
  }
};

std::shared_ptr<ReplicaGroup> make_replica_group(int R, std::shared_ptr<LocalLink> link) {
  auto g = std::make_shared<ReplicaGroup>();
  g->R = R;
  g->link = link;
  g->G.assign(R, nullptr);
  g->ev_bwd.assign(R, nullptr);
  g->ev_sum.assign(R, nullptr);
  for (int r = 0; r < R; ++r) {
    cudaEventCreateWithFlags(&g->ev_bwd[r], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&g->ev_sum[r], cudaEventDisableTiming);
  }
  std::lock_guard<std::mutex> lk(link->extra_mu);
  link->extra_cvs.push_back(&g->cv);
  return g;
}

st_status replica_reduce_local(ReplicaGroup* g, int replica, float* G, size_t n, cudaStream_t s) {
  g->G[replica] = G;
  ST_CUDA_TRY(cudaEventRecord(g->ev_bwd[replica], s));
  ST_TRY(g->barrier());
  for (int j = 0; j < g->R; ++j)
    if (j != replica) ST_CUDA_TRY(cudaStreamWaitEvent(s, g->ev_bwd[j], 0));
  const size_t b = n * (size_t)replica / g->R, e = n * (size_t)(replica + 1) / g->R;
  ST_TRY(launch_replica_sum(g->G.data(), g->R, b, e, s));
  ST_CUDA_TRY(cudaEventRecord(g->ev_sum[replica], s));
  ST_TRY(g->barrier());
  for (int j = 0; j < g->R; ++j)
    if (j != replica) ST_CUDA_TRY(cudaStreamWaitEvent(s, g->ev_sum[j], 0));
  return ST_OK;
}

}  // namespace st
