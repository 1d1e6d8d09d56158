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
  NcclTransport(ncclComm_t f, ncclComm_t b, int N, int k) : fwd_(f), bwd_(b), N_(N), k_(k) {}
  ~NcclTransport() override {
    if (aborted_) return;
    if (fwd_) ncclCommDestroy(fwd_);
    if (bwd_) ncclCommDestroy(bwd_);
  }
  st_status send(int kind, int64_t mb, const float* buf, size_t count, cudaStream_t s) override {
    const bool f = kind == CK_SEND_FWD;
    if (!f && kind != CK_SEND_BWD) return set_error(ST_ERR_INPUT, "nccl send: bad kind %d", kind);
    const int peer = f ? k_ + 1 : k_ - 1;
    if (peer < 0 || peer >= N_) return set_error(ST_ERR_STATE, "stage %d: no peer %d", k_, peer);
    ncclResult_t r = ncclSend(buf, count, ncclFloat32, peer, f ? fwd_ : bwd_, s);
    if (r != ncclSuccess)
      return set_error(ST_ERR_NCCL, "stage %d: ncclSend(mb %lld -> %d): %s", k_, (long long)mb, peer,
                       ncclGetErrorString(r));
    return ST_OK;
  }
  st_status recv(int kind, int64_t mb, float* buf, size_t count, cudaStream_t s) override {
    const bool f = kind == CK_RECV_FWD;
    if (!f && kind != CK_RECV_BWD) return set_error(ST_ERR_INPUT, "nccl recv: bad kind %d", kind);
    const int peer = f ? k_ - 1 : k_ + 1;
    if (peer < 0 || peer >= N_) return set_error(ST_ERR_STATE, "stage %d: no peer %d", k_, peer);
    ncclResult_t r = ncclRecv(buf, count, ncclFloat32, peer, f ? fwd_ : bwd_, s);
    if (r != ncclSuccess)
      return set_error(ST_ERR_NCCL, "stage %d: ncclRecv(mb %lld <- %d): %s", k_, (long long)mb, peer,
                       ncclGetErrorString(r));
    return ST_OK;
  }
  st_status poll() override {
    if (aborted_) return set_error(ST_ERR_NCCL, "stage %d: communicators were aborted", k_);
    for (ncclComm_t c : {fwd_, bwd_}) {
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
    ncclCommAbort(fwd_);
    t.join();
  }

 private:
  ncclComm_t fwd_, bwd_;
  int N_, k_;
  bool aborted_ = false;
};

}  // namespace

std::unique_ptr<Transport> make_nccl_transport(const uint8_t id[128], int N, int k, int device, st_status* err) {
  *err = ST_OK;
  if (N == 1) return nullptr;  // a 1-stage pipeline never communicates
  ncclUniqueId uid;
  static_assert(sizeof(uid.internal) == 128, "ncclUniqueId size");
  memcpy(uid.internal, id, 128);
  if (cudaSetDevice(device) != cudaSuccess) {
    *err = set_error(ST_ERR_CUDA, "cudaSetDevice(%d)", device);
    return nullptr;
  }
  ncclComm_t f = nullptr, b = nullptr;
  ncclResult_t r = ncclCommInitRank(&f, N, uid, k);
  if (r != ncclSuccess) {
    *err = set_error(ST_ERR_NCCL, "ncclCommInitRank(N=%d, rank=%d): %s", N, k, ncclGetErrorString(r));
    return nullptr;
  }
  // the gradient-direction communicator: same ranks, same order (collective over all stages)
  r = ncclCommSplit(f, 0, k, &b, nullptr);
  if (r != ncclSuccess || !b) {
    *err = set_error(ST_ERR_NCCL, "ncclCommSplit (gradient communicator, rank %d): %s", k, ncclGetErrorString(r));
    ncclCommDestroy(f);
    return nullptr;
  }
  return std::unique_ptr<Transport>(new NcclTransport(f, b, N, k));
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
  std::vector<std::unique_ptr<Channel>> fwd, bwd;  // fwd[k]: k→k+1, bwd[k]: k+1→k
};

std::shared_ptr<LocalLink> make_local_link(int N) {
  auto l = std::make_shared<LocalLink>();
  l->N = N;
  for (int k = 0; k + 1 < N; ++k) {
    l->fwd.emplace_back(new Channel());
    l->bwd.emplace_back(new Channel());
  }
  return l;
}

void abort_local_link(LocalLink* l) {
  if (!l) return;
  l->aborted = true;
  for (auto* v : {&l->fwd, &l->bwd})
    for (auto& ch : *v) {
      { std::lock_guard<std::mutex> g(ch->mu); }
      ch->cv.notify_all();
    }
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

  st_status setup(float* ring_fwd, float* ring_bwd, size_t fwd_elems, size_t bwd_elems) {
    const int N = link_->N;
    const int R = kRingSlots(N);
    // As sender: own the ring + ready events of my outgoing channels.
    if (k_ + 1 < N) ST_TRY(init_sender(*link_->fwd[k_], ring_fwd, fwd_elems, R));
    if (k_ > 0) ST_TRY(init_sender(*link_->bwd[k_ - 1], ring_bwd, bwd_elems, R));
    // As receiver: consumed events of my incoming channels.
    if (k_ > 0) ST_TRY(init_receiver(*link_->fwd[k_ - 1], R));
    if (k_ + 1 < N) ST_TRY(init_receiver(*link_->bwd[k_], R));
    return ST_OK;
  }

  st_status send(int kind, int64_t mb, const float* buf, size_t count, cudaStream_t s) override {
    switch (kind) {
      case CK_SEND_FWD: return do_send(*link_->fwd[k_], mb, buf, count, s);
      case CK_SEND_BWD: return do_send(*link_->bwd[k_ - 1], mb, buf, count, s);
      default: return set_error(ST_ERR_INPUT, "local transport: bad send kind %d", kind);
    }
  }
  st_status recv(int kind, int64_t mb, float* buf, size_t count, cudaStream_t s) override {
    switch (kind) {
      case CK_RECV_FWD: return do_recv(*link_->fwd[k_ - 1], mb, buf, count, s);
      case CK_RECV_BWD: return do_recv(*link_->bwd[k_], mb, buf, count, s);
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
                                                float* ring_bwd, size_t fwd_elems, size_t bwd_elems,
                                                st_status* err) {
  auto t = std::unique_ptr<LocalTransport>(new LocalTransport(std::move(link), k));
  *err = t->setup(ring_fwd, ring_bwd, fwd_elems, bwd_elems);
  if (*err != ST_OK) return nullptr;
  return std::unique_ptr<Transport>(t.release());
}

}  // namespace st
