// Stage-to-stage transports.
//
// NCCL: one process per GPU; every message is an ncclSend/ncclRecv between
// adjacent stages issued on the stage's compute stream, grouped exactly as the
// host comm plan says (schedule.cpp), so the peers' sequences pair in order.
//
// LOCAL: several stage contexts in one process (tests run an N-stage pipeline on
// one GPU; bench can oversubscribe). Each directed channel k→k+1 / k+1→k is a
// host queue of (mini-batch, ring slot) records plus a device ring owned by the
// sender: send = stream-ordered copy into the ring slot + CUDA event; receive =
// blocking pop, wait on the event, copy out, record a "consumed" event the sender
// waits on before reusing the slot. Same plan, same ordering per channel.
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <deque>
#include <mutex>

#include "engine.hpp"

namespace st {

// ------------------------------------------------------------------ NCCL
namespace {

class NcclTransport final : public Transport {
 public:
  NcclTransport(ncclComm_t c, int N, int k) : comm_(c), N_(N), k_(k) {}
  ~NcclTransport() override {
    if (comm_) ncclCommDestroy(comm_);
  }
  bool eager_groups() const override { return true; }
  st_status group(const CommOp* ops, int n, cudaStream_t stream) override {
    ncclResult_t r = ncclGroupStart();
    if (r != ncclSuccess) return set_error(ST_ERR_NCCL, "ncclGroupStart: %s", ncclGetErrorString(r));
    for (int i = 0; i < n && r == ncclSuccess; ++i) {
      const CommOp& o = ops[i];
      switch (o.kind) {
        case CK_SEND_FWD: r = ncclSend(o.buf, o.count, ncclFloat32, k_ + 1, comm_, stream); break;
        case CK_RECV_FWD: r = ncclRecv(o.buf, o.count, ncclFloat32, k_ - 1, comm_, stream); break;
        case CK_SEND_BWD: r = ncclSend(o.buf, o.count, ncclFloat32, k_ - 1, comm_, stream); break;
        case CK_RECV_BWD: r = ncclRecv(o.buf, o.count, ncclFloat32, k_ + 1, comm_, stream); break;
        default: r = ncclInvalidArgument;
      }
    }
    ncclResult_t r2 = ncclGroupEnd();
    if (r != ncclSuccess) return set_error(ST_ERR_NCCL, "ncclSend/Recv: %s", ncclGetErrorString(r));
    if (r2 != ncclSuccess) return set_error(ST_ERR_NCCL, "ncclGroupEnd: %s", ncclGetErrorString(r2));
    return ST_OK;
  }

 private:
  ncclComm_t comm_;
  int N_, k_;
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
  ncclComm_t comm = nullptr;
  ncclResult_t r = ncclCommInitRank(&comm, N, uid, k);
  if (r != ncclSuccess) {
    *err = set_error(ST_ERR_NCCL, "ncclCommInitRank(N=%d, rank=%d): %s", N, k, ncclGetErrorString(r));
    return nullptr;
  }
  return std::unique_ptr<Transport>(new NcclTransport(comm, N, k));
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

namespace {

constexpr int kRingSlots(int N) { return N + 1; }
constexpr double kTimeoutS = 600.0;

class LocalTransport final : public Transport {
 public:
  LocalTransport(std::shared_ptr<LocalLink> l, int k) : link_(std::move(l)), k_(k) {}
  ~LocalTransport() override {
    for (auto& e : owned_) cudaEventDestroy(e);
  }
  bool eager_groups() const override { return false; }

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

  st_status group(const CommOp* ops, int n, cudaStream_t stream) override {
    for (int pass = 0; pass < 2; ++pass)  // sends first, then receives
      for (int i = 0; i < n; ++i) {
        const CommOp& o = ops[i];
        const bool is_send = (o.kind == CK_SEND_FWD || o.kind == CK_SEND_BWD);
        if (is_send != (pass == 0)) continue;
        switch (o.kind) {
          case CK_SEND_FWD: ST_TRY(send(*link_->fwd[k_], o, stream)); break;
          case CK_SEND_BWD: ST_TRY(send(*link_->bwd[k_ - 1], o, stream)); break;
          case CK_RECV_FWD: ST_TRY(recv(*link_->fwd[k_ - 1], o, stream)); break;
          case CK_RECV_BWD: ST_TRY(recv(*link_->bwd[k_], o, stream)); break;
          default: return set_error(ST_ERR_INPUT, "local transport: bad op kind %d", o.kind);
        }
      }
    return ST_OK;
  }

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

  st_status send(Channel& ch, const CommOp& o, cudaStream_t stream) {
    std::unique_lock<std::mutex> lk(ch.mu);
    if (o.count > ch.elems) return set_error(ST_ERR_SHAPE, "local send: %zu > ring slot %zu", o.count, ch.elems);
    // never reuse a slot whose previous message has not been taken by the receiver
    if (!ch.cv.wait_for(lk, std::chrono::duration<double>(kTimeoutS), [&] { return ch.sent - ch.received < ch.R; }))
      return set_error(ST_ERR_STATE, "local transport: send timeout (stage %d, mb %lld)", k_, (long long)o.mb);
    const int slot = (int)(ch.sent % ch.R);
    if (ch.consumed_recorded.size() == (size_t)ch.R && ch.consumed_recorded[slot])
      ST_CUDA_TRY(cudaStreamWaitEvent(stream, ch.consumed[slot], 0));
    float* dst = ch.ring + (size_t)slot * ch.elems;
    ST_CUDA_TRY(cudaMemcpyAsync(dst, o.buf, o.count * sizeof(float), cudaMemcpyDefault, stream));
    ST_CUDA_TRY(cudaEventRecord(ch.ready[slot], stream));
    ch.q.push_back({o.mb, slot, o.count});
    ch.sent++;
    lk.unlock();
    ch.cv.notify_all();
    return ST_OK;
  }

  st_status recv(Channel& ch, const CommOp& o, cudaStream_t stream) {
    std::unique_lock<std::mutex> lk(ch.mu);
    if (!ch.cv.wait_for(lk, std::chrono::duration<double>(kTimeoutS), [&] { return !ch.q.empty(); }))
      return set_error(ST_ERR_STATE, "local transport: receive timeout (stage %d, mb %lld)", k_, (long long)o.mb);
    Channel::Msg m = ch.q.front();
    ch.q.pop_front();
    if (m.mb != o.mb || m.count != o.count)
      return set_error(ST_ERR_STATE, "local transport: expected mb %lld (%zu floats), got mb %lld (%zu)",
                       (long long)o.mb, o.count, (long long)m.mb, m.count);
    ST_CUDA_TRY(cudaStreamWaitEvent(stream, ch.ready[m.slot], 0));
    ST_CUDA_TRY(cudaMemcpyAsync(o.buf, ch.ring + (size_t)m.slot * ch.elems, o.count * sizeof(float),
                                cudaMemcpyDefault, stream));
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
