// P2P transport: inter-stage transfer fused into the producing kernels over peer
// memory ("activations and gradients are transferred
// between GPUs", "sent to the next GPU ... to hide the latency").
//
// No separate copy or send exists. Stage k's last forward GEMM writes its output
// straight into stage k+1's stash slot for that mini-batch (the buffer k+1's first
// layer reads and its backward re-reads), and stage k+1's layer-0 dX GEMM writes the
// masked gradient straight into stage k's gradient ring slot. The peer buffers are
// mapped into this process: CUDA IPC across processes (NVLink / NVSwitch peer memory
// between GPUs, or two processes sharing one GPU), plain pointers between contexts of
// one process. Hand-over is by monotonically increasing 64-bit flags in the WAITER's
// memory, written by the peer with a system-scope release after the producing kernel
// completed (p2p_signal_kernel) and polled with a system-scope acquire by a one-thread
// kernel on the waiter's compute stream (p2p_wait_kernel), so the stream order carries
// the dependency with no host involvement:
//
//   flag              lives on   written by   value after mini-batch mb
//   FWD_READY[slot]   k+1        k            base + mb + 1 (activation in slot mb % S_{k+1})
//   BWD_READY[b]      k          k+1          base + mb + 1 (gradient in ring slot mb % 2)
//   NEXT_BWD_COUNT    k          k+1          base + mb + 1 (k+1 finished B(mb): its stash slot is free)
//   PREV_BWD_COUNT    k+1        k            base + mb + 1 (k finished B(mb): its ring slot is free)
//
// `base` = backwards this stage completed before the current session (identical on
// every stage at a session start), so the flags keep increasing across sessions. A
// wait kernel also watches a host-mapped abort word: a hung or dead peer is handled
// by the engine's wait loop (timeout -> abort), which releases spinning kernels.
#include <unistd.h>

#include <cstring>

#include "engine.hpp"

namespace st {

namespace {

__global__ void p2p_wait_kernel(const long long* flag, long long target, const volatile int* abort_word,
                                int* failed) {
  if (threadIdx.x != 0) return;
  unsigned ns = 32;
  for (;;) {
    long long v;
    asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= target) return;
    if (*abort_word) {
      atomicExch(failed, 1);
      return;
    }
    __nanosleep(ns);
    if (ns < 2048) ns <<= 1;
  }
}

__global__ void p2p_signal_kernel(long long* flag, long long value) {
  if (threadIdx.x != 0) return;
  __threadfence_system();  // the producing kernel's peer stores precede the flag (stream order + fence)
  asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(flag), "l"(value) : "memory");
}

// the part of the exported descriptor that locates one buffer
struct Region {
  cudaIpcMemHandle_t h;  // of the allocation containing the buffer
  uint64_t off;          // byte offset of the buffer inside that allocation
  uint64_t raw;          // the pointer itself (used by contexts of the same process)
};

struct Desc {
  uint32_t magic, version;
  int32_t pid, device, k, N;
  int64_t R, in_first, out_last;
  int32_t S;  // stash slots
  int32_t pad;
  int64_t slot_elems, off0;  // floats per stash slot, offset of the stage input inside a slot
  int64_t ring_elems;        // floats between the two gradient ring slots
  Region stash, ring, flags;
};
static_assert(sizeof(Desc) <= sizeof(st_p2p_desc), "st_p2p_desc too small");
constexpr uint32_t kMagic = 0x53545032u;  // "STP2"

using AddrRangeFn = int (*)(unsigned long long*, size_t*, unsigned long long);

st_status region_of(const void* p, Region* r) {
  static AddrRangeFn fn = nullptr;
  if (!fn) {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &q, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess)
      return set_error(ST_ERR_CUDA, "p2p: cuMemGetAddressRange unavailable");
    fn = reinterpret_cast<AddrRangeFn>(q);
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (fn(&base, &size, (unsigned long long)(uintptr_t)p) != 0)
    return set_error(ST_ERR_INPUT, "p2p: %p is not device memory", p);
  memset(r, 0, sizeof *r);
  r->raw = (uint64_t)(uintptr_t)p;
  r->off = (uint64_t)(uintptr_t)p - base;
  const cudaError_t e = cudaIpcGetMemHandle(&r->h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_error(ST_ERR_INPUT,
                     "p2p: cudaIpcGetMemHandle: %s (the stash / work arenas must be cudaMalloc-backed: "
                     "no expandable segments)",
                     cudaGetErrorString(e));
  }
  return ST_OK;
}

}  // namespace

// per-context state of the P2P transport
struct P2pState {
  long long* flags = nullptr;  // own flag block (device, library-owned)
  int* abort_host = nullptr;   // host-mapped abort word
  int* abort_dev = nullptr;
  int* failed = nullptr;       // set by a wait kernel released by an abort (device)
  long long* prev_flags = nullptr;
  long long* next_flags = nullptr;
  float* next_stash = nullptr;
  int next_S = 0;
  int64_t next_slot_elems = 0, next_off0 = 0;
  float* prev_ring = nullptr;
  int64_t prev_ring_elems = 0;
  std::vector<void*> opened;  // IPC mappings to close
  int64_t base = 0;           // backwards completed before the current session
  int64_t bwd_total = 0;      // backwards completed so far
};

enum { F_FWD_READY = 0, F_BWD_READY = 64, F_NEXT_BWD_COUNT = 66, F_PREV_BWD_COUNT = 67, F_COUNT = 68 };

namespace {

class P2pTransport final : public Transport {
 public:
  explicit P2pTransport(P2pState* s) : s_(s) {}
  st_status send(int, int64_t, const float*, size_t, cudaStream_t, int) override {
    return set_error(ST_ERR_STATE, "p2p transport: messages are written by the producing kernels");
  }
  st_status recv(int, int64_t, float*, size_t, cudaStream_t, int) override {
    return set_error(ST_ERR_STATE, "p2p transport: messages are written by the producing kernels");
  }
  st_status poll() override {
    if (*reinterpret_cast<volatile int*>(s_->abort_host))
      return set_error(ST_ERR_STATE, "p2p transport: aborted (a peer stage failed or hung)");
    return ST_OK;
  }
  void abort() override { *reinterpret_cast<volatile int*>(s_->abort_host) = 1; }

 private:
  P2pState* s_;
};

}  // namespace

st_status p2p_alloc(st_ctx* c) {
  if (c->N > 65) return set_error(ST_ERR_INPUT, "p2p transport: at most 65 stages (64 stash-slot flags)");
  c->p2p = new P2pState();
  ST_CUDA_TRY(cudaMalloc(&c->p2p->flags, F_COUNT * sizeof(long long) + 64));
  ST_CUDA_TRY(cudaMemset(c->p2p->flags, 0, F_COUNT * sizeof(long long) + 64));
  c->p2p->failed = reinterpret_cast<int*>(c->p2p->flags + F_COUNT);
  ST_CUDA_TRY(cudaHostAlloc(&c->p2p->abort_host, sizeof(int), cudaHostAllocMapped));
  *c->p2p->abort_host = 0;
  ST_CUDA_TRY(cudaHostGetDevicePointer(&c->p2p->abort_dev, c->p2p->abort_host, 0));
  c->tp.reset(new P2pTransport(c->p2p));
  return ST_OK;
}

void p2p_free(st_ctx* c) {
  if (!c->p2p) return;
  for (void* p : c->p2p->opened) cudaIpcCloseMemHandle(p);
  if (c->p2p->flags) cudaFree(c->p2p->flags);
  if (c->p2p->abort_host) cudaFreeHost(c->p2p->abort_host);
  delete c->p2p;
  c->p2p = nullptr;
}

st_status p2p_export(st_ctx* c, st_p2p_desc* out) {
  if (!c->p2p) return set_error(ST_ERR_STATE, "p2p_export: context was not created with ST_TRANSPORT_P2P");
  ST_CUDA_TRY(cudaSetDevice(c->device));
  Desc d{};
  d.magic = kMagic;
  d.version = 1;
  d.pid = (int32_t)getpid();
  d.device = c->device;
  d.k = c->k;
  d.N = c->N;
  d.R = c->R;
  d.in_first = c->in_first;
  d.out_last = c->out_last;
  d.S = c->S;
  d.slot_elems = c->slot_elems;
  d.off0 = c->layers[0].stash_off;
  d.ring_elems = c->recv_bwd2[1] && c->recv_bwd2[0] ? (int64_t)(c->recv_bwd2[1] - c->recv_bwd2[0]) : 0;
  if (!c->first_stage) ST_TRY(region_of(c->stash, &d.stash));
  if (!c->last_stage) ST_TRY(region_of(c->recv_bwd2[0], &d.ring));
  ST_TRY(region_of(c->p2p->flags, &d.flags));
  memset(out, 0, sizeof *out);
  memcpy(out->bytes, &d, sizeof d);
  return ST_OK;
}

static st_status open_region(st_ctx* c, const Desc& d, const Region& r, void** p) {
  if (d.pid == (int32_t)getpid()) {  // a context of this process: its pointer is valid here
    // Contexts of one process on one GPU share that device's hardware work queues
    // (streams are multiplexed onto CUDA_DEVICE_MAX_CONNECTIONS channels, and torch
    // alone creates 64 pool streams): a spinning wait kernel can end up ahead of the very
    // kernels it waits for in one channel and neither progresses (measured: a 2-stage
    // pipeline hangs). Separate processes have separate channels — run P2P stages that
    // share a GPU as separate processes (or use ST_TRANSPORT_LOCAL in one process).
    if (d.device == c->device)
      return set_error(ST_ERR_INPUT,
                       "p2p: stages %d and %d are contexts of one process on GPU %d — run them as separate "
                       "processes (their wait kernels would share hardware queues) or use ST_TRANSPORT_LOCAL",
                       c->k, d.k, c->device);
    *p = reinterpret_cast<void*>((uintptr_t)r.raw);
    return ST_OK;
  }
  void* base = nullptr;
  const cudaError_t e = cudaIpcOpenMemHandle(&base, r.h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_error(ST_ERR_CUDA, "p2p: cudaIpcOpenMemHandle (stage %d -> %d): %s", c->k, d.k,
                     cudaGetErrorString(e));
  }
  c->p2p->opened.push_back(base);
  *p = static_cast<char*>(base) + r.off;
  return ST_OK;
}

st_status p2p_connect(st_ctx* c, const st_p2p_desc* prev, const st_p2p_desc* next) {
  if (!c->p2p) return set_error(ST_ERR_STATE, "p2p_connect: context was not created with ST_TRANSPORT_P2P");
  if (c->first_stage != !prev || c->last_stage != !next)
    return set_error(ST_ERR_INPUT, "p2p_connect: stage %d of %d needs %s prev and %s next descriptor", c->k, c->N,
                     c->first_stage ? "no" : "a", c->last_stage ? "no" : "a");
  ST_CUDA_TRY(cudaSetDevice(c->device));
  if (prev) {
    Desc d;
    memcpy(&d, prev->bytes, sizeof d);
    if (d.magic != kMagic || d.version != 1) return set_error(ST_ERR_INPUT, "p2p_connect: bad prev descriptor");
    if (d.k != c->k - 1 || d.N != c->N || d.R != c->R || d.out_last != c->in_first)
      return set_error(ST_ERR_SHAPE, "p2p_connect: prev descriptor (stage %d/%d, %lld x %lld) does not feed stage "
                       "%d/%d (%lld x %d)", d.k, d.N, (long long)d.R, (long long)d.out_last, c->k, c->N,
                       (long long)c->R, c->in_first);
    void* p = nullptr;
    ST_TRY(open_region(c, d, d.flags, &p));
    c->p2p->prev_flags = static_cast<long long*>(p);
    ST_TRY(open_region(c, d, d.ring, &p));
    c->p2p->prev_ring = static_cast<float*>(p);
    c->p2p->prev_ring_elems = d.ring_elems;
  }
  if (next) {
    Desc d;
    memcpy(&d, next->bytes, sizeof d);
    if (d.magic != kMagic || d.version != 1) return set_error(ST_ERR_INPUT, "p2p_connect: bad next descriptor");
    if (d.k != c->k + 1 || d.N != c->N || d.R != c->R || d.in_first != c->out_last)
      return set_error(ST_ERR_SHAPE, "p2p_connect: next descriptor (stage %d/%d) does not follow stage %d/%d", d.k,
                       d.N, c->k, c->N);
    void* p = nullptr;
    ST_TRY(open_region(c, d, d.flags, &p));
    c->p2p->next_flags = static_cast<long long*>(p);
    ST_TRY(open_region(c, d, d.stash, &p));
    c->p2p->next_stash = static_cast<float*>(p);
    c->p2p->next_S = d.S;
    c->p2p->next_slot_elems = d.slot_elems;
    c->p2p->next_off0 = d.off0;
  }
  return ST_OK;
}

static st_status launch_wait(st_ctx* c, long long* flag, long long target) {
  p2p_wait_kernel<<<1, 32, 0, c->stream>>>(flag, target, c->p2p->abort_dev, c->p2p->failed);
  ST_CUDA_TRY(cudaGetLastError());
  c->launches += 1;
  return ST_OK;
}

static st_status launch_signal(st_ctx* c, long long* flag, long long value) {
  p2p_signal_kernel<<<1, 32, 0, c->stream>>>(flag, value);
  ST_CUDA_TRY(cudaGetLastError());
  c->launches += 1;
  return ST_OK;
}

void p2p_begin_session(st_ctx* c) {
  if (c->p2p) c->p2p->base = c->p2p->bwd_total;
}

// before F(mb): the input has landed (k > 0); the peer's stash slot for the output is
// free (k < N−1) — the output pointer is that slot
st_status p2p_before_forward(st_ctx* c, int64_t mb) {
  P2pState* s = c->p2p;
  if (!c->first_stage) ST_TRY(launch_wait(c, s->flags + F_FWD_READY + mb % c->S, s->base + mb + 1));
  if (!c->last_stage) {
    if (!s->next_stash) return set_error(ST_ERR_STATE, "stage %d: p2p transport not connected", c->k);
    const int64_t need = std::max<int64_t>(s->base, s->base + mb - s->next_S + 1);
    if (need > 0) ST_TRY(launch_wait(c, s->flags + F_NEXT_BWD_COUNT, need));
    c->send_fwd = s->next_stash + (mb % s->next_S) * s->next_slot_elems + s->next_off0;
  }
  return ST_OK;
}

st_status p2p_after_forward(st_ctx* c, int64_t mb) {
  P2pState* s = c->p2p;
  if (!c->last_stage) ST_TRY(launch_signal(c, s->next_flags + F_FWD_READY + mb % s->next_S, s->base + mb + 1));
  return ST_OK;
}

// before B(mb): the gradient from k+1 has landed (k < N−1); the peer's ring slot for
// the layer-0 dX is free (k > 0) — the dX output pointer is that slot
st_status p2p_before_backward(st_ctx* c, int64_t mb) {
  P2pState* s = c->p2p;
  if (!c->last_stage) {
    ST_TRY(launch_wait(c, s->flags + F_BWD_READY + mb % 2, s->base + mb + 1));
    c->recv_bwd = c->recv_bwd2[mb % 2];
  }
  if (!c->first_stage) {
    if (!s->prev_ring) return set_error(ST_ERR_STATE, "stage %d: p2p transport not connected", c->k);
    const int64_t need = std::max<int64_t>(s->base, s->base + mb - 2 + 1);
    if (need > 0) ST_TRY(launch_wait(c, s->flags + F_PREV_BWD_COUNT, need));
    c->send_bwd = s->prev_ring + (mb % 2) * s->prev_ring_elems;
  }
  return ST_OK;
}

// right after the layer-0 dX of B(mb) (k > 0): the gradient is in k−1's ring slot
st_status p2p_after_dx(st_ctx* c, int64_t mb) {
  P2pState* s = c->p2p;
  return launch_signal(c, s->prev_flags + F_BWD_READY + mb % 2, s->base + mb + 1);
}

// after B(mb) (every reader of the stash slot and of the ring slot joined): tell both
// neighbours
st_status p2p_after_backward(st_ctx* c, int64_t mb) {
  P2pState* s = c->p2p;
  if (!c->first_stage) ST_TRY(launch_signal(c, s->prev_flags + F_NEXT_BWD_COUNT, s->base + mb + 1));
  if (!c->last_stage) ST_TRY(launch_signal(c, s->next_flags + F_PREV_BWD_COUNT, s->base + mb + 1));
  s->bwd_total += 1;
  return ST_OK;
}

std::string p2p_describe(st_ctx* c) {
  long long f[F_COUNT] = {};
  // the flag block is read with a plain copy on a fresh stream (the compute stream may
  // still hold released waits)
  cudaStream_t s;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return "";
  cudaMemcpyAsync(f, c->p2p->flags, sizeof f, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  char buf[512];
  int n = snprintf(buf, sizeof buf, "; p2p base %lld, backwards %lld, flags: fwd_ready", (long long)c->p2p->base,
                   (long long)c->p2p->bwd_total);
  for (int i = 0; i < c->S && i < 8 && n < (int)sizeof buf; ++i) n += snprintf(buf + n, sizeof buf - n, " %lld", f[F_FWD_READY + i]);
  if (n < (int)sizeof buf)
    snprintf(buf + n, sizeof buf - n, ", bwd_ready %lld %lld, next_bwd %lld, prev_bwd %lld", f[F_BWD_READY],
             f[F_BWD_READY + 1], f[F_NEXT_BWD_COUNT], f[F_PREV_BWD_COUNT]);
  return buf;
}

// a wait released by an abort leaves its failure in device memory (read at sync points)
st_status p2p_check(st_ctx* c) {
  if (!c->p2p) return ST_OK;
  int failed = 0;
  ST_CUDA_TRY(cudaMemcpy(&failed, c->p2p->failed, sizeof failed, cudaMemcpyDeviceToHost));
  if (failed) return set_error(ST_ERR_STATE, "stage %d: p2p wait released by an abort (peer failed or hung)", c->k);
  return ST_OK;
}

}  // namespace st
