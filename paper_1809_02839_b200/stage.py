"""PyTorch-side owner of one pipeline stage context (memory + stream plumbing only).

`Stage` allocates the arenas `st_query_sizes` asks for as CUDA tensors, binds
them with `st_init`, and forwards every verb to the C-ABI. All arithmetic of the
SpecTrain step (GEMMs, CE, the fused update/prediction) happens in
libspectrain.so's kernels.
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib as L
from ._lib import check, lib

Layers = Sequence[Tuple[int, int, int, int]]  # (n_in, n_out, act, bias)


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


class Stage:
    """Stage k of an N-stage SpecTrain pipeline on `device`.

    layers/cuts describe the WHOLE network (the same on every stage); the
    context keeps layers [cuts[k-1], cuts[k])."""

    def __init__(self, layers: Layers, cuts: Sequence[int], stage: int, batch: int, lr: float, gamma: float = 0.9,
                 pred: int = L.ST_PRED_SPECTRAIN, momentum: int = L.ST_MOMENTUM_EMA, gemm: int = L.ST_GEMM_FP32X3,
                 transport: int = L.ST_TRANSPORT_NCCL, device: int = 0, max_minibatches: int = 256,
                 nccl_id: Optional[bytes] = None, stream: Optional[torch.cuda.Stream] = None, seq_len: int = 1,
                 comm_streams: Optional[Tuple[torch.cuda.Stream, torch.cuda.Stream]] = None,
                 replicas: Optional[Sequence[int]] = None, replica: int = 0):
        """replicas / replica: hybrid data × pipeline parallelism (st_config.replicas; `batch`
        stays the global mini-batch, a replica of a replicated stage computes its row slice)."""
        self.layers = [tuple(int(v) for v in l) for l in layers]
        self.replicas = list(replicas) if replicas is not None else None
        self.replica = replica
        self.cuts = list(cuts)
        self.k = stage
        self.N = len(cuts) + 1
        self.batch = batch
        self.device = torch.device("cuda", device)
        self.seq_len = seq_len
        self.cfg, self._keep = L.make_config(self.layers, self.cuts, stage, batch, lr, gamma, pred, momentum, gemm,
                                             transport, device, max_minibatches, nccl_id, seq_len, replicas,
                                             replica)
        self.sizes = L.query_sizes(self.cfg)
        self.stream = stream if stream is not None else torch.cuda.Stream(device=self.device)
        # activation / gradient transfer streams (None: the library creates its own)
        self.comm_streams = comm_streams

        def buf(nbytes: int) -> Optional[torch.Tensor]:
            if nbytes <= 0:
                return None
            return torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)

        s = self.sizes
        # a parameter-free stage (e.g. a lone max-pool) still binds 256-byte arenas
        self.W, self.V, self.G = buf(max(256, s.w_bytes)), buf(max(256, s.v_bytes)), buf(max(256, s.g_bytes))
        self.WF, self.WB = buf(s.wf_bytes), buf(s.wb_bytes)
        self.stash, self.work = buf(max(256, s.stash_bytes)), buf(max(256, s.work_bytes))
        bufs = L.StBuffers(_ptr(self.W), _ptr(self.V), _ptr(self.G), _ptr(self.WF), _ptr(self.WB),
                           _ptr(self.stash), _ptr(self.work))
        self.ctx = ctypes.c_void_p()
        cf, cb = (None, None) if comm_streams is None else (comm_streams[0].cuda_stream, comm_streams[1].cuda_stream)
        check(lib.st_init(ctypes.byref(self.cfg), ctypes.byref(bufs), ctypes.c_void_p(self.stream.cuda_stream),
                          ctypes.c_void_p(cf), ctypes.c_void_p(cb), ctypes.byref(self.ctx)))

    # ---- lifecycle ------------------------------------------------------------
    def close(self) -> None:
        if self.ctx:
            lib.st_destroy(self.ctx)
            self.ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def params(self) -> int:
        return int(self.sizes.params)

    @property
    def is_first(self) -> bool:
        return self.k == 0

    @property
    def is_last(self) -> bool:
        return self.k == self.N - 1

    def set_params(self, host) -> None:
        """host: a float32 numpy array, or a contiguous float32 CUDA tensor on this device."""
        if isinstance(host, torch.Tensor):
            assert host.dtype == torch.float32 and host.is_contiguous()
            torch.cuda.synchronize(host.device)
            check(lib.st_set_params(self.ctx, host.data_ptr(), host.numel()))
            return
        a = np.ascontiguousarray(host, dtype=np.float32)
        check(lib.st_set_params(self.ctx, a.ctypes.data, a.size))

    def get_params(self) -> Tuple[np.ndarray, np.ndarray, int]:
        W = np.empty(self.params, np.float32)
        V = np.empty(self.params, np.float32)
        ver = ctypes.c_int64()
        check(lib.st_get_params(self.ctx, W.ctypes.data, V.ctypes.data, W.size, ctypes.byref(ver)))
        return W, V, ver.value

    # ---- verbs ------------------------------------------------------------------
    def forward(self, mb: int, x: Optional[torch.Tensor] = None, y: Optional[torch.Tensor] = None,
                want_loss: bool = False) -> Optional[float]:
        loss = ctypes.c_float(float("nan"))
        check(lib.st_stage_forward(self.ctx, mb, _ptr(x), _ptr(y), ctypes.byref(loss) if want_loss else None))
        return loss.value if want_loss else None

    def backward(self, mb: int) -> None:
        check(lib.st_stage_backward(self.ctx, mb))

    def predict_and_update(self) -> None:
        check(lib.st_predict_and_update(self.ctx))

    def step(self, x: Optional[torch.Tensor] = None, y: Optional[torch.Tensor] = None) -> L.StStepInfo:
        info = L.StStepInfo()
        check(lib.st_step(self.ctx, _ptr(x), _ptr(y), ctypes.byref(info)))
        return info

    def run(self, M: int, xs: Optional[torch.Tensor] = None, ys: Optional[torch.Tensor] = None,
            want_losses: bool = False) -> Optional[np.ndarray]:
        out = np.empty(max(1, M), np.float32) if (want_losses and self.is_last) else None
        check(lib.st_run(self.ctx, M, _ptr(xs), _ptr(ys), out.ctypes.data if out is not None else None))
        return out[:M] if out is not None else None

    def run_host(self, M: int, xs_host, ys_host, losses_host: Optional[np.ndarray] = None) -> None:
        """End-to-end run from host buffers (numpy arrays or pinned CPU torch tensors)."""
        def p(a):
            return None if a is None else (a.data_ptr() if isinstance(a, torch.Tensor) else a.ctypes.data)
        check(lib.st_run_host(self.ctx, M, p(xs_host), p(ys_host), p(losses_host)))

    def trace(self) -> List[Tuple[int, int, int, int, int, int, int]]:
        n = ctypes.c_size_t()
        check(lib.st_get_trace(self.ctx, None, 0, ctypes.byref(n)))
        arr = (L.StEvent * max(1, n.value))()
        check(lib.st_get_trace(self.ctx, arr, n.value, ctypes.byref(n)))
        return L._events(arr, n.value)

    def sync(self) -> None:
        check(lib.st_sync(self.ctx))

    def record_after_backward(self, mb: int, event: torch.cuda.Event) -> None:
        """Record `event` on the compute stream once B(mb) has been issued (measurement
        window of SURVEY §8(d) / P:415)."""
        event.record(self.stream)  # materialise the CUDA event (torch creates it lazily)
        check(lib.st_record_after_backward(self.ctx, mb, ctypes.c_void_p(event.cuda_event)))

    def losses_device_ptr(self) -> int:
        return lib.st_losses_device(self.ctx) or 0

    def set_profiling(self, on, classes=None) -> None:
        """on: bool; classes: kernel-class names to bracket (default: all)."""
        mask = 0
        if on:
            names = L.KERNEL_CLASSES if classes is None else classes
            mask = sum(1 << L.KERNEL_CLASSES.index(n) for n in names)
        check(lib.st_set_profiling(self.ctx, mask))

    def profile(self):
        ms = (ctypes.c_double * 6)()
        n = (ctypes.c_int64 * 6)()
        check(lib.st_get_profile(self.ctx, ms, n))
        return {name: (ms[i], n[i]) for i, name in enumerate(L.KERNEL_CLASSES)}

    def set_graph_mode(self, on: bool) -> None:
        """st_set_graph_mode: run() sessions captured into one CUDA graph and launched once."""
        check(lib.st_set_graph_mode(self.ctx, 1 if on else 0))

    def set_layer_profiling(self, on: bool) -> None:
        """Per-layer forward / backward brackets (ST_PROF_LAYERS; the backward runs
        serialised while on)."""
        check(lib.st_set_profiling(self.ctx, L.ST_PROF_LAYERS if on else 0))

    def layer_profile(self) -> np.ndarray:
        """[n_layers × 2] total ms of each layer's forward / backward work since
        set_layer_profiling(True), and [n_layers × 2] pass counts."""
        bounds = [0] + self.cuts + [len(self.layers)]
        n = 2 * (bounds[self.k + 1] - bounds[self.k])
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int64 * n)()
        check(lib.st_get_layer_profile(self.ctx, ms, cnt, n))
        return np.array(ms[:]).reshape(-1, 2), np.array(cnt[:]).reshape(-1, 2)

    def kernel_launches(self) -> int:
        return int(lib.st_kernel_launches(self.ctx))


def p2p_export(stage: Stage) -> bytes:
    """The stage's P2P descriptor (st_p2p_export): 1024 opaque bytes to hand to its
    neighbours (same process, or another process through torch.distributed)."""
    buf = ctypes.create_string_buffer(L.P2P_DESC_BYTES)
    check(lib.st_p2p_export(stage.ctx, buf))
    return buf.raw


def p2p_connect(stage: Stage, prev: Optional[bytes], nxt: Optional[bytes]) -> None:
    """Map the neighbours' buffers (st_p2p_connect): prev = stage k−1's descriptor
    (None for stage 0), nxt = stage k+1's (None for the last stage)."""
    def b(d):
        return None if d is None else ctypes.create_string_buffer(bytes(d), L.P2P_DESC_BYTES)
    check(lib.st_p2p_connect(stage.ctx, b(prev), b(nxt)))


def connect_p2p_local(stages: Sequence[Stage]) -> None:
    """P2P transport between the stage contexts of THIS process (run them with
    run_group): the producing kernels write each other's buffers directly."""
    descs = [p2p_export(s) for s in stages]
    for k, s in enumerate(stages):
        p2p_connect(s, descs[k - 1] if k > 0 else None, descs[k + 1] if k + 1 < len(stages) else None)


def connect_p2p(stage: Stage, group=None) -> None:
    """P2P transport across processes (one stage per rank, rank = stage index): the
    descriptors are all-gathered over `group` (torch.distributed, any backend) and the
    neighbours' buffers opened with CUDA IPC (NVLink / NVSwitch peer memory, or a GPU
    shared by several processes)."""
    import torch.distributed as dist
    descs = [None] * dist.get_world_size(group)
    dist.all_gather_object(descs, p2p_export(stage), group=group)
    k, n = stage.k, len(descs)
    p2p_connect(stage, descs[k - 1] if k > 0 else None, descs[k + 1] if k + 1 < n else None)


def connect_local(stages: Sequence[Stage]) -> None:
    arr = (ctypes.c_void_p * len(stages))(*[s.ctx.value for s in stages])
    check(lib.st_connect_local(arr, len(stages)))


def run_group(stages: Sequence[Stage], M: int, xs: torch.Tensor, ys: torch.Tensor,
              want_losses: bool = True) -> Optional[np.ndarray]:
    arr = (ctypes.c_void_p * len(stages))(*[s.ctx.value for s in stages])
    out = np.empty(max(1, M), np.float32) if want_losses else None
    check(lib.st_run_group(arr, len(stages), M, _ptr(xs), _ptr(ys), out.ctypes.data if out is not None else None))
    return out[:M] if out is not None else None


# ---- raw kernel hooks (tests / bench) --------------------------------------------

def update_predict_raw(W: torch.Tensor, V: torch.Tensor, G: torch.Tensor, WF: Optional[torch.Tensor],
                       WB: Optional[torch.Tensor], lr: float, gamma: float, sF: int, sB: int,
                       momentum: int = L.ST_MOMENTUM_EMA, stream: Optional[torch.cuda.Stream] = None) -> None:
    st = stream or torch.cuda.current_stream(W.device)
    check(lib.st_update_predict_raw(_ptr(W), _ptr(V), _ptr(G), _ptr(WF), _ptr(WB), W.numel(), lr, gamma, sF, sB,
                                    momentum, ctypes.c_void_p(st.cuda_stream)))


def prediction_error_raw(W_old: torch.Tensor, V_old: torch.Tensor, W_now: torch.Tensor, s: int, lr: float,
                         stream: Optional[torch.cuda.Stream] = None) -> Tuple[float, float]:
    """Fig. 7: (Σ (W_old − s·lr·V_old − W_now)², Σ (W_old − W_now)²), fp64."""
    st = stream or torch.cuda.current_stream(W_old.device)
    work = torch.empty(int(lib.st_prediction_error_work_bytes()), dtype=torch.uint8, device=W_old.device)
    out = (ctypes.c_double * 2)()
    check(lib.st_prediction_error_raw(_ptr(W_old), _ptr(V_old), _ptr(W_now), W_old.numel(), s, lr, out, _ptr(work),
                                      ctypes.c_void_p(st.cuda_stream)))
    return float(out[0]), float(out[1])


def gemm_raw(op: int, mode: int, B: int, n_in: int, n_out: int, a: torch.Tensor, b: torch.Tensor,
             aux: Optional[torch.Tensor], aux_out: Optional[torch.Tensor], out: torch.Tensor, relu: bool = False,
             work: Optional[torch.Tensor] = None, stream: Optional[torch.cuda.Stream] = None) -> None:
    st = stream or torch.cuda.current_stream(out.device)
    if work is None:
        work = torch.empty(int(lib.st_gemm_workspace_bytes(B, n_in, n_out)), dtype=torch.uint8, device=out.device)
    check(lib.st_gemm_raw(op, mode, B, n_in, n_out, _ptr(a), _ptr(b), _ptr(aux), _ptr(aux_out), _ptr(out),
                          1 if relu else 0, _ptr(work), ctypes.c_void_p(st.cuda_stream)))


def dw_update_raw(mode: int, X: torch.Tensor, dZ: torch.Tensor, W: torch.Tensor, V: torch.Tensor,
                  WF: Optional[torch.Tensor], WB: Optional[torch.Tensor], lr: float, gamma: float, sF: int, sB: int,
                  momentum: int = L.ST_MOMENTUM_EMA, work: Optional[torch.Tensor] = None,
                  G_scratch: Optional[torch.Tensor] = None, stream: Optional[torch.cuda.Stream] = None) -> None:
    """Fused dW + K-B update on one layer block (W, V, WF, WB: in·out + out fp32)."""
    B, n_in = X.shape
    n_out = dZ.shape[1]
    st = stream or torch.cuda.current_stream(X.device)
    if work is None:
        work = torch.empty(int(lib.st_gemm_workspace_bytes(B, n_in, n_out)), dtype=torch.uint8, device=X.device)
    if G_scratch is None:
        G_scratch = torch.empty_like(W)
    check(lib.st_dw_update_raw(mode, B, n_in, n_out, _ptr(X), _ptr(dZ), _ptr(W), _ptr(V), _ptr(WF), _ptr(WB), lr,
                               gamma, sF, sB, momentum, _ptr(G_scratch), _ptr(work), ctypes.c_void_p(st.cuda_stream)))


def softmax_ce_raw(logits: torch.Tensor, labels: torch.Tensor, loss: torch.Tensor, dlogits: torch.Tensor,
                   stream: Optional[torch.cuda.Stream] = None) -> None:
    B, C = logits.shape
    st = stream or torch.cuda.current_stream(logits.device)
    work = torch.empty(B, dtype=torch.float32, device=logits.device)
    check(lib.st_softmax_ce_raw(_ptr(logits), _ptr(labels), B, C, _ptr(loss), _ptr(dlogits), _ptr(work),
                                ctypes.c_void_p(st.cuda_stream)))
