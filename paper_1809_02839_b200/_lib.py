"""ctypes binding of libspectrain.so (include/spectrain.h) — argument marshalling only.

Every step of the SpecTrain path runs inside the library's CUDA kernels; this
module only builds the C structs, allocates the caller-owned device arenas with
PyTorch (memory, streams and process groups are PyTorch's job) and raises on a
non-zero st_status. There is no Python or CPU fallback: if the shared library is
missing, importing this module fails loudly.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# ST_LIB_PATH: a development variant built by build.build(lib=...) (still in-tree, still loud if missing)
LIB_PATH = os.environ.get("ST_LIB_PATH") or os.path.join(HERE, "libspectrain.so")

ST_FWD, ST_BWD = 0, 1
ST_ACT_NONE, ST_ACT_RELU = 0, 1
ST_LAYER_DENSE, ST_LAYER_EMBED, ST_LAYER_LSTM, ST_LAYER_CONV, ST_LAYER_POOL = 0, 1, 2, 3, 4
ST_PRED_SPECTRAIN, ST_PRED_NONE, ST_PRED_STASH, ST_PRED_STALENESS_FREE = 0, 1, 2, 3
ST_MOMENTUM_EMA, ST_MOMENTUM_HEAVY_BALL = 0, 1
ST_GEMM_FP32X3, ST_GEMM_TF32, ST_GEMM_SIMT = 0, 1, 2
ST_LOSS_SOFTMAX_CE = 0
ST_TRANSPORT_NCCL, ST_TRANSPORT_LOCAL, ST_TRANSPORT_P2P = 0, 1, 2
P2P_DESC_BYTES = 1024  # sizeof(st_p2p_desc)
KERNEL_CLASSES = ("update", "gemm_fwd", "gemm_dx", "gemm_dw", "loss", "comm")

STATUS = {0: "ST_OK", 1: "ST_ERR_INPUT", 2: "ST_ERR_SHAPE", 3: "ST_ERR_STATE", 4: "ST_ERR_CUDA",
          5: "ST_ERR_NCCL", 6: "ST_ERR_OOM", 7: "ST_ERR_DIVERGED", 8: "ST_ERR_UNSUPPORTED"}


class SpecTrainError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status


class StLayer(ctypes.Structure):
    _fields_ = [("n_in", ctypes.c_int32), ("n_out", ctypes.c_int32), ("act", ctypes.c_int32), ("bias", ctypes.c_int32),
                ("kind", ctypes.c_int32), ("hw", ctypes.c_int32)]


class StConfig(ctypes.Structure):
    _fields_ = [
        ("num_layers", ctypes.c_int32), ("layers", ctypes.POINTER(StLayer)),
        ("num_stages", ctypes.c_int32), ("cuts", ctypes.POINTER(ctypes.c_int32)),
        ("stage", ctypes.c_int32), ("batch", ctypes.c_int32), ("seq_len", ctypes.c_int32),
        ("lr", ctypes.c_float), ("gamma", ctypes.c_float),
        ("pred", ctypes.c_int32), ("momentum", ctypes.c_int32), ("gemm", ctypes.c_int32),
        ("loss", ctypes.c_int32), ("transport", ctypes.c_int32), ("device", ctypes.c_int32),
        ("max_minibatches", ctypes.c_int64), ("nccl_id", ctypes.c_uint8 * 128),
        ("replicas", ctypes.POINTER(ctypes.c_int32)), ("replica", ctypes.c_int32),
    ]


class StSizes(ctypes.Structure):
    _fields_ = [("params", ctypes.c_int64), ("w_bytes", ctypes.c_int64), ("v_bytes", ctypes.c_int64),
                ("g_bytes", ctypes.c_int64), ("wf_bytes", ctypes.c_int64), ("wb_bytes", ctypes.c_int64),
                ("stash_bytes", ctypes.c_int64), ("work_bytes", ctypes.c_int64),
                ("s_fwd", ctypes.c_int32), ("s_bwd", ctypes.c_int32)]


class StBuffers(ctypes.Structure):
    _fields_ = [("W", ctypes.c_void_p), ("V", ctypes.c_void_p), ("G", ctypes.c_void_p), ("WF", ctypes.c_void_p),
                ("WB", ctypes.c_void_p), ("stash", ctypes.c_void_p), ("work", ctypes.c_void_p)]


class StEvent(ctypes.Structure):
    _fields_ = [("stage", ctypes.c_int32), ("op_idx", ctypes.c_int32), ("dir", ctypes.c_int32), ("pad_", ctypes.c_int32),
                ("mb", ctypes.c_int64), ("base_version", ctypes.c_int64), ("s", ctypes.c_int64),
                ("target", ctypes.c_int64)]


class StCommGroup(ctypes.Structure):
    _fields_ = [("before_op", ctypes.c_int32), ("n_ops", ctypes.c_int32), ("kind", ctypes.c_int32 * 2),
                ("mb", ctypes.c_int64 * 2)]


class StStepInfo(ctypes.Structure):
    _fields_ = [("ops_run", ctypes.c_int32), ("ran_forward", ctypes.c_int32), ("ran_backward", ctypes.c_int32),
                ("done", ctypes.c_int32), ("loss", ctypes.c_float)]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I, I64, U, F, S = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t, ctypes.c_float, ctypes.c_int
    sig = {
        "st_version_difference": (I, [I, I, I]),
        "st_program": (S, [I, I, I64, I, ctypes.POINTER(StEvent), U, ctypes.POINTER(U)]),
        "st_partition": (S, [ctypes.POINTER(ctypes.c_double), I, I, ctypes.POINTER(ctypes.c_int32),
                             ctypes.POINTER(ctypes.c_double)]),
        "st_comm_plan": (S, [I, I, I64, ctypes.POINTER(StCommGroup), U, ctypes.POINTER(U)]),
        "st_query_sizes": (S, [ctypes.POINTER(StConfig), ctypes.POINTER(StSizes)]),
        "st_get_nccl_id": (S, [ctypes.POINTER(ctypes.c_uint8 * 128)]),
        "st_init": (S, [ctypes.POINTER(StConfig), ctypes.POINTER(StBuffers), P, P, P, ctypes.POINTER(P)]),
        "st_record_after_backward": (S, [P, I64, P]),
        "st_connect_local": (S, [ctypes.POINTER(P), ctypes.c_int32]),
        "st_destroy": (None, [P]),
        "st_set_params": (S, [P, P, U]),
        "st_get_params": (S, [P, P, P, U, ctypes.POINTER(I64)]),
        "st_stage_forward": (S, [P, I64, P, P, P]),
        "st_stage_backward": (S, [P, I64]),
        "st_predict_and_update": (S, [P]),
        "st_step": (S, [P, P, P, ctypes.POINTER(StStepInfo)]),
        "st_run": (S, [P, I64, P, P, P]),
        "st_run_host": (S, [P, I64, P, P, P]),
        "st_run_group": (S, [ctypes.POINTER(P), ctypes.c_int32, I64, P, P, P]),
        "st_get_trace": (S, [P, ctypes.POINTER(StEvent), U, ctypes.POINTER(U)]),
        "st_losses_device": (P, [P]),
        "st_sync": (S, [P]),
        "st_set_profiling": (S, [P, I]),
        "st_set_graph_mode": (S, [P, I]),
        "st_p2p_export": (S, [P, P]),
        "st_p2p_connect": (S, [P, P, P]),
        "st_get_profile": (S, [P, P, P]),
        "st_get_layer_profile": (S, [P, P, P, U]),
        "st_kernel_launches": (I64, [P]),
        "st_update_predict_raw": (S, [P, P, P, P, P, U, F, F, I, I, I, P]),
        "st_prediction_error_work_bytes": (I64, []),
        "st_prediction_error_raw": (S, [P, P, P, U, I, F, ctypes.POINTER(ctypes.c_double), P, P]),
        "st_gemm_raw": (S, [I, I, I, I, I, P, P, P, P, P, I, P, P]),
        "st_gemm_workspace_bytes": (I64, [I, I, I]),
        "st_softmax_ce_raw": (S, [P, P, I, I, P, P, P, P]),
        "st_dw_update_raw": (S, [I, I, I, I, P, P, P, P, P, P, F, F, I, I, I, P, P, P]),
        "st_last_error": (ctypes.c_char_p, []),
        "st_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
EXPORTED = ("st_version_difference", "st_program", "st_partition", "st_comm_plan", "st_query_sizes", "st_get_nccl_id", "st_init",
            "st_connect_local", "st_destroy", "st_set_params", "st_get_params", "st_stage_forward",
            "st_stage_backward", "st_predict_and_update", "st_step", "st_run", "st_run_host", "st_run_group", "st_get_trace",
            "st_losses_device", "st_sync", "st_record_after_backward", "st_p2p_export", "st_p2p_connect", "st_set_profiling", "st_set_graph_mode", "st_get_profile", "st_get_layer_profile", "st_kernel_launches",
            "st_update_predict_raw", "st_prediction_error_work_bytes", "st_prediction_error_raw", "st_gemm_raw", "st_gemm_workspace_bytes", "st_softmax_ce_raw", "st_dw_update_raw",
            "st_last_error", "st_version")


ST_PROF_LAYERS = 1 << 30  # st_set_profiling bit: per-layer brackets (include/spectrain.h)


def check(status: int) -> None:
    if status != 0:
        raise SpecTrainError(status, lib.st_last_error().decode())


# ---------------------------------------------------------------- host-only calls

def version_difference(k: int, N: int, direction: int) -> int:
    return lib.st_version_difference(k, N, direction)


def _events(arr, n) -> List[Tuple[int, int, int, int, int, int, int]]:
    return [(e.stage, e.op_idx, e.dir, e.mb, e.base_version, e.s, e.target) for e in arr[:n]]


def program(N: int, k: int, M: int, pred: int = ST_PRED_SPECTRAIN):
    """(stage, op_idx, dir, mb, base_version, s, target) per task of stage k."""
    n = ctypes.c_size_t()
    check(lib.st_program(N, k, M, pred, None, 0, ctypes.byref(n)))
    arr = (StEvent * max(1, n.value))()
    check(lib.st_program(N, k, M, pred, arr, n.value, ctypes.byref(n)))
    return _events(arr, n.value)


def partition(costs, N: int):
    """(cuts, max stage cost): min-max contiguous partition of per-layer costs into N
    stages (st_partition; cuts in the st_config convention, first layer of stages 1..N−1)."""
    c = (ctypes.c_double * max(1, len(costs)))(*[float(x) for x in costs])
    cuts = (ctypes.c_int32 * max(1, N - 1))()
    best = ctypes.c_double()
    check(lib.st_partition(c, len(costs), N, cuts, ctypes.byref(best)))
    return [int(cuts[i]) for i in range(N - 1)], best.value


def comm_plan(N: int, k: int, M: int):
    """[(before_op, [(kind, mb), ...])] — kinds 0 send_fwd, 1 recv_fwd, 2 send_bwd, 3 recv_bwd."""
    n = ctypes.c_size_t()
    check(lib.st_comm_plan(N, k, M, None, 0, ctypes.byref(n)))
    arr = (StCommGroup * max(1, n.value))()
    check(lib.st_comm_plan(N, k, M, arr, n.value, ctypes.byref(n)))
    return [(g.before_op, [(g.kind[i], g.mb[i]) for i in range(g.n_ops)]) for g in arr[:n.value]]


def nccl_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    check(lib.st_get_nccl_id(ctypes.byref(buf)))
    return bytes(buf)


def make_config(layers, cuts: Sequence[int], stage: int, batch: int,
                lr: float, gamma: float, pred: int = ST_PRED_SPECTRAIN, momentum: int = ST_MOMENTUM_EMA,
                gemm: int = ST_GEMM_FP32X3, transport: int = ST_TRANSPORT_NCCL, device: int = 0,
                max_minibatches: int = 256, nccl_id_bytes: Optional[bytes] = None, seq_len: int = 1,
                replicas: Optional[Sequence[int]] = None, replica: int = 0):
    """layers: (n_in, n_out, act, bias[, kind[, hw]]) tuples. Returns (StConfig, keepalive) —
    keepalive holds the arrays the struct points to."""
    def mk(t):
        t = tuple(int(v) for v in t)
        return StLayer(t[0], t[1], t[2], t[3], t[4] if len(t) > 4 else ST_LAYER_DENSE, t[5] if len(t) > 5 else 1)
    L = (StLayer * len(layers))(*[mk(t) for t in layers])
    C = (ctypes.c_int32 * max(1, len(cuts)))(*[int(c) for c in cuts]) if cuts else (ctypes.c_int32 * 1)()
    cfg = StConfig()
    cfg.num_layers = len(layers)
    cfg.layers = ctypes.cast(L, ctypes.POINTER(StLayer))
    cfg.num_stages = len(cuts) + 1
    cfg.cuts = ctypes.cast(C, ctypes.POINTER(ctypes.c_int32))
    cfg.stage, cfg.batch, cfg.lr, cfg.gamma = stage, batch, lr, gamma
    cfg.seq_len = seq_len
    cfg.pred, cfg.momentum, cfg.gemm, cfg.loss = pred, momentum, gemm, ST_LOSS_SOFTMAX_CE
    cfg.transport, cfg.device, cfg.max_minibatches = transport, device, max_minibatches
    if nccl_id_bytes is not None:
        ctypes.memmove(cfg.nccl_id, nccl_id_bytes, 128)
    Rp = None
    if replicas is not None:
        Rp = (ctypes.c_int32 * len(replicas))(*[int(r) for r in replicas])
        cfg.replicas = ctypes.cast(Rp, ctypes.POINTER(ctypes.c_int32))
    cfg.replica = int(replica)
    return cfg, (L, C, Rp)


def query_sizes(cfg: StConfig) -> StSizes:
    s = StSizes()
    check(lib.st_query_sizes(ctypes.byref(cfg), ctypes.byref(s)))
    return s
