"""Shared helpers for the -m gpu parity tests: build an N-stage pipeline of
LOCAL-transport stage contexts on one GPU through the C-ABI, run it, and compare
with the oracle."""
from __future__ import annotations

import numpy as np
import torch

import synthdata as sd
from oracle import spectrain_oracle as O


def layers_of(model: sd.Model):
    import paper_1809_02839_b200 as st
    kinds = {sd.DENSE: st.ST_LAYER_DENSE, sd.EMBED: st.ST_LAYER_EMBED, sd.LSTM: st.ST_LAYER_LSTM,
             sd.CONV: st.ST_LAYER_CONV, sd.POOL: st.ST_LAYER_POOL}
    return [(l.n_in, l.n_out, st.ST_ACT_RELU if l.act == sd.RELU else st.ST_ACT_NONE, 1 if l.bias else 0,
             kinds[l.kind], l.hw) for l in model.layers]


def rel_l2(a, b) -> float:
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def build_pipeline(model: sd.Model, batch: int, lr: float, gamma: float = 0.9, pred=None, momentum=None, gemm=None,
                   max_mb: int = 64, device: int = 0):
    import paper_1809_02839_b200 as st
    pred = st.ST_PRED_SPECTRAIN if pred is None else pred
    momentum = st.ST_MOMENTUM_EMA if momentum is None else momentum
    gemm = st.ST_GEMM_FP32X3 if gemm is None else gemm
    stages = [st.Stage(layers_of(model), model.cuts, k, batch, lr, gamma, pred=pred, momentum=momentum, gemm=gemm,
                       transport=st.ST_TRANSPORT_LOCAL, device=device, max_minibatches=max_mb,
                       seq_len=model.seq_len)
              for k in range(model.num_stages)]
    st.connect_local(stages)
    return stages


def run_pipeline(stages, w0, X, Y):
    import paper_1809_02839_b200 as st
    for s, w in zip(stages, w0):
        s.set_params(w)
    dev = stages[0].device
    xs = torch.from_numpy(np.ascontiguousarray(X, np.int32 if X.dtype.kind in "iu" else np.float32)).to(dev)
    ys = torch.from_numpy(np.ascontiguousarray(Y, np.int32)).to(dev)
    losses = st.run_group(stages, X.shape[0], xs, ys, want_losses=True)
    out = [s.get_params() for s in stages]
    traces = [s.trace() for s in stages]
    return [o[0] for o in out], [o[1] for o in out], losses, traces


def oracle_run(model, w0, X, Y, lr, gamma=0.9, pred=O.PRED_SPECTRAIN, momentum=O.MOMENTUM_EMA):
    Xo = X if X.dtype.kind in "iu" else X.astype(np.float64)
    return O.run(model, sd.widen(w0), Xo, Y, float(np.float32(lr)), float(np.float32(gamma)),
                 pred=pred, momentum=momentum)


def assert_parity(model, res_gpu, res_or, tol=1e-4):
    W, V, losses, traces = res_gpu
    for k in range(model.num_stages):
        assert traces[k] == [e.as_tuple() for e in res_or.trace[k]], f"trace mismatch at stage {k}"
    rw = rel_l2(np.concatenate(W), np.concatenate(res_or.W))
    rl = rel_l2(losses, res_or.losses)
    assert np.all(np.isfinite(losses))
    assert rw <= tol, f"W rel-L2 {rw:.3e} > {tol}"
    assert rl <= tol, f"loss rel-L2 {rl:.3e} > {tol}"
    return rw, rl
