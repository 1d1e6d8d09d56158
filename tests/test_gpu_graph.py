"""CUDA-graph sessions (st_set_graph_mode): a whole st_run session
captured into one CUDA graph and launched once must compute exactly what the eager
session computes — same kernels, same order, so bit-identical weights, smoothed
gradients, losses and trace — across the layer kinds and both update paths (fused dW
epilogue, side-stream overlap, serialised large layers are exercised by the wide
layers), and over several consecutive sessions."""
import numpy as np
import pytest
import torch

import synthdata as sd
from tests.gpu_helpers import layers_of, oracle_run, rel_l2

pytestmark = pytest.mark.gpu


def _inputs(model, M, B, seed=0):
    if model.layers[0].kind == sd.EMBED:
        w0 = sd.to_f32_params(sd.glorot_params(model, seed))
        X, Y = sd.tokens(model.layers[0].n_in, M, B, model.seq_len, seed + 1)
        return w0, X, Y
    return sd.parity_inputs(model, M, B, seed=seed)


def _run(model, B, lr, w0, X, Y, graph, sessions=(None,)):
    import paper_1809_02839_b200 as st
    dev = torch.device("cuda", 0)
    s = st.Stage(layers_of(model), [], 0, B, lr, 0.9, transport=st.ST_TRANSPORT_NCCL, device=0,
                 max_minibatches=X.shape[0], seq_len=model.seq_len)
    try:
        s.set_graph_mode(graph)
        s.set_params(np.concatenate(w0))
        xs = torch.from_numpy(np.ascontiguousarray(X, np.int32 if X.dtype.kind in "iu" else np.float32)).to(dev)
        ys = torch.from_numpy(np.ascontiguousarray(Y, np.int32)).to(dev)
        M = X.shape[0]
        bounds = [0, M] if sessions == (None,) else [0, *sessions, M]
        losses = []
        for a, b in zip(bounds[:-1], bounds[1:]):
            losses.append(s.run(b - a, xs[a:b], ys[a:b], want_losses=True))
        W, V, ver = s.get_params()
        return W, V, np.concatenate(losses), s.trace(), ver
    finally:
        s.close()


CASES = [
    ("mlp", lambda: sd.mlp([784, 256, 256, 10], cuts=[]), 8, 32, 0.05),
    ("deep_mlp", lambda: sd.config_deep_mlp(1), 6, 128, 0.02),
    ("wide", lambda: sd.mlp([784, 2048, 2048, 10], cuts=[]), 5, 128, 0.01),
    ("lstm_lm", lambda: sd.lstm_lm(vocab=96, hidden=64, layers=2, cuts=[], seq_len=5), 4, 16, 0.1),
    ("vgg", lambda: sd.vgg(cfg=(32, "M", 64, "M"), fc=(64,), classes=10, hw=8, cuts=[]), 4, 16, 0.02),
]


@pytest.mark.parametrize("name,mk,M,B,lr", CASES, ids=[c[0] for c in CASES])
def test_graph_session_bitwise_equals_eager(name, mk, M, B, lr):
    model = mk()
    w0, X, Y = _inputs(model, M, B)
    eager = _run(model, B, lr, w0, X, Y, False, sessions=(M // 2,))
    graph = _run(model, B, lr, w0, X, Y, True, sessions=(M // 2,))
    assert eager[3] == graph[3] and eager[4] == graph[4]
    assert np.array_equal(eager[0], graph[0]) and np.array_equal(eager[1], graph[1])
    assert np.array_equal(eager[2], graph[2])
    if name == "mlp":  # and against the oracle (one session)
        W, V, losses, trace, _ = _run(model, B, lr, w0, X, Y, True)
        ref = oracle_run(model, w0, X, Y, lr)
        assert trace == [e.as_tuple() for e in ref.trace[0]]
        assert rel_l2(W, np.concatenate(ref.W)) <= 1e-4 and rel_l2(losses, ref.losses) <= 1e-4
