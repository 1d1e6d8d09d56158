"""NEXT-4: PipeDream-style profiled partitioning.

The engine's per-layer profile (ST_PROF_LAYERS / st_get_layer_profile) brackets each
layer's forward and backward work with CUDA events; st_partition cuts the measured
costs into stages. Checked here: the profile covers every layer of every pass, the
serialised profiled backward computes exactly what the overlapped one computes
(bitwise: the kernels are deterministic, only their scheduling changes), and the cut
st_partition returns for the measured costs is the min-max optimum (brute force).
"""
from __future__ import annotations

import itertools

import numpy as np
import pytest
import torch

import synthdata as sd
from tests.gpu_helpers import build_pipeline, layers_of, run_pipeline

pytestmark = pytest.mark.gpu


def _run_one_stage(st, model, w0, X, Y, lr, profile):
    s = st.Stage(layers_of(model), [], 0, X.shape[1], lr, 0.9, transport=st.ST_TRANSPORT_NCCL, device=0,
                 max_minibatches=X.shape[0])
    try:
        s.set_params(np.concatenate(w0))
        if profile:
            s.set_layer_profiling(True)
        dev = torch.device("cuda", 0)
        losses = s.run(X.shape[0], torch.from_numpy(X).to(dev), torch.from_numpy(Y).to(dev), want_losses=True)
        prof = s.layer_profile() if profile else None
        W, V, _ = s.get_params()
    finally:
        s.close()
    return W, V, losses, prof


def test_layer_profile_counts_and_bitwise_equal_results():
    import paper_1809_02839_b200 as st
    model = sd.mlp([784, 512, 512, 256, 10], cuts=[])
    M, B, lr = 4, 64, 0.05
    w0, X, Y = sd.parity_inputs(model, M, B, seed=3)
    W0, V0, l0, _ = _run_one_stage(st, model, w0, X, Y, lr, profile=False)
    W1, V1, l1, (ms, cnt) = _run_one_stage(st, model, w0, X, Y, lr, profile=True)
    assert np.array_equal(W0, W1) and np.array_equal(V0, V1) and np.array_equal(l0, l1)
    assert ms.shape == (len(model.layers), 2)
    assert np.all(cnt == M), cnt
    assert np.all(ms > 0), ms


def test_profiled_partition_is_min_max_optimal():
    import paper_1809_02839_b200 as st
    model = sd.mlp([784, 2048, 256, 1024, 1024, 128, 10], cuts=[])
    M, B, lr = 5, 128, 0.01
    w0, X, Y = sd.parity_inputs(model, M, B, seed=4)
    _, _, _, (ms, cnt) = _run_one_stage(st, model, w0, X, Y, lr, profile=True)
    costs = list((ms[:, 0] / cnt[:, 0] + ms[:, 1] / cnt[:, 1]).astype(float))
    n = len(costs)
    for S in (2, 3, 4):
        cuts, best = st.partition(costs, S)
        assert list(cuts) == sorted(cuts) and 0 < cuts[0] and cuts[-1] < n
        bounds = [0] + list(cuts) + [n]
        got = max(sum(costs[bounds[i]:bounds[i + 1]]) for i in range(S))
        brute = min(max(sum(costs[b[i]:b[i + 1]]) for i in range(S))
                    for c in itertools.combinations(range(1, n), S - 1) for b in [[0, *c, n]])
        assert abs(got - brute) <= 1e-9 * brute and abs(best - brute) <= 1e-9 * brute


def test_layer_profile_in_a_pipeline_stage():
    """Each stage of a co-located pipeline profiles only its own layers."""
    model = sd.mlp([784, 256, 256, 256, 10], cuts=[2])
    M, B = 5, 32
    w0, X, Y = sd.parity_inputs(model, M, B, seed=5)
    stages = build_pipeline(model, B, 0.05)
    try:
        for s in stages:
            s.set_layer_profiling(True)
        run_pipeline(stages, w0, X, Y)
        for s in stages:
            ms, cnt = s.layer_profile()
            assert ms.shape == (len(model.stage_layers(s.k)), 2)
            assert np.all(cnt == M) and np.all(ms > 0)
    finally:
        for s in stages:
            s.close()
