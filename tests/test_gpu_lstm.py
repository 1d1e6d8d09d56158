"""LSTM language-model stages on the GPU (-m gpu): embedding (a9), LSTM with BPTT (a8)
and the large-vocabulary softmax (a9) through the C-ABI, against the fp64 oracle.
Gates as for the FC models: trace bit-exact, weights and loss within 1e-4 rel-L2."""
import os

import numpy as np
import pytest
import torch

import synthdata as sd
from oracle import spectrain_oracle as O
from tests.gpu_helpers import assert_parity, build_pipeline, oracle_run, rel_l2, run_pipeline

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def st():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1809_02839_b200 as st
    return st


def _lm_parity(st, model, batch, M, lr, seed=0, gemm=None):
    w0 = sd.to_f32_params(sd.glorot_params(model, seed))
    X, Y = sd.tokens(model.layers[0].n_in, M, batch, model.seq_len, seed + 1)
    stages = build_pipeline(model, batch, lr, gemm=gemm, max_mb=M)
    try:
        res = run_pipeline(stages, w0, X, Y)
    finally:
        for s in stages:
            s.close()
    ref = oracle_run(model, w0, X, Y, lr)
    rw, rl = assert_parity(model, res, ref)
    assert rel_l2(np.concatenate(ref.W), np.concatenate(sd.widen(w0))) > 1e-4
    return rw, rl


def test_lstm_lm_4stage_tma_shapes(st):
    """{Emb}{LSTM}{LSTM}{Softmax} (BJ configs[2] structure) at widths the TMA/tcgen05
    GEMMs take (H = 64, 4H = 256, V = 96), T = 5, B = 16."""
    model = sd.lstm_lm(vocab=96, hidden=64, layers=2, cuts=[1, 2, 3], seq_len=5)
    _lm_parity(st, model, 16, 12, 0.5)


def test_lstm_lm_single_stage_and_ragged(st):
    """All layers on one stage (LSTM→LSTM and LSTM→softmax aliasing inside a stage),
    ragged widths (H = 6, V = 13: CUDA-core GEMM path), T = 4."""
    model = sd.lstm_lm(vocab=13, hidden=6, layers=2, cuts=[], seq_len=4)
    _lm_parity(st, model, 3, 8, 0.5, seed=3)
    model = sd.lstm_lm(vocab=40, hidden=32, layers=2, cuts=[2], seq_len=3)
    _lm_parity(st, model, 8, 8, 0.5, seed=4)


def test_lstm_lm_simt_mode(st):
    model = sd.lstm_lm(vocab=96, hidden=64, layers=1, cuts=[1, 2], seq_len=4)
    _lm_parity(st, model, 8, 6, 0.5, seed=5, gemm=st.ST_GEMM_SIMT)


@pytest.mark.parametrize("vocab,hidden,layers,T,B,M", [
    (96, 64, 2, 5, 16, 8),     # fwd: 2 gate-interleaved tiles; bwd: 1 tile, 8 K splits
    (50, 100, 2, 6, 40, 6),    # ragged: last fwd tile 4 units, bwd tile 100 rows, B not a multiple of 16
    (64, 260, 1, 3, 128, 4),   # bwd: 3 tiles, 33 K splits of one K-block each; fwd: 9 tiles × 9 splits
    (32, 64, 2, 1, 8, 4),      # T = 1: no recurrent product, cell phase only
])
def test_lstm_single_stage_recurrence_shapes(st, vocab, hidden, layers, T, B, M):
    """One stage (no co-located contexts) at shapes that exercise the recurrence tiling:
    parity with the oracle. Under the development opt-in ST_LSTM_PERSIST=1 (run by
    tests/test_gpu_variants.py) each layer's recurrence is ONE persistent cooperative launch
    per direction (k_lstm_rec.cu: MMA phase, per-tile sync, cell phase, grid sync per step):
    then also a launch count that does not grow with T."""
    def run(T_):
        model = sd.lstm_lm(vocab=vocab, hidden=hidden, layers=layers, cuts=[], seq_len=T_)
        w0 = sd.to_f32_params(sd.glorot_params(model, 11))
        X, Y = sd.tokens(vocab, M, B, T_, 12)
        stages = build_pipeline(model, B, 0.5, max_mb=M)
        try:
            res = run_pipeline(stages, w0, X, Y)
            per_mb = stages[0].kernel_launches() / M
        finally:
            for s in stages:
                s.close()
        return model, w0, X, Y, res, per_mb

    model, w0, X, Y, res, per_mb = run(T)
    ref = oracle_run(model, w0, X, Y, 0.5)
    assert_parity(model, res, ref)
    if os.environ.get("ST_LSTM_PERSIST") == "1":
        assert run(T + 3)[-1] == per_mb
