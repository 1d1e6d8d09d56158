"""LSTM language-model stages on the GPU (-m gpu): embedding (a9), LSTM with BPTT (a8)
and the large-vocabulary softmax (a9) through the C-ABI, against the fp64 oracle.
Gates as for the FC models: trace bit-exact, weights and loss within 1e-4 rel-L2."""
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
