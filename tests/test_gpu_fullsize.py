"""Parity at BASELINE.json's full size (-m gpu), in the launch configuration bench.py
times: the wide FCN 784 → 8 × 8192 → 10 (configs[1], 476M parameters), batch 128, through
`Stage.run` (st_run: fused dW + K-B update overlapped with the next layer's dX on SM
budgets, CTA-pair forward / dX GEMMs, 3xTF32) and, for two co-located stages,
`run_group` (LOCAL transport, SpecTrain predictions active on stage 0: s_F = 1).

The oracle runs the same mini-batches in fp64 on the host. Gates: the trace bit-exact;
W and the loss within 1e-4 rel-L2 (the north-star gate). V — the smoothed gradient,
stored directly in fp32 and not masked by the weights' magnitude like W — is checked
loosely (reading D24): through 8 ReLU layers of width 8192, a pre-activation within the
fp32 accumulation error of 0 (K = 8192 terms: ~1e-5 of the operand scale on the tensor
cores, ~1e-6 with fp32 FMAs) takes the other ReLU decision than in fp64, and each such
flip moves a whole gradient row; measured V rel-L2 ~7e-3 (3xTF32) and ~2e-3 (CUDA-core
fp32) against the fp64 oracle, while the output layer (no ReLU decision after its input)
stays at ~1e-4. Gates: output layer ≤ 1e-3, all layers ≤ 3e-2."""
import numpy as np
import pytest
import torch

import synthdata as sd
from oracle import spectrain_oracle as O
from tests.gpu_helpers import layers_of, rel_l2

pytestmark = pytest.mark.gpu

LR = 0.01  # material but stable for this width (the bench uses 1e-3)


@pytest.fixture(scope="module")
def st():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1809_02839_b200 as st
    return st


def _check(model, w0, X, Y, Ws, Vs, losses, traces, v_hidden_tol):
    ref = O.run(model, sd.widen(w0), X.astype(np.float64), Y, float(np.float32(LR)), float(np.float32(0.9)))
    for k in range(model.num_stages):
        assert traces[k] == [e.as_tuple() for e in ref.trace[k]], f"trace mismatch at stage {k}"
    assert rel_l2(losses, ref.losses) <= 1e-4
    W, Wr = np.concatenate(Ws), np.concatenate(ref.W)
    V, Vr = np.concatenate(Vs), np.concatenate(ref.V)
    assert rel_l2(W, Wr) <= 1e-4
    # the weights moved (a few mini-batches at init move 476M weights by only ~4e-6 of their
    # norm, which is why V, not W, carries the gradient check here)
    assert rel_l2(Wr, np.concatenate(sd.widen(w0))) > 1e-6
    n_out = model.layers[-1].n_params  # the output layer's block ends the last stage's arena
    rv_out = rel_l2(Vs[-1][-n_out:], ref.V[-1][-n_out:])
    rv = rel_l2(V, Vr)
    assert rv_out <= 1e-3, rv_out
    assert rv <= v_hidden_tol, rv


def _single_stage(st, gemm, seed):
    model = sd.config_wide_fcn(1)
    M, B = 2, 128
    w0, X, Y = sd.parity_inputs(model, M, B, seed=seed)
    dev = torch.device("cuda", 0)
    s = st.Stage(layers_of(model), model.cuts, 0, B, LR, 0.9, transport=st.ST_TRANSPORT_NCCL, device=0,
                 max_minibatches=M, gemm=gemm)
    try:
        s.set_params(w0[0])
        losses = s.run(M, torch.from_numpy(X).to(dev), torch.from_numpy(Y).to(dev), want_losses=True)
        W, V, _ = s.get_params()
        tr = s.trace()
    finally:
        s.close()
    return model, w0, X, Y, [W], [V], losses, [tr]


def test_wide_fcn_full_size_single_stage_bench_path(st):
    _check(*_single_stage(st, st.ST_GEMM_FP32X3, seed=0), v_hidden_tol=3e-2)


def test_wide_fcn_full_size_single_stage_fp32_simt(st):
    _check(*_single_stage(st, st.ST_GEMM_SIMT, seed=0), v_hidden_tol=3e-2)


def test_wide_fcn_full_size_two_stages_with_prediction(st):
    model = sd.config_wide_fcn(2)
    M, B = 3, 128
    w0, X, Y = sd.parity_inputs(model, M, B, seed=1)
    dev = torch.device("cuda", 0)
    stages = [st.Stage(layers_of(model), model.cuts, k, B, LR, 0.9, transport=st.ST_TRANSPORT_LOCAL, device=0,
                       max_minibatches=M) for k in range(2)]
    try:
        st.connect_local(stages)
        assert stages[0].sizes.s_fwd == 1
        for s, w in zip(stages, w0):
            s.set_params(w)
        losses = st.run_group(stages, M, torch.from_numpy(X).to(dev), torch.from_numpy(Y).to(dev),
                              want_losses=True)
        out = [s.get_params() for s in stages]
        trs = [s.trace() for s in stages]
    finally:
        for s in stages:
            s.close()
    _check(model, w0, X, Y, [o[0] for o in out], [o[1] for o in out], losses, trs, v_hidden_tol=3e-2)


def test_vgg16_full_size_single_stage_bench_path(st):
    """BJ configs[3] at full size: VGG-16 on 32×32×3 images, batch 128, one stage through
    st_run (RGB first conv via the padded im2col, implicit-GEMM convs on the TMEM-A
    kernel, max-pools, FC head). Max-pool choices, like ReLU decisions, are taken in fp32
    here and in fp64 by the oracle (D24), so V gets the same loose hidden-layer gate."""
    model = sd.config_vgg16(1)
    M, B = 2, 128
    w0, X, Y = sd.parity_inputs(model, M, B, seed=0)
    dev = torch.device("cuda", 0)
    s = st.Stage(layers_of(model), model.cuts, 0, B, LR, 0.9, transport=st.ST_TRANSPORT_NCCL, device=0,
                 max_minibatches=M)
    try:
        s.set_params(w0[0])
        losses = s.run(M, torch.from_numpy(X).to(dev), torch.from_numpy(Y).to(dev), want_losses=True)
        W, V, _ = s.get_params()
        tr = s.trace()
    finally:
        s.close()
    _check(model, w0, X, Y, [W], [V], losses, [tr], v_hidden_tol=3e-2)


def test_lstm_lm_full_size_single_stage_bench_path(st):
    """BJ configs[2] at full size: embedding 10k × 1500 → 2 × LSTM(1500) → softmax over
    10k, T = 35, batch 128 (4480 token rows), one stage through st_run (recurrent GEMMs
    with split-K partials summed by the cell kernels, TMEM-A dW, the 4480 × 10 000 CE).
    No ReLU or max decisions on this path, so V is gated tightly (measured 1.2e-5)."""
    model = sd.config_lstm_lm(1)
    M, B = 2, 128
    w0 = sd.to_f32_params(sd.glorot_params(model, 0))
    X, Y = sd.tokens(model.layers[0].n_in, M, B, model.seq_len, 1)
    dev = torch.device("cuda", 0)
    s = st.Stage(layers_of(model), model.cuts, 0, B, LR, 0.9, transport=st.ST_TRANSPORT_NCCL, device=0,
                 max_minibatches=M, seq_len=model.seq_len)
    try:
        s.set_params(w0[0])
        losses = s.run(M, torch.from_numpy(X).to(dev), torch.from_numpy(Y).to(dev), want_losses=True)
        W, V, _ = s.get_params()
        tr = s.trace()
    finally:
        s.close()
    ref = O.run(model, sd.widen(w0), X, Y, float(np.float32(LR)), float(np.float32(0.9)))
    assert tr == [e.as_tuple() for e in ref.trace[0]]
    assert rel_l2(losses, ref.losses) <= 1e-4
    assert rel_l2(W, ref.W[0]) <= 1e-4
    rv = rel_l2(V, ref.V[0])
    assert rv <= 1e-4, rv
