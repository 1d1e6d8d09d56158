"""Parity at BASELINE.json's full sizes (-m gpu), in the launch configuration bench.py
times (`Stage.run` = st_run: fused dW + K-B update overlapped with the next layer's dX
on SM budgets, CTA-pair forward / dX GEMMs, 3xTF32), north_star's 20 mini-batches:

- the wide FCN 784 → 8 × 8192 → 10 (configs[1], 476M parameters), batch 128, at 1 stage
  (3xTF32 and CUDA-core fp32) and at 2 co-located stages (LOCAL transport, SpecTrain
  prediction on stage 0: s_F = 1);
- a 16384-wide FCN 784 → 3 × 16384 → 10 (550M parameters: the large FCN's layer shape,
  configs[4]) at 1 stage — its second 16384² layer takes the one-CTA-per-m-tile dW budget
  (128 CTAs) the large FCN runs with — and at 2 co-located stages.

The oracle runs the same mini-batches in fp64 on the host. Gates (north_star: trace
bit-exact, W and loss ≤ 1e-4 rel-L2), plus gates that see the gradient:
- ΔW = W_M − W_0 against the oracle's ΔW: a skipped update gives 1.0;
- V (the smoothed gradient, stored directly): whole-vector rel-L2 and, per layer, the
  MEDIAN over weight rows of the row rel-error. Reading D24: a pre-activation within
  fp32 rounding of 0 takes the other ReLU branch than in fp64 and moves a whole gradient
  row, so the rel-L2 of V / ΔW at full width is set by a few flipped rows — the same
  spread a plain NumPy float32 run of the oracle's own arithmetic shows against fp64
  (tools/d24_fp32_vs_fp64.py → profiles/r2_d24_fp32_vs_fp64.json, no GPU involved). The
  gates are 2× that CPU figure. A systematic error moves every row: the row-median gate
  (1e-3) catches a 1% gradient error that a rel-L2 gate at the D24 level would not.
Measured figures are appended to gpurun_out/fullsize_metrics.jsonl."""
import json
import os

import numpy as np
import pytest
import torch

import synthdata as sd
from oracle import spectrain_oracle as O
from tests.gpu_helpers import layers_of, rel_l2

pytestmark = pytest.mark.gpu

LR = 0.01  # material but stable for these widths (the bench uses 1e-3)
M_FULL = 20  # north_star: "after 20 steps"
# 2x the NumPy-float32-vs-float64 spread of the oracle's own arithmetic at full width (D24)
GATE_V = 3e-2
GATE_DW = 3e-2
GATE_ROW_MEDIAN = 1e-3

_ORACLE = {}


@pytest.fixture(scope="module")
def st():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1809_02839_b200 as st
    return st


def _oracle(key, model, w0, X, Y):
    if key not in _ORACLE:
        _ORACLE[key] = O.run(model, sd.widen(w0), X.astype(np.float64), Y, float(np.float32(LR)),
                             float(np.float32(0.9)))
    return _ORACLE[key]


def _row_median(a, b, n_in, n_out):
    a = np.asarray(a, np.float64).reshape(n_in, n_out)
    b = np.asarray(b, np.float64).reshape(n_in, n_out)
    nb = np.linalg.norm(b, axis=1)
    ok = nb > 0
    return float(np.median(np.linalg.norm(a - b, axis=1)[ok] / nb[ok]))


def _record(name, d):
    try:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        os.makedirs(os.path.join(root, "gpurun_out"), exist_ok=True)
        with open(os.path.join(root, "gpurun_out", "fullsize_metrics.jsonl"), "a") as f:
            f.write(json.dumps({"test": name, **d}) + "\n")
    except OSError:
        pass


def _check(name, model, w0, ref, Ws, Vs, losses, traces, v_tol=GATE_V, dw_tol=GATE_DW):
    for k in range(model.num_stages):
        assert traces[k] == [e.as_tuple() for e in ref.trace[k]], f"trace mismatch at stage {k}"
    W, Wr = np.concatenate(Ws), np.concatenate(ref.W)
    V, Vr = np.concatenate(Vs), np.concatenate(ref.V)
    W0 = np.concatenate(sd.widen(w0))
    m = {"loss": rel_l2(losses, ref.losses), "w": rel_l2(W, Wr), "dw": rel_l2(W - W0, Wr - W0),
         "v": rel_l2(V, Vr)}
    # per dense layer: V row medians (the flat arena is the layers' blocks in order)
    rows, off = [], 0
    for L in model.layers:
        if L.kind == sd.DENSE:
            n = L.n_in * L.n_out
            rows.append(_row_median(V[off:off + n], Vr[off:off + n], L.n_in, L.n_out))
        off += L.n_params
    m["v_row_median"] = rows
    n_out = model.layers[-1].n_params  # the output layer's block ends the last stage's arena
    m["v_out"] = rel_l2(Vs[-1][-n_out:], ref.V[-1][-n_out:])
    _record(name, m)
    assert m["loss"] <= 1e-4, m
    assert m["w"] <= 1e-4, m
    assert m["dw"] <= dw_tol, m
    assert m["v"] <= v_tol, m
    assert max(rows) <= GATE_ROW_MEDIAN, m
    assert m["v_out"] <= 1e-3, m
    return m


def _run_single(st, model, M, seed, gemm=None):
    B = 128
    w0, X, Y = sd.parity_inputs(model, M, B, seed=seed)
    dev = torch.device("cuda", 0)
    s = st.Stage(layers_of(model), model.cuts, 0, B, LR, 0.9, transport=st.ST_TRANSPORT_NCCL, device=0,
                 max_minibatches=M, gemm=st.ST_GEMM_FP32X3 if gemm is None else gemm)
    try:
        s.set_params(w0[0])
        losses = s.run(M, torch.from_numpy(X).to(dev), torch.from_numpy(Y).to(dev), want_losses=True)
        W, V, _ = s.get_params()
        tr = s.trace()
    finally:
        s.close()
    return w0, X, Y, [W], [V], losses, [tr]


def _run_local(st, model, M, seed):
    B = 128
    w0, X, Y = sd.parity_inputs(model, M, B, seed=seed)
    dev = torch.device("cuda", 0)
    stages = [st.Stage(layers_of(model), model.cuts, k, B, LR, 0.9, transport=st.ST_TRANSPORT_LOCAL, device=0,
                       max_minibatches=M) for k in range(model.num_stages)]
    try:
        st.connect_local(stages)
        assert stages[0].sizes.s_fwd == model.num_stages - 1
        for s, w in zip(stages, w0):
            s.set_params(w)
        losses = st.run_group(stages, M, torch.from_numpy(X).to(dev), torch.from_numpy(Y).to(dev),
                              want_losses=True)
        out = [s.get_params() for s in stages]
        trs = [s.trace() for s in stages]
    finally:
        for s in stages:
            s.close()
    return w0, X, Y, [o[0] for o in out], [o[1] for o in out], losses, trs


def test_wide_fcn_full_size_single_stage_bench_path(st):
    model = sd.config_wide_fcn(1)
    w0, X, Y, Ws, Vs, losses, trs = _run_single(st, model, M_FULL, seed=0)
    ref = _oracle(("wide", 1), model, w0, X, Y)
    _check("wide_fcn_1stage_fp32x3", model, w0, ref, Ws, Vs, losses, trs)


def test_wide_fcn_full_size_single_stage_fp32_simt(st):
    model = sd.config_wide_fcn(1)
    w0, X, Y, Ws, Vs, losses, trs = _run_single(st, model, M_FULL, seed=0, gemm=st.ST_GEMM_SIMT)
    ref = _oracle(("wide", 1), model, w0, X, Y)
    _check("wide_fcn_1stage_simt", model, w0, ref, Ws, Vs, losses, trs)


def test_wide_fcn_full_size_two_stages_with_prediction(st):
    model = sd.config_wide_fcn(2)
    w0, X, Y, Ws, Vs, losses, trs = _run_local(st, model, M_FULL, seed=1)
    ref = _oracle(("wide", 2), model, w0, X, Y)
    _check("wide_fcn_2stages", model, w0, ref, Ws, Vs, losses, trs)


def _fcn16k(stages):
    return sd.mlp([784, 16384, 16384, 16384, 10], cuts=sd.even_cuts(4, stages))


def test_fcn_16384_wide_single_stage_bench_path(st):
    """The large FCN's 16384² layer shape (configs[4]): 16384-wide TMA maps, the fused
    dW + update at one CTA per m-tile (128 CTAs) overlapped with the next layer's dX."""
    model = _fcn16k(1)
    w0, X, Y, Ws, Vs, losses, trs = _run_single(st, model, M_FULL, seed=2)
    ref = _oracle(("16k", 1), model, w0, X, Y)
    _check("fcn16k_1stage", model, w0, ref, Ws, Vs, losses, trs)


def test_fcn_16384_wide_two_stages_with_prediction(st):
    model = _fcn16k(2)
    w0, X, Y, Ws, Vs, losses, trs = _run_local(st, model, M_FULL, seed=3)
    ref = _oracle(("16k", 2), model, w0, X, Y)
    _check("fcn16k_2stages", model, w0, ref, Ws, Vs, losses, trs)


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
    ref = _oracle(("vgg16", 1), model, w0, X, Y)
    _check("vgg16_1stage", model, w0, ref, [W], [V], losses, [tr], dw_tol=5e-2)


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
    W0 = sd.widen(w0)[0]
    rdw = rel_l2(W - W0, ref.W[0] - W0)
    rv = rel_l2(V, ref.V[0])
    _record("lstm_lm_1stage", {"dw": rdw, "v": rv})
    assert rv <= 1e-4, rv
    assert rdw <= 1e-2, rdw
