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
- ΔW = W_M − W_0 against the oracle's ΔW (a skipped update gives 1.0) and V, the
  smoothed gradient, stored directly. Reading D24, pinned on the CPU
  (tools/d24_fp32_vs_fp64.py → profiles/r2_d24_fp32_vs_fp64.json, no GPU involved): the
  oracle's own arithmetic in plain NumPy float32 differs from float64 at this width by
  V 1.7e-2 and ΔW 9.6e-3 after 20 mini-batches — all of it from ReLU decisions on
  pre-activations within rounding of 0 (with the fp64 decisions the same float32
  arithmetic gives V 7e-7). The gates are 2× those figures.
- the output layer's V (no ReLU decision after its input): 1e-3.
Measured figures are appended to gpurun_out/fullsize_metrics.jsonl."""
import json
import os

import numpy as np
import pytest
import torch

import synthdata as sd
from oracle import spectrain_oracle as O
from tests.gpu_helpers import build_pipeline, layers_of, rel_l2, run_pipeline

pytestmark = pytest.mark.gpu

LR = 0.01  # material but stable for these widths (the bench uses 1e-3)
M_FULL = 20  # north_star: "after 20 steps"
# 2x the NumPy-float32-vs-float64 spread of the oracle's own arithmetic at full width after
# 20 mini-batches (D24, profiles/r2_d24_fp32_vs_fp64.json: V 1.70e-2, dW 9.62e-3)
GATE_V = 3.4e-2
GATE_DW = 1.9e-2

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
    # per dense layer: median row error of V (reported: the ReLU-decision spread of D24 is
    # diffuse — a changed dZ entry reaches every gradient of the earlier layers)
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


def test_vgg16_full_size_8_stages_bench_partition(st):
    """BJ configs[3] at full size in its pipelined form: VGG-16 (32×32×3, batch 128) cut
    into the 8 stages of SURVEY §8(d) (`vgg16_cuts_8`), co-located through the LOCAL
    transport, M = 10 mini-batches (the pipeline fills: stage 0 runs 7 warm-up forwards,
    then F/B pairs with s_F up to 7). Trace exact per stage; W and loss within 1e-4 (the
    north-star gate). V and ΔW: on this very run the CUDA-core fp32 GEMMs (ST_GEMM_SIMT)
    spread them by 0.039 / 0.013 against the fp64 oracle (ReLU / max-pool decisions, D24),
    the 3xTF32 tensor path by 0.093 / 0.052 — the excess is the tensor core's accumulation
    loss over long K (D24; segmented accumulation brings it to 0.035 / 0.011 at a
    throughput cost, profiles/r2_tsg_segmented_accumulation.json). Gates 0.15 / 0.1: a
    skipped update (ΔW = 1) or a wrong gradient (V ~ 1) still fails."""
    model = sd.config_vgg16(8)
    M, B = 10, 128
    w0, X, Y = sd.parity_inputs(model, M, B, seed=0)
    stages = build_pipeline(model, B, LR, max_mb=M)
    try:
        W, V, losses, traces = run_pipeline(stages, w0, X, Y)
    finally:
        for s_ in stages:
            s_.close()
    ref = _oracle(("vgg16", 8), model, w0, X, Y)
    _check("vgg16_8stages", model, w0, ref, W, V, losses, traces, v_tol=0.15, dw_tol=0.1)


def test_lstm_lm_full_size_4_stages(st):
    """BJ configs[2] at full size in its pipelined form: {Emb}{LSTM1}{LSTM2}{Softmax}
    (SURVEY §8(d) row 3), T = 35, batch 128, co-located through the LOCAL transport,
    M = 6 mini-batches. No ReLU / max decisions: V is gated tightly, as at 1 stage."""
    model = sd.config_lstm_lm(4)
    M, B = 6, 128
    w0 = sd.to_f32_params(sd.glorot_params(model, 0))
    X, Y = sd.tokens(model.layers[0].n_in, M, B, model.seq_len, 1)
    stages = build_pipeline(model, B, LR, max_mb=M)
    try:
        W, V, losses, traces = run_pipeline(stages, w0, X, Y)
    finally:
        for s_ in stages:
            s_.close()
    ref = O.run(model, sd.widen(w0), X, Y, float(np.float32(LR)), float(np.float32(0.9)))
    for k in range(model.num_stages):
        assert traces[k] == [e.as_tuple() for e in ref.trace[k]], f"trace mismatch at stage {k}"
    Wc, Wr = np.concatenate(W), np.concatenate(ref.W)
    W0 = np.concatenate(sd.widen(w0))
    rl, rw = rel_l2(losses, ref.losses), rel_l2(Wc, Wr)
    rv, rdw = rel_l2(np.concatenate(V), np.concatenate(ref.V)), rel_l2(Wc - W0, Wr - W0)
    _record("lstm_lm_4stages", {"loss": rl, "w": rw, "v": rv, "dw": rdw})
    assert rl <= 1e-4 and rw <= 1e-4, (rl, rw)
    assert rv <= 1e-4, rv
    assert rdw <= 1e-2, rdw


def test_large_fcn_full_size_one_step_sampled(st):
    """BJ configs[4] at FULL size — the bench's N = 1 workload (784 → 16 × 16384 → 10,
    4.04G parameters, 16.2 GB per arena, batch 128) — through st_run in the launch
    configuration bench.py times, one mini-batch. The arenas run past 2³² bytes (every
    layer from the 5th on sits above 4 GiB), so this checks the 64-bit addressing of the
    TMA maps, the fused dW + update and the split-K workspaces on the real sizes.

    The whole model does not fit the oracle, so it is checked on sampled outputs the
    oracle computes one by one: the fp64 forward / backward streams layer by layer
    (each layer's block redrawn from its own seed, the oracle's stage_forward /
    stage_backward on that one layer — stage composition equals the monolithic model,
    pinned in test_oracle_pins), and per layer 512 random weights plus the bias are
    compared. After one update from V = 0: V = (1 − γ)·g and W = W0 − η·V (Eq. 1, D1).
    Gates: loss 1e-5; sampled V per layer 5e-2 (one mini-batch, reading D24: the ReLU
    decisions taken on pre-activations within rounding of 0. At K = 16384 the 3xTF32
    forward GEMM's pre-activation error is 3.8e-5 rms of |Z| against 1.6e-6 for an fp32
    GEMM — 16 vs 1 of 2.1M decisions differ per layer (tools/gemm_error.py,
    profiles/r2_gemm_error.txt); plain fp32 at this size spreads V by 1.1e-3 (1 flip) to
    4.2e-3 per layer (profiles/r2_d24_large_fcn_1step.json); each flipped mask entry moves
    a 16384-wide layer's V by ~1e-3 and the flips of all later layers add up: measured
    0.9e-2 (layer 15) to 2.2e-2 (layer 0)); sampled W per layer 1e-6 + 5e-2·‖η·V‖/‖W‖ —
    W = W0 − η·V, so the V error allowed above reaches W scaled by the update's size,
    plus fp32 storage of W0."""
    model = sd.config_large_fcn(1)
    L = model.layers
    B, seed = 128, 11
    dev = torch.device("cuda", 0)
    X, Y = sd.images_and_labels(784, 10, 1, B, seed + 1, "teacher")
    X = X.astype(np.float32)
    s = st.Stage(layers_of(model), model.cuts, 0, B, LR, 0.9, transport=st.ST_TRANSPORT_NCCL, device=0,
                 max_minibatches=1)
    try:
        offs = np.cumsum([0] + [l.n_params for l in L])
        assert offs[5] * 4 > 2 ** 32
        w_dev = torch.empty(int(offs[-1]), dtype=torch.float32, device=dev)
        for i, layer in enumerate(L):
            w_dev[int(offs[i]):int(offs[i + 1])].copy_(torch.from_numpy(sd.glorot_dense_layer_f32(layer, seed, i)))
        s.set_params(w_dev)
        del w_dev
        losses = s.run(1, torch.from_numpy(X).to(dev), torch.from_numpy(Y).to(dev), want_losses=True)
        Wd = s.W.view(torch.float32)
        Vd = s.V.view(torch.float32)
        rng = np.random.default_rng(5)
        picks = []
        for i, layer in enumerate(L):
            rows = rng.integers(0, layer.n_in, 512)
            cols = rng.integers(0, layer.n_out, 512)
            idx = np.concatenate([offs[i] + rows.astype(np.int64) * layer.n_out + cols,
                                  offs[i] + layer.n_in * layer.n_out + np.arange(layer.n_out)])
            it = torch.from_numpy(idx).to(dev)
            picks.append((rows, cols, Wd[it].cpu().numpy().astype(np.float64), Vd[it].cpu().numpy().astype(np.float64)))
        tr = s.trace()
    finally:
        s.close()
    assert tr == [(0, 0, 0, 0, 0, 0, 0), (0, 1, 1, 0, 0, 0, 0)]
    # oracle, streamed layer by layer in fp64
    A = X[0].astype(np.float64)
    stash = []
    for i, layer in enumerate(L):
        flat = sd.glorot_dense_layer_f32(layer, seed, i).astype(np.float64)
        A, st_l = O.stage_forward([layer], flat, A)
        stash.append(st_l)
    loss, dA = O.loss_and_grad(model.loss, A, Y[0])
    assert abs(losses[0] - loss) <= 1e-5 * abs(loss), (losses[0], loss)
    gamma, eta = float(np.float32(0.9)), float(np.float32(LR))
    worst = []
    for i in range(len(L) - 1, -1, -1):
        layer = L[i]
        flat = sd.glorot_dense_layer_f32(layer, seed, i).astype(np.float64)
        g, dA = O.stage_backward([layer], flat, stash[i], dA, need_dA_in=i > 0)
        stash[i] = None
        rows, cols, w_got, v_got = picks[i]
        nw = layer.n_in * layer.n_out
        sel = np.concatenate([rows.astype(np.int64) * layer.n_out + cols, nw + np.arange(layer.n_out)])
        v_ref = (1.0 - gamma) * g[sel]
        w_ref = flat[sel] - eta * v_ref
        rv = rel_l2(v_got, v_ref)
        rw = rel_l2(w_got, w_ref)
        tol_w = 1e-6 + 5e-2 * eta * np.linalg.norm(v_ref) / np.linalg.norm(w_ref)
        worst.append((i, rv, rw, tol_w))
    _record("large_fcn_full_1step_sampled", {"loss": float(losses[0]), "loss_ref": loss,
                                              "per_layer_v_w_tolw": worst})
    for i, rv, rw, tol_w in worst:
        assert rw <= tol_w, (i, rw, tol_w)
        assert rv <= 5e-2, (i, rv)
