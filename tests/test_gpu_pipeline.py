"""End-to-end parity of the SpecTrain pipeline on the GPU (-m gpu): every stage
runs through the C-ABI on cuda:0 (LOCAL transport: N stage contexts in one
process), compared with the fp64 oracle on the same seeded inputs.

Gates (BASELINE.json north_star): per-stage trace bit-exact; fp32 weights and
loss within 1e-4 relative L2 after 20 mini-batches."""
import numpy as np
import pytest
import torch

import synthdata as sd
from oracle import spectrain_oracle as O
from tests.gpu_helpers import assert_parity, build_pipeline, layers_of, oracle_run, rel_l2, run_pipeline

pytestmark = pytest.mark.gpu

PARITY_GEMM = "fp32x3"


@pytest.fixture(scope="module")
def st():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1809_02839_b200 as st
    return st


def gemm_mode(st):
    return {"simt": st.ST_GEMM_SIMT, "fp32x3": st.ST_GEMM_FP32X3}[PARITY_GEMM]


def _parity(st, model, batch, M, lr, seed=0, pred=O.PRED_SPECTRAIN, momentum=O.MOMENTUM_EMA, labels="teacher"):
    w0, X, Y = sd.parity_inputs(model, M, batch, seed, labels)
    cpred = {O.PRED_SPECTRAIN: st.ST_PRED_SPECTRAIN, O.PRED_NONE: st.ST_PRED_NONE, O.PRED_STASH: st.ST_PRED_STASH,
             O.PRED_STALENESS_FREE: st.ST_PRED_STALENESS_FREE}[pred]
    cmom = st.ST_MOMENTUM_EMA if momentum == O.MOMENTUM_EMA else st.ST_MOMENTUM_HEAVY_BALL
    stages = build_pipeline(model, batch, lr, pred=cpred, momentum=cmom, gemm=gemm_mode(st), max_mb=M)
    try:
        res = run_pipeline(stages, w0, X, Y)
    finally:
        for s in stages:
            s.close()
    ref = oracle_run(model, w0, X, Y, lr, pred=pred, momentum=momentum)
    rw, rl = assert_parity(model, res, ref)
    # the run must have moved the weights materially
    dw = rel_l2(np.concatenate(ref.W), np.concatenate(sd.widen(w0)))
    assert dw > 1e-4
    return res, ref


def test_mlp_2stage_config0(st):
    """BJ configs[0]: MLP 784-256-256-10, 2 stages, batch 32, 20 steps."""
    _parity(st, sd.config_mlp_2stage(), 32, 20, 0.05)


def test_mlp_2stage_config0_simt_mode(st):
    """The CUDA-core diagnostic GEMM mode reaches the same parity."""
    global PARITY_GEMM
    old, PARITY_GEMM = PARITY_GEMM, "simt"
    try:
        _parity(st, sd.config_mlp_2stage(), 32, 20, 0.05)
    finally:
        PARITY_GEMM = old


def test_deep_mlp_8stage(st):
    """784-1024×8-10, one layer per stage, B=128, η=0.02."""
    _parity(st, sd.config_deep_mlp(8), 128, 20, 0.02)


@pytest.mark.parametrize("N", [1, 3, 4])
def test_pipeline_depths(st, N):
    model = sd.mlp([784, 200, 160, 96, 10], cuts=sd.even_cuts(4, N))
    _parity(st, model, 48, 20, 0.05, seed=N)


def test_vanilla_and_heavy_ball(st):
    model = sd.mlp([784, 128, 128, 10], cuts=[1, 2])
    res, ref = _parity(st, model, 32, 20, 0.05, pred=O.PRED_NONE)
    assert all(e[5] == 0 for tr in res[3] for e in tr)
    _parity(st, model, 32, 20, 0.02, momentum=O.MOMENTUM_HEAVY_BALL)


def test_weight_stashing(st):
    """PipeDream weight stashing (NEXT-2): each backward runs on its forward's
    stashed weights; the update refills that slot for the next forward. Trace bit-exact
    (a backward records its forward's version), W / loss within the gate — 3 and 4 stages
    with multi-layer early stages (fused dW + update writing the stash slot), ragged
    widths (unfused K-B fallback) and M < N."""
    model = sd.mlp([784, 128, 96, 64, 10], cuts=[2, 3])
    res, ref = _parity(st, model, 32, 20, 0.05, pred=O.PRED_STASH)
    assert all(e[5] == 0 for tr in res[3] for e in tr)
    _parity(st, sd.mlp([784, 160, 128, 96, 64, 10], cuts=[2, 3, 4]), 24, 20, 0.05, seed=2, pred=O.PRED_STASH)
    model = sd.mlp([77, 45, 31, 29, 13, 5], cuts=[2, 4])
    _parity(st, model, 7, 11, 0.05, seed=7, pred=O.PRED_STASH)
    _parity(st, model, 7, 2, 0.05, seed=8, pred=O.PRED_STASH)


def test_staleness_free_variant(st):
    """NEXT-2: s_F = N−k−1, s_B = 0 on the same kernels — trace bit-exact
    (both passes of mini-batch i target stage version i in steady state), W / loss within
    the gate; the 8-stage deep MLP (WF written on every stage but the last, WB never) and
    a ragged 4-stage net (unfused K-B fallback)."""
    model = sd.config_deep_mlp(8)
    res, ref = _parity(st, model, 128, 20, 0.02, pred=O.PRED_STALENESS_FREE)
    N = model.num_stages
    for k, tr in enumerate(res[3]):
        for e in tr:
            if e[3] >= N - k - 1:  # steady state: the target is the mini-batch index
                assert e[6] == e[3], (k, e)
    _parity(st, sd.mlp([77, 45, 31, 29, 13, 5], cuts=[1, 2, 4]), 7, 11, 0.05, seed=9, pred=O.PRED_STALENESS_FREE)


def test_ragged_shapes_and_M_smaller_than_depth(st):
    """Ragged widths (not multiples of any tile) and M < N (no steady state)."""
    model = sd.mlp([77, 45, 31, 29, 13, 5], cuts=[1, 2, 4])
    _parity(st, model, 7, 3, 0.05, seed=5)
    _parity(st, model, 7, 11, 0.05, seed=6)


def test_verbs_api_matches_run(st):
    """Drive a 3-stage pipeline task by task through st_stage_forward /
    st_stage_backward / st_predict_and_update from one thread in a
    dependency-respecting order; result equals the oracle."""
    model = sd.mlp([784, 96, 64, 10], cuts=[1, 2])
    M, B, lr = 9, 16, 0.05
    w0, X, Y = sd.parity_inputs(model, M, B, 3)
    stages = build_pipeline(model, B, lr, gemm=gemm_mode(st), max_mb=M)
    dev = stages[0].device
    xs = torch.from_numpy(X).to(dev)
    ys = torch.from_numpy(Y).to(dev)
    for s, w in zip(stages, w0):
        s.set_params(w)
    N = model.num_stages
    progs = [O.stage_program(N, k, M) for k in range(N)]
    pc = [0] * N
    done_f = set()
    done_b = set()
    losses = np.full(M, np.nan)
    while any(pc[k] < len(progs[k]) for k in range(N)):
        for k in range(N):
            while pc[k] < len(progs[k]):
                d, i = progs[k][pc[k]]
                if d == O.FWD and (k == 0 or (k - 1, i) in done_f):
                    l = stages[k].forward(i, xs[i] if k == 0 else None, ys[i] if k == N - 1 else None,
                                          want_loss=(k == N - 1))
                    if k == N - 1:
                        losses[i] = l
                    done_f.add((k, i))
                elif d == O.BWD and (k == N - 1 or (k + 1, i) in done_b):
                    stages[k].backward(i)
                    stages[k].predict_and_update()
                    done_b.add((k, i))
                else:
                    break
                pc[k] += 1
    W = [s.get_params()[0] for s in stages]
    tr = [s.trace() for s in stages]
    ref = oracle_run(model, w0, X, Y, lr)
    assert_parity(model, (W, None, losses, tr), ref)
    # out-of-order task → ST_ERR_STATE; the program is finished
    with pytest.raises(st.SpecTrainError, match="STATE"):
        stages[0].forward(0, xs[0])
    for s in stages:
        s.close()


def test_step_api_single_stage(st):
    """st_step on a 1-stage pipeline == sequential momentum SGD (oracle)."""
    model = sd.mlp([784, 64, 10], cuts=[])
    M, B, lr = 6, 8, 0.05
    w0, X, Y = sd.parity_inputs(model, M, B, 4)
    (s,) = build_pipeline(model, B, lr, gemm=gemm_mode(st), max_mb=M)
    s.set_params(w0[0])
    xs = torch.from_numpy(X).to(s.device)
    ys = torch.from_numpy(Y).to(s.device)
    losses = []
    for i in range(M):
        info = s.step(xs[i], ys[i])
        assert info.ran_forward == i and info.ran_backward == i and info.ops_run == 3
        losses.append(info.loss)
    assert s.step().done == 1
    W, V, ver = s.get_params()
    assert ver == M
    Ws, ls = O.sequential_momentum_sgd(model, sd.widen(w0)[0], X.astype(np.float64), Y, float(np.float32(lr)),
                                       float(np.float32(0.9)))
    assert rel_l2(W, Ws) < 1e-5
    assert rel_l2(losses, ls) < 1e-5
    s.close()


def test_errors_are_reported(st):
    model = sd.mlp([16, 8, 4], cuts=[1])
    stages = build_pipeline(model, 4, 0.1, gemm=gemm_mode(st), max_mb=4)
    with pytest.raises(st.SpecTrainError, match="SHAPE"):
        stages[0].set_params(np.zeros(3, np.float32))
    with pytest.raises(st.SpecTrainError, match="STATE"):
        stages[0].backward(0)  # program starts with F(0)
    with pytest.raises(st.SpecTrainError, match="INPUT"):
        stages[0].run(5)  # M > max_minibatches
    for s in stages:
        s.close()


def test_diverged_loss_detected(st):
    model = sd.mlp([16, 8, 4], cuts=[])
    (s,) = build_pipeline(model, 4, 0.1, gemm=gemm_mode(st), max_mb=2)
    w = np.full(s.params, np.nan, np.float32)
    s.set_params(w)
    xs = torch.zeros(2, 4, 16, device=s.device)
    ys = torch.zeros(2, 4, dtype=torch.int32, device=s.device)
    with pytest.raises(st.SpecTrainError, match="DIVERGED"):
        s.run(2, xs, ys, want_losses=True)
    s.close()


def test_kernel_launch_accounting_and_profile(st):
    model = sd.mlp([784, 256, 10], cuts=[])
    (s,) = build_pipeline(model, 32, 0.05, gemm=gemm_mode(st), max_mb=4)
    w0, X, Y = sd.parity_inputs(model, 4, 32, 9)
    s.set_params(w0[0])
    s.set_profiling(True)
    n0 = s.kernel_launches()
    s.run(4, torch.from_numpy(X).to(s.device), torch.from_numpy(Y).to(s.device))
    prof = s.profile()
    # st_run fuses the K-B update into each layer's dW (no standalone update launches)
    assert prof["update"][1] == 0 and prof["gemm_fwd"][1] == 8 and prof["gemm_dw"][1] == 8
    assert prof["gemm_dw"][0] > 0
    assert s.kernel_launches() - n0 >= 4 * (1 + 2 + 1 + 2 + 2)
    s.close()


def test_profiling_class_mask(st):
    """st_set_profiling with a class mask brackets only the selected classes."""
    model = sd.mlp([784, 256, 10], cuts=[])
    (s,) = build_pipeline(model, 32, 0.05, gemm=gemm_mode(st), max_mb=4)
    w0, X, Y = sd.parity_inputs(model, 4, 32, 9)
    s.set_params(w0[0])
    s.set_profiling(True, ["gemm_dw"])
    s.run(4, torch.from_numpy(X).to(s.device), torch.from_numpy(Y).to(s.device))
    prof = s.profile()
    assert prof["gemm_dw"][1] == 8 and prof["gemm_dw"][0] > 0
    assert all(prof[k][1] == 0 for k in prof if k != "gemm_dw")
    s.set_profiling(False)
    s.close()


def test_fused_and_unfused_update_paths_agree(st):
    """st_run (K-B fused into the dW epilogues) and the verb path (st_stage_backward
    writes G, st_predict_and_update runs K-B) give the same weights bit for bit."""
    model = sd.mlp([784, 256, 128, 10], cuts=[])
    M, B, lr = 5, 64, 0.05
    w0, X, Y = sd.parity_inputs(model, M, B, 11)
    (a,) = build_pipeline(model, B, lr, gemm=gemm_mode(st), max_mb=M)
    (b,) = build_pipeline(model, B, lr, gemm=gemm_mode(st), max_mb=M)
    a.set_params(w0[0])
    b.set_params(w0[0])
    xs = torch.from_numpy(X).to(a.device)
    ys = torch.from_numpy(Y).to(a.device)
    a.run(M, xs, ys)
    for i in range(M):
        b.forward(i, xs[i], ys[i])
        b.backward(i)
        b.predict_and_update()
    Wa, Va, _ = a.get_params()
    Wb, Vb, _ = b.get_params()
    np.testing.assert_array_equal(Wa, Wb)
    np.testing.assert_array_equal(Va, Vb)
    a.close()
    b.close()
