"""Pins for the CPU oracle (-m "not gpu"): each check ties the oracle to something
other than itself — the paper's worked example, closed forms, a library routine
(torch.optim.SGD / torch autograd), finite differences, or an independent
exact-rational brute force. A plausible slip in the oracle (dropped term, wrong
sign, off-by-one version, transposed operand) fails at least one of these.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

import synthdata as sd
from oracle import spectrain_oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- Eq. 5 / 6

def test_version_difference_paper_example():
    # "at the 4-th time unit ... s = ⌊0/2⌋ + 3 − 0 − 1 = 2"
    assert O.version_difference(0, 3, O.FWD) == 2
    # backward at k=0 never predicts (Eq. 6)
    for N in range(1, 17):
        assert O.version_difference(0, N, O.BWD) == 0


def test_version_difference_invariants():
    # 0 ≤ s_B ≤ s_F ≤ N−1; s_F(N−1) = s_B(N−1); s_F − s_B = N−k−1
    for N in range(1, 17):
        for k in range(N):
            sf, sb = O.version_difference(k, N, O.FWD), O.version_difference(k, N, O.BWD)
            assert 0 <= sb <= sf <= N - 1
            assert sf - sb == N - k - 1
        assert O.version_difference(N - 1, N, O.FWD) == O.version_difference(N - 1, N, O.BWD)
    assert O.version_difference(0, 1, O.FWD) == 0 and O.version_difference(0, 1, O.BWD) == 0
    assert O.version_difference(3, 3, O.FWD) == -1 and O.version_difference(-1, 3, O.BWD) == -1
    # SURVEY App. A table for N=8
    table8 = [(7, 0), (6, 0), (6, 1), (5, 1), (5, 2), (4, 2), (4, 3), (3, 3)]
    assert [(O.version_difference(k, 8, O.FWD), O.version_difference(k, 8, O.BWD)) for k in range(8)] == table8


# ---------------------------------------------------------------- Eq. 1 / Eq. 4

def test_update_smoothed_closed_forms():
    v = np.zeros(3)
    g = np.ones(3)
    v1 = O.update_smoothed(v, g, 0.9)
    np.testing.assert_allclose(v1, 0.1, rtol=0, atol=1e-15)
    v3 = O.update_smoothed(O.update_smoothed(v1, g, 0.9), g, 0.9)
    np.testing.assert_allclose(v3, 1 - 0.9 ** 3, atol=1e-15)  # 0.271
    rng = np.random.default_rng(3)
    v, g = rng.standard_normal(50), rng.standard_normal(50)
    np.testing.assert_array_equal(O.update_smoothed(v, g, 1.0), v)  # γ = 1 → v unchanged
    # contraction toward g: |v' − g| = γ |v − g|
    np.testing.assert_allclose(np.abs(O.update_smoothed(v, g, 0.7) - g), 0.7 * np.abs(v - g), rtol=1e-13)
    # heavy-ball convention: γv + g
    np.testing.assert_allclose(O.update_smoothed(v, g, 0.9, O.MOMENTUM_HEAVY_BALL), 0.9 * v + g, rtol=1e-15)


def test_predict_closed_forms():
    W = np.array([1.0])
    assert O.predict(W, np.array([0.5]), 2, 0.1)[0] == pytest.approx(0.9, abs=1e-15)
    rng = np.random.default_rng(4)
    W, v = rng.standard_normal(40), rng.standard_normal(40)
    assert O.predict(W, v, 0, 0.3) is W  # s = 0 → W bit-exact
    # linear in s; s=2 == one-step prediction applied twice with v fixed (Eq. 3 → Eq. 4)
    np.testing.assert_allclose(O.predict(W, v, 5, 0.3) - W, (O.predict(W, v, 2, 0.3) - W) + (O.predict(W, v, 3, 0.3) - W), atol=1e-14)
    np.testing.assert_allclose(O.predict(O.predict(W, v, 1, 0.3), v, 1, 0.3), O.predict(W, v, 2, 0.3), atol=1e-15)


# ---------------------------------------------------------------- schedule

@pytest.mark.parametrize("N", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("M", [1, 3, 8, 20])
def test_schedule_invariants(N, M):
    """c_F = max(0, i−(N−k−1)), c_B = i; in steady state F and B of the same
    mini-batch target i + ⌊k/2⌋."""
    model = sd.mlp([3] + [3] * N, cuts=list(range(1, N)))
    w0 = sd.glorot_params(model, 0)
    X = np.random.default_rng(1).random((M, 2, 3))
    Y = np.random.default_rng(2).integers(0, 3, (M, 2))
    res = O.run(model, w0, X, Y, 0.01, 0.9)
    for k in range(N):
        ev = res.trace[k]
        assert [(e.dir, e.mb) for e in ev] == O.stage_program(N, k, M)
        assert [e.op_idx for e in ev] == list(range(2 * M))
        for e in ev:
            if e.dir == O.FWD:
                assert e.base_version == max(0, e.mb - (N - k - 1))
                assert e.s == k // 2 + N - k - 1
            else:
                assert e.base_version == e.mb
                assert e.s == k // 2
        # steady state: same target for F and B of one mini-batch
        for i in range(N - k - 1, M):
            f = [e for e in ev if e.dir == O.FWD and e.mb == i][0]
            b = [e for e in ev if e.dir == O.BWD and e.mb == i][0]
            assert f.target == b.target == i + k // 2


def test_vanilla_span_paper_example():
    """with N=3 vanilla pipelining a mini-batch's round trip sees a span of
    N−1 = 2 versions at GPU 0 (W4..W6); its backward sees the staleness-free one."""
    N, M = 3, 8
    model = sd.mlp([2, 2, 2, 2], cuts=[1, 2])
    res = O.run(model, sd.glorot_params(model, 0), np.ones((M, 1, 2)), np.zeros((M, 1), np.int32), 0.01, 0.9, pred=O.PRED_NONE)
    ev0 = res.trace[0]
    for i in range(N - 1, M):
        f = [e for e in ev0 if e.dir == O.FWD and e.mb == i][0]
        b = [e for e in ev0 if e.dir == O.BWD and e.mb == i][0]
        assert b.base_version - f.base_version == N - 1
        assert f.s == b.s == 0


def test_program_counts():
    for N in range(1, 9):
        for k in range(N):
            for M in (1, 2, N - 1 if N > 1 else 1, N, 20):
                p = O.stage_program(N, k, M)
                assert sorted(i for d, i in p if d == O.FWD) == list(range(M))
                assert sorted(i for d, i in p if d == O.BWD) == list(range(M))
                # F(i) precedes B(i) on every stage; at most N−k in flight
                pos = {op: n for n, op in enumerate(p)}
                inflight = 0
                for d, i in p:
                    assert d == O.BWD or True
                    inflight += 1 if d == O.FWD else -1
                    assert 0 <= inflight <= N - k
                for i in range(M):
                    assert pos[(O.FWD, i)] < pos[(O.BWD, i)]


# ---------------------------------------------------------------- App. C brute force

def _appc_bruteforce(pred, heavy: bool, w_init, xs, ts, eta, gamma):
    """Independent exact-rational hand-stepping of the scalar chain. The per-stage
    task ORDER is not taken from the oracle: it emerges from a time-stepped
    round-robin simulation (P:211-212 'issues a forward task and a backward task in
    a round-robin manner', 'asynchronously executes the next one') in which a stage
    holds at most N−k mini-batches in flight and prefers a ready backward.
    pred: True = Eq. 5/6 (written out here), False = s ≡ 0, or
    "staleness_free" = s_F = N−k−1 (the number of mini-batches a stage holds in flight
    besides the current one, i.e. the updates that land between F(i) and B(i)), s_B = 0."""
    def s_fwd(k, N):
        if pred == "staleness_free":
            return N - k - 1
        return (k // 2 + N - k - 1) if pred else 0

    def s_bwd(k, N):
        if pred == "staleness_free":
            return 0
        return (k // 2) if pred else 0

    N, M = len(w_init), len(xs)
    F = Fraction
    w = [F(x) for x in w_init]
    v = [F(0)] * N
    ver = [0] * N
    nxt_f = [0] * N
    done_b = [0] * N
    inflight = [0] * N
    act_in = {}  # (k, i) input activation available at stage k
    grad_in = {}  # (k, i) upstream gradient available at stage k
    stash = {}
    losses = [None] * M
    trace = {k: [] for k in range(N)}
    for i in range(M):
        act_in[(0, i)] = F(xs[i])
    t = 0
    while any(done_b[k] < M for k in range(N)):
        t += 1
        posted = []
        for k in range(N):
            j = done_b[k]
            did = False
            if j < M and (k, j) in grad_in:
                # backward of the oldest in-flight mini-batch
                s = s_bwd(k, N)
                w_hat = w[k] - s * F(eta) * v[k]
                trace[k].append(f"B{j}({ver[k]},{s},{ver[k] + s})")
                a_in = stash.pop((k, j))
                dy = grad_in.pop((k, j))
                g = dy * a_in
                if k > 0:
                    posted.append(((k - 1, j), dy * w_hat))
                v[k] = gamma_f(gamma) * v[k] + (g if heavy else (1 - gamma_f(gamma)) * g)
                w[k] = w[k] - F(eta) * v[k]
                ver[k] += 1
                done_b[k] += 1
                inflight[k] -= 1
                did = True
            if not did:
                i = nxt_f[k]
                if i < M and (k, i) in act_in and inflight[k] < N - k:
                    s = s_fwd(k, N)
                    w_hat = w[k] - s * F(eta) * v[k]
                    trace[k].append(f"F{i}({ver[k]},{s},{ver[k] + s})")
                    a = act_in.pop((k, i))
                    stash[(k, i)] = a
                    out = w_hat * a
                    if k == N - 1:
                        d = out - F(ts[i])
                        losses[i] = d * d / 2
                        grad_in[(k, i)] = d
                    else:
                        posted.append(("act", (k + 1, i), out))
                    nxt_f[k] += 1
                    inflight[k] += 1
        # messages produced in this time unit become visible in the next one
        for p in posted:
            if p[0] == "act":
                act_in[p[1]] = p[2]
            else:
                grad_in[p[0]] = p[1]
        assert t < 100 * (M + N)
    return w, v, losses, trace


def gamma_f(g):
    return Fraction(g).limit_denominator(1000)


def test_appc_bruteforce_rational_matches_golden():
    gold = json.load(open(os.path.join(GOLDEN, "appc_scalar_chain.json")))
    w, v, losses, trace = _appc_bruteforce(True, False, gold["w_init"], gold["x"], gold["t"],
                                           Fraction(1, 10), 0.9)
    g = gold["spectrain"]
    np.testing.assert_allclose([float(a) for a in w], g["W"], rtol=1e-12)
    np.testing.assert_allclose([float(a) for a in v], g["V"], rtol=1e-12)
    np.testing.assert_allclose([float(a) for a in losses], g["losses"], rtol=1e-11)
    for k in range(3):
        assert " ".join(trace[k]) == g["trace"][str(k)]
    wv, _, lv, _ = _appc_bruteforce(False, False, gold["w_init"], gold["x"], gold["t"], Fraction(1, 10), 0.9)
    np.testing.assert_allclose([float(a) for a in wv], gold["vanilla"]["W"], rtol=1e-12)
    np.testing.assert_allclose([float(a) for a in lv], gold["vanilla"]["losses"], rtol=2e-5)
    wh, _, _, _ = _appc_bruteforce(True, True, gold["w_init"], gold["x"], gold["t"], Fraction(1, 10), 0.9)
    np.testing.assert_allclose([float(a) for a in wh], gold["heavy_ball"]["W"], rtol=1e-12)


def _scalar_chain(n):
    return sd.Model(tuple(sd.Layer(1, 1, sd.NONE, False) for _ in range(n)), tuple(range(1, n)), "half_mse")


def _appc_oracle(pred, momentum, w_init=None):
    gold = json.load(open(os.path.join(GOLDEN, "appc_scalar_chain.json")))
    w_init = gold["w_init"] if w_init is None else w_init
    model = _scalar_chain(len(w_init))
    X = np.array(gold["x"]).reshape(-1, 1, 1)
    Y = np.array(gold["t"]).reshape(-1, 1, 1)
    return gold, O.run(model, [np.array([w]) for w in w_init], X, Y, 0.1, 0.9, pred=pred, momentum=momentum)


def test_appc_oracle_spectrain():
    gold, res = _appc_oracle(O.PRED_SPECTRAIN, O.MOMENTUM_EMA)
    g = gold["spectrain"]
    np.testing.assert_allclose(np.concatenate(res.W), g["W"], rtol=1e-12)
    np.testing.assert_allclose(np.concatenate(res.V), g["V"], rtol=1e-12)
    np.testing.assert_allclose(res.losses, g["losses"], rtol=1e-11)
    for k in range(3):
        got = " ".join(f"{'F' if e.dir == O.FWD else 'B'}{e.mb}({e.base_version},{e.s},{e.target})" for e in res.trace[k])
        assert got == g["trace"][str(k)]


def test_appc_oracle_vanilla_and_heavy_ball():
    gold, res = _appc_oracle(O.PRED_NONE, O.MOMENTUM_EMA)
    np.testing.assert_allclose(np.concatenate(res.W), gold["vanilla"]["W"], rtol=1e-12)
    np.testing.assert_allclose(res.losses, gold["vanilla"]["losses"], rtol=2e-5)
    assert all(e.s == 0 for ev in res.trace for e in ev)
    gold, res = _appc_oracle(O.PRED_SPECTRAIN, O.MOMENTUM_HEAVY_BALL)
    np.testing.assert_allclose(np.concatenate(res.W), gold["heavy_ball"]["W"], rtol=1e-12)


def _tr(res, k):
    return " ".join(f"{'F' if e.dir == O.FWD else 'B'}{e.mb}({e.base_version},{e.s},{e.target})" for e in res.trace[k])


@pytest.mark.parametrize("w_init", [[0.9, 1.1, 0.8], [0.9, 1.1, 0.8, 1.2, 0.7]])
def test_staleness_free_oracle_vs_exact_bruteforce(w_init):
    """NEXT-2 staleness-free variant: the oracle against the independent exact-rational
    brute force (App. C chain, 3 and 5 stages): W, V, losses and the full trace."""
    gold = json.load(open(os.path.join(GOLDEN, "appc_scalar_chain.json")))
    w, v, losses, trace = _appc_bruteforce("staleness_free", False, w_init, gold["x"], gold["t"], Fraction(1, 10), 0.9)
    _, res = _appc_oracle(O.PRED_STALENESS_FREE, O.MOMENTUM_EMA, w_init=w_init)
    np.testing.assert_allclose(np.concatenate(res.W), [float(a) for a in w], rtol=1e-12)
    np.testing.assert_allclose(np.concatenate(res.V), [float(a) for a in v], rtol=1e-12)
    np.testing.assert_allclose(res.losses, [float(a) for a in losses], rtol=1e-11)
    for k in range(len(w_init)):
        assert _tr(res, k) == " ".join(trace[k])


def test_staleness_free_targets_and_special_cases():
    """The variant's defining property (P:271 'the entire round trip of a mini-batch
    should adopt the same weight version'): in steady state F(i) and B(i) of every
    stage target stage version i. Special cases: N = 1 is plain momentum SGD; stages 0
    and 1 use exactly Eq. 5/6 (⌊k/2⌋ = 0 there), so for N ≤ 2 the variant IS SpecTrain;
    the last stage never predicts."""
    for N in range(1, 9):
        M = 12
        res = O.run(_scalar_chain(N), [np.array([1.0])] * N, np.ones((M, 1, 1)), np.zeros((M, 1, 1)), 0.01, 0.9,
                    pred=O.PRED_STALENESS_FREE)
        for k in range(N):
            for e in res.trace[k]:
                assert e.s == ((N - k - 1) if e.dir == O.FWD else 0)
                if e.dir == O.BWD or e.mb >= N - k - 1:
                    assert e.target == e.mb, (N, k, e)
    gold = json.load(open(os.path.join(GOLDEN, "appc_scalar_chain.json")))
    _, a = _appc_oracle(O.PRED_STALENESS_FREE, O.MOMENTUM_EMA, w_init=[1.0])
    np.testing.assert_allclose(a.W[0], gold["single_w1"]["W"], rtol=1e-11)
    for w_init in ([0.9, 1.1], [0.7]):
        _, a = _appc_oracle(O.PRED_STALENESS_FREE, O.MOMENTUM_EMA, w_init=w_init)
        _, b = _appc_oracle(O.PRED_SPECTRAIN, O.MOMENTUM_EMA, w_init=w_init)
        np.testing.assert_array_equal(np.concatenate(a.W), np.concatenate(b.W))
        assert [_tr(a, k) for k in range(len(w_init))] == [_tr(b, k) for k in range(len(w_init))]


def test_appc_single_weight_momentum_sgd():
    gold, res = _appc_oracle(O.PRED_SPECTRAIN, O.MOMENTUM_EMA, w_init=[1.0])
    np.testing.assert_allclose(res.W[0], gold["single_w1"]["W"], rtol=1e-11)


# ---------------------------------------------------------------- library routines

def _torch_model_loss(model, flat, x, y):
    """Monolithic forward with torch ops (autograd supplies the reference gradient)."""
    off = 0
    a = x
    for L in model.layers:
        W = flat[off:off + L.n_in * L.n_out].view(L.n_in, L.n_out)
        off += L.n_in * L.n_out
        z = a @ W
        if L.bias:
            z = z + flat[off:off + L.n_out]
            off += L.n_out
        a = torch.relu(z) if L.act == sd.RELU else z
    if model.loss == "softmax_ce":
        return torch.nn.functional.cross_entropy(a, y.long())
    return 0.5 * ((a - y) ** 2).sum() / a.shape[0]


@pytest.mark.parametrize("cuts", [[], [1], [1, 2]])
def test_stage_composed_grads_equal_autograd(cuts):
    """composing stage backward == monolithic gradient (torch autograd, fp64)."""
    model = sd.mlp([7, 6, 5, 4], cuts=cuts)
    w = np.concatenate(sd.glorot_params(model, 5))
    w[np.arange(w.size) % 7 == 0] += 0.1  # non-zero biases
    rng = np.random.default_rng(6)
    x = rng.standard_normal((5, 7))
    y = rng.integers(0, 4, 5)
    # oracle, stage by stage
    flats, off = [], 0
    for k in range(model.num_stages):
        n = model.stage_params(k)
        flats.append(w[off:off + n])
        off += n
    a, stashes = x, []
    for k in range(model.num_stages):
        a, st = O.stage_forward(model.stage_layers(k), flats[k], a)
        stashes.append(st)
    loss, d = O.loss_and_grad("softmax_ce", a, y)
    grads = [None] * model.num_stages
    for k in range(model.num_stages - 1, -1, -1):
        grads[k], d = O.stage_backward(model.stage_layers(k), flats[k], stashes[k], d, need_dA_in=k > 0)
    g_oracle = np.concatenate(grads)
    tw = torch.tensor(w, dtype=torch.float64, requires_grad=True)
    tl = _torch_model_loss(model, tw, torch.tensor(x), torch.tensor(y))
    tl.backward()
    assert loss == pytest.approx(tl.item(), rel=1e-13)
    np.testing.assert_allclose(g_oracle, tw.grad.numpy(), rtol=1e-12, atol=1e-14)


def test_finite_difference_gradients():
    """central differences, h = 1e-5, relative error < 1e-5 (3-layer net, batch 4)."""
    model = sd.mlp([4, 5, 3, 3], cuts=[])
    w = np.concatenate(sd.glorot_params(model, 11)) + 0.05
    rng = np.random.default_rng(12)
    x = rng.standard_normal((4, 4))
    y = rng.integers(0, 3, 4)

    def f(wv):
        out, _ = O.stage_forward(model.layers, wv, x)
        return O.loss_and_grad("softmax_ce", out, y)[0]

    out, st = O.stage_forward(model.layers, w, x)
    _, dz = O.loss_and_grad("softmax_ce", out, y)
    g, _ = O.stage_backward(model.layers, w, st, dz, need_dA_in=False)
    h = 1e-5
    for i in range(w.size):
        e = np.zeros_like(w)
        e[i] = h
        fd = (f(w + e) - f(w - e)) / (2 * h)
        assert abs(fd - g[i]) <= 1e-5 * max(1e-3, abs(g[i])) + 1e-9, (i, fd, g[i])


def test_cross_entropy_uniform_logits():
    """uniform logits over C classes → loss ln C; grad rows sum to 0."""
    Z = np.full((6, 10), 0.37)
    loss, d = O.loss_and_grad("softmax_ce", Z, np.arange(6) % 10)
    assert loss == pytest.approx(math.log(10), rel=1e-15)
    np.testing.assert_allclose(d.sum(axis=1), 0, atol=1e-16)


def test_single_stage_equals_torch_sgd_dampened():
    """N=1 SpecTrain ≡ momentum SGD ≡ torch.optim.SGD(lr=η, momentum=γ,
    dampening=γ) with momentum_buffer pre-set to zeros (SURVEY §8(c) pins)."""
    model = sd.mlp([12, 9, 7, 5], cuts=[])
    w0 = np.concatenate(sd.glorot_params(model, 21))
    X, Y = sd.images_and_labels(12, 5, 10, 6, seed=22)
    eta, gamma = 0.05, 0.9
    res = O.run(model, [w0], X, Y, eta, gamma)
    tw = torch.tensor(w0, dtype=torch.float64, requires_grad=True)
    opt = torch.optim.SGD([tw], lr=eta, momentum=gamma, dampening=gamma)
    opt.state[tw]["momentum_buffer"] = torch.zeros_like(tw)
    losses = []
    for i in range(10):
        opt.zero_grad()
        l = _torch_model_loss(model, tw, torch.tensor(X[i]), torch.tensor(Y[i]))
        l.backward()
        opt.step()
        losses.append(l.item())
    np.testing.assert_allclose(res.W[0], tw.detach().numpy(), rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose(res.losses, losses, rtol=1e-11)
    np.testing.assert_allclose(res.V[0], opt.state[tw]["momentum_buffer"].numpy(), rtol=1e-10, atol=1e-15)
    # and the oracle's own sequential trainer agrees bit-for-bit
    Ws, ls = O.sequential_momentum_sgd(model, w0, X, Y, eta, gamma)
    np.testing.assert_array_equal(Ws, res.W[0])
    np.testing.assert_array_equal(ls, res.losses)


def test_interpretation_order_independent():
    model = sd.config_deep_mlp(num_stages=4, width=16, depth=5)
    w0 = sd.glorot_params(model, 0)
    X, Y = sd.images_and_labels(784, 10, 9, 4, seed=1)
    a = O.run(model, w0, X, Y, 0.02, 0.9, order="round_robin")
    b = O.run(model, w0, X, Y, 0.02, 0.9, order="stage_major")
    for wa, wb in zip(a.W, b.W):
        np.testing.assert_array_equal(wa, wb)
    np.testing.assert_array_equal(a.losses, b.losses)


def test_spectrain_differs_from_vanilla_and_staleness_witness():
    """S:356 staleness witness: for N ≥ 2 some mini-batch's F weights on device 0
    differ from the weights current at its B; SpecTrain changes the result."""
    model = sd.mlp([8, 8, 8, 4], cuts=[1, 2])
    w0 = sd.glorot_params(model, 3)
    X, Y = sd.images_and_labels(8, 4, 8, 4, seed=4)
    a = O.run(model, w0, X, Y, 0.05, 0.9, pred=O.PRED_SPECTRAIN)
    b = O.run(model, w0, X, Y, 0.05, 0.9, pred=O.PRED_NONE)
    assert not np.allclose(np.concatenate(a.W), np.concatenate(b.W), rtol=1e-9)
    assert any(f.base_version != bb.base_version for f in b.trace[0] for bb in b.trace[0]
               if f.dir == O.FWD and bb.dir == O.BWD and f.mb == bb.mb)


# ---------------------------------------------------------------- LSTM LM (a8, a9)

def _torch_lm_loss(model, flat, x_tok, y_tok):
    """The same LM with torch library modules (nn.Embedding, nn.LSTM with PyTorch's
    i, f, g, o gate order, nn.Linear), fp64, time-major [T, B]."""
    T = model.seq_len
    B = x_tok.shape[0] // T
    off = 0
    a = None
    for L in model.layers:
        if L.kind == sd.EMBED:
            E = flat[off:off + L.n_in * L.n_out].view(L.n_in, L.n_out)
            off += L.n_in * L.n_out
            a = torch.nn.functional.embedding(x_tok.long(), E)
        elif L.kind == sd.LSTM:
            h = L.n_out
            W_ih = flat[off:off + L.n_in * 4 * h].view(L.n_in, 4 * h)
            off += L.n_in * 4 * h
            W_hh = flat[off:off + h * 4 * h].view(h, 4 * h)
            off += h * 4 * h
            b = flat[off:off + 4 * h]
            off += 4 * h
            out = torch._VF.lstm(a.view(T, B, L.n_in), (torch.zeros(1, B, h, dtype=a.dtype), torch.zeros(1, B, h, dtype=a.dtype)),
                                    [W_ih.t(), W_hh.t(), b, torch.zeros_like(b)], True, 1, 0.0, False, False, False)[0]
            a = out.reshape(T * B, h)
        else:
            W = flat[off:off + L.n_in * L.n_out].view(L.n_in, L.n_out)
            off += L.n_in * L.n_out
            z = a @ W
            if L.bias:
                z = z + flat[off:off + L.n_out]
                off += L.n_out
            a = torch.relu(z) if L.act == sd.RELU else z
    return torch.nn.functional.cross_entropy(a, y_tok.long())


@pytest.mark.parametrize("cuts", [[], [1, 2, 3], [2]])
def test_lstm_lm_grads_equal_torch_lstm(cuts):
    """Embedding / LSTM / softmax stages composed stage by stage
    == torch's LSTM + autograd on the monolithic model (library routine)."""
    model = sd.lstm_lm(vocab=13, hidden=6, layers=2, cuts=cuts, seq_len=4)
    w = np.concatenate(sd.glorot_params(model, 3))
    w = w + 0.05 * np.random.default_rng(4).standard_normal(w.size)  # non-zero biases
    X, Y = sd.tokens(13, 1, 3, 4, seed=5)
    flats, off = [], 0
    for k in range(model.num_stages):
        n = model.stage_params(k)
        flats.append(w[off:off + n])
        off += n
    a, stashes = X[0], []
    for k in range(model.num_stages):
        a, st = O.stage_forward(model.stage_layers(k), flats[k], a, model.seq_len)
        stashes.append(st)
    loss, d = O.loss_and_grad("softmax_ce", a, Y[0])
    grads = [None] * model.num_stages
    for k in range(model.num_stages - 1, -1, -1):
        grads[k], d = O.stage_backward(model.stage_layers(k), flats[k], stashes[k], d, need_dA_in=k > 0,
                                       T=model.seq_len)
    tw = torch.tensor(w, dtype=torch.float64, requires_grad=True)
    tl = _torch_lm_loss(model, tw, torch.tensor(X[0]), torch.tensor(Y[0]))
    tl.backward()
    assert loss == pytest.approx(tl.item(), rel=1e-12)
    np.testing.assert_allclose(np.concatenate(grads), tw.grad.numpy(), rtol=1e-10, atol=1e-13)


def test_lstm_finite_differences():
    model = sd.lstm_lm(vocab=7, hidden=3, layers=1, cuts=[], seq_len=3)
    w = np.concatenate(sd.glorot_params(model, 9)) + 0.05
    X, Y = sd.tokens(7, 1, 2, 3, seed=10, dist="uniform")

    def f(wv):
        out, _ = O.stage_forward(model.layers, wv, X[0], 3)
        return O.loss_and_grad("softmax_ce", out, Y[0])[0]

    out, st = O.stage_forward(model.layers, w, X[0], 3)
    _, dz = O.loss_and_grad("softmax_ce", out, Y[0])
    g, _ = O.stage_backward(model.layers, w, st, dz, need_dA_in=False, T=3)
    h = 1e-6
    for i in range(w.size):
        e = np.zeros_like(w)
        e[i] = h
        fd = (f(w + e) - f(w - e)) / (2 * h)
        assert abs(fd - g[i]) <= 1e-6 * max(1e-2, abs(g[i])) + 1e-9, (i, fd, g[i])


def test_lstm_lm_pipeline_single_stage_equals_torch_sgd():
    """N=1 SpecTrain on the LM == torch.optim.SGD(momentum=γ, dampening=γ) driving
    torch's LSTM (zero momentum buffer)."""
    model = sd.lstm_lm(vocab=11, hidden=5, layers=2, cuts=[], seq_len=3)
    w0 = np.concatenate(sd.glorot_params(model, 21))
    X, Y = sd.tokens(11, 4, 2, 3, seed=22)
    res = O.run(model, [w0], X, Y, 0.1, 0.9)
    tw = torch.tensor(w0, dtype=torch.float64, requires_grad=True)
    opt = torch.optim.SGD([tw], lr=0.1, momentum=0.9, dampening=0.9)
    opt.state[tw]["momentum_buffer"] = torch.zeros_like(tw)
    for i in range(4):
        opt.zero_grad()
        _torch_lm_loss(model, tw, torch.tensor(X[i]), torch.tensor(Y[i])).backward()
        opt.step()
    np.testing.assert_allclose(res.W[0], tw.detach().numpy(), rtol=1e-10, atol=1e-13)


# ---------------------------------------------------------------- VGG conv stages (a10)

def _torch_vgg_loss(model, flat, x, y):
    off = 0
    a = x.view(x.shape[0], model.layers[0].hw, model.layers[0].hw, model.layers[0].n_in).permute(0, 3, 1, 2)
    for L in model.layers:
        if L.kind == sd.CONV:
            W = flat[off:off + 9 * L.n_in * L.n_out].view(3, 3, L.n_in, L.n_out)
            off += 9 * L.n_in * L.n_out
            b = flat[off:off + L.n_out]
            off += L.n_out
            a = torch.nn.functional.conv2d(a, W.permute(3, 2, 0, 1), b, padding=1)
            a = torch.relu(a) if L.act == sd.RELU else a
        elif L.kind == sd.POOL:
            a = torch.nn.functional.max_pool2d(a, 2)
        else:
            if a.dim() == 4:
                a = a.permute(0, 2, 3, 1).reshape(a.shape[0], -1)
            W = flat[off:off + L.n_in * L.n_out].view(L.n_in, L.n_out)
            off += L.n_in * L.n_out
            a = a @ W + flat[off:off + L.n_out]
            off += L.n_out
            a = torch.relu(a) if L.act == sd.RELU else a
    return torch.nn.functional.cross_entropy(a, y.long())


@pytest.mark.parametrize("cuts", [[], [2, 4], [1, 3, 5]])
def test_vgg_stage_grads_equal_torch_conv(cuts):
    """conv 3×3 (pad 1) + ReLU, 2×2 max-pool, FC head, composed stage by stage ==
    torch.nn.functional.conv2d / max_pool2d + autograd (library routines)."""
    model = sd.vgg(cfg=(4, "M", 6, 6, "M"), fc=(7,), classes=5, hw=8, in_ch=3, cuts=cuts)
    w = np.concatenate(sd.glorot_params(model, 31))
    w = w + 0.05 * np.random.default_rng(2).standard_normal(w.size)
    X, Y = sd.images_and_labels(model.layers[0].width_in, 5, 1, 3, seed=33)
    X = X - 0.5
    flats, off = [], 0
    for k in range(model.num_stages):
        n = model.stage_params(k)
        flats.append(w[off:off + n])
        off += n
    a, stashes = X[0], []
    for k in range(model.num_stages):
        a, st = O.stage_forward(model.stage_layers(k), flats[k], a)
        stashes.append(st)
    loss, d = O.loss_and_grad("softmax_ce", a, Y[0])
    grads = [None] * model.num_stages
    for k in range(model.num_stages - 1, -1, -1):
        grads[k], d = O.stage_backward(model.stage_layers(k), flats[k], stashes[k], d, need_dA_in=k > 0)
    tw = torch.tensor(w, dtype=torch.float64, requires_grad=True)
    tl = _torch_vgg_loss(model, tw, torch.tensor(X[0]), torch.tensor(Y[0]))
    tl.backward()
    assert loss == pytest.approx(tl.item(), rel=1e-12)
    np.testing.assert_allclose(np.concatenate(grads), tw.grad.numpy(), rtol=1e-10, atol=1e-13)


def test_maxpool_tie_rule_first_in_row_major():
    X = np.zeros((1, 2, 2, 1))
    X[0, 0, 1, 0] = X[0, 1, 0, 0] = 1.0  # two equal maxima
    Y, arg = O.maxpool2_forward(X)
    assert Y[0, 0, 0, 0] == 1.0 and arg[0, 0, 0, 0] == 1
    dX = O.maxpool2_backward(arg, np.ones((1, 1, 1, 1)), X.shape)
    assert dX[0, 0, 1, 0] == 1.0 and dX.sum() == 1.0


# ---------------------------------------------------------------- PipeDream weight stashing (NEXT-2)

def _stash_version_indexed(model, W0, X, Y, eta, gamma):
    """Weight stashing written from its definition, independently of the
    oracle's interpreter: mini-batch j sees, at every stage k, the single version
    c_F(j, k) = max(0, j − (N−k−1)) in BOTH passes (1F1B base version of its forward,
    D8), so its gradient is plain autograd of the whole model with the stage weights at
    those versions; stage k's update j then gives version j+1 (Eq. 1, D1)."""
    N = model.num_stages
    hist = [[torch.tensor(w, dtype=torch.float64)] for w in W0]  # hist[k][v] = stage k at version v
    V = [torch.zeros_like(h[0]) for h in hist]
    losses = []
    for j in range(X.shape[0]):
        used = [hist[k][max(0, j - (N - k - 1))].clone().requires_grad_(True) for k in range(N)]
        loss = _torch_model_loss(model, torch.cat(used), torch.tensor(X[j], dtype=torch.float64),
                                 torch.tensor(Y[j]))
        grads = torch.autograd.grad(loss, used)
        losses.append(float(loss.detach()))
        for k in range(N):
            V[k] = gamma * V[k] + (1.0 - gamma) * grads[k]
            hist[k].append(hist[k][-1] - eta * V[k])
    return [h[-1].numpy() for h in hist], np.array(losses)


@pytest.mark.parametrize("cuts", [[2], [2, 3], [1, 2, 3]])
def test_stash_equals_version_indexed_autograd(cuts):
    model = sd.mlp([20, 16, 12, 12, 5], cuts=cuts)
    w0, X, Y = sd.parity_inputs(model, 9, 4, seed=3)
    W0 = sd.widen(w0)
    res = O.run(model, W0, X.astype(np.float64), Y, 0.05, 0.9, pred=O.PRED_STASH)
    Wr, lr = _stash_version_indexed(model, W0, X.astype(np.float64), Y, 0.05, 0.9)
    for a, b in zip(res.W, Wr):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-12)
    np.testing.assert_allclose(res.losses, lr, rtol=1e-12)
    # the trace: s ≡ 0, the forward base version is c_F, and the backward records the
    # version its forward used (the stashed copy)
    N = model.num_stages
    for k in range(N):
        fwd_base = {}
        for e in res.trace[k]:
            assert e.s == 0 and e.target == e.base_version
            if e.dir == O.FWD:
                assert e.base_version == max(0, e.mb - (N - k - 1))
                fwd_base[e.mb] = e.base_version
            else:
                assert e.base_version == fwd_base[e.mb]


def test_stash_single_stage_is_sequential_sgd_and_differs_from_vanilla():
    model = sd.mlp([20, 16, 12, 5], cuts=[])
    w0, X, Y = sd.parity_inputs(model, 6, 4, seed=4)
    res = O.run(model, sd.widen(w0), X.astype(np.float64), Y, 0.05, 0.9, pred=O.PRED_STASH)
    W, losses = O.sequential_momentum_sgd(model, np.concatenate(sd.widen(w0)), X, Y, 0.05, 0.9)
    np.testing.assert_array_equal(np.concatenate(res.W), W)
    # N = 3 with multi-layer early stages: stashing changes the backward weights
    model = sd.mlp([20, 16, 12, 12, 5], cuts=[2, 3])
    w0, X, Y = sd.parity_inputs(model, 8, 4, seed=5)
    a = O.run(model, sd.widen(w0), X.astype(np.float64), Y, 0.05, 0.9, pred=O.PRED_STASH)
    b = O.run(model, sd.widen(w0), X.astype(np.float64), Y, 0.05, 0.9, pred=O.PRED_NONE)
    assert np.linalg.norm(np.concatenate(a.W) - np.concatenate(b.W)) > 1e-6


# ---------------------------------------------------------------- Fig. 7 prediction accuracy (NEXT-2)

def test_prediction_rmse_closed_forms():
    """A constant gradient g with γ = 0 makes v = g after one step, so the weights move by
    exactly η·g per update: the prediction W_{t−s} − sηv is exact (RMSE 0) and the stale
    weights are off by sηg (RMSE = sη·rms(g)). With γ > 0, v → g geometrically, so the
    prediction error decays to 0 while the stale error stays sη·rms(g)."""
    rng = np.random.default_rng(0)
    g = rng.standard_normal(50)
    eta = 0.1
    for gamma, exact in ((0.0, True), (0.9, False)):
        W, V = np.zeros(50), np.zeros(50)
        hist = [(W.copy(), V.copy())]
        for _ in range(200):
            V = O.update_smoothed(V, g, gamma)
            W = W - eta * V
            hist.append((W.copy(), V.copy()))
        for s_ in (1, 2, 3):
            t = len(hist) - 1
            rp, rs = O.prediction_rmse(hist[t - s_][0], hist[t - s_][1], hist[t][0], s_, eta)
            np.testing.assert_allclose(rs, s_ * eta * np.sqrt(np.mean(g ** 2)), rtol=1e-6 if not exact else 1e-12)
            assert rp < 1e-9 * rs
        # early on (t = 3, γ = 0.9: v far from g) the prediction is worse than at the end
        if not exact:
            rp_early, _ = O.prediction_rmse(hist[2][0], hist[2][1], hist[3][0], 1, eta)
            assert rp_early > 1e-3
    # s = 0: both errors are the plain distance
    a, b = rng.standard_normal(7), rng.standard_normal(7)
    rp, rs = O.prediction_rmse(a, rng.standard_normal(7), b, 0, 0.1)
    assert rp == rs == pytest.approx(np.sqrt(np.mean((a - b) ** 2)), rel=1e-15)


# ---------------------------------------------------------------- data-parallel comparator (NEXT-1)

def test_data_parallel_equals_global_batch_sgd():
    """Reading D23: averaging the batch-mean gradients of equal shards is the gradient of
    the global batch mean, so 2-way data parallelism (each replica: forward + backward on
    its half, gradients averaged, the same Eq. 1 / D1 update) equals the oracle's 1-stage
    run on the whole batch — checked with the oracle's per-stage building blocks."""
    model = sd.mlp([20, 16, 12, 5], cuts=[])
    w0, X, Y = sd.parity_inputs(model, 6, 8, seed=9)
    W = np.concatenate(sd.widen(w0))
    V = np.zeros_like(W)
    losses = []
    for i in range(X.shape[0]):
        gs, ls = [], []
        for half in (slice(0, 4), slice(4, 8)):
            out, stash = O.stage_forward(model.layers, W, X[i][half].astype(np.float64))
            loss, dZ = O.loss_and_grad(model.loss, out, Y[i][half])
            g, _ = O.stage_backward(model.layers, W, stash, dZ, need_dA_in=False)
            gs.append(g)
            ls.append(loss)
        V = O.update_smoothed(V, 0.5 * (gs[0] + gs[1]), 0.9)
        W = O.apply_update(W, V, None, 0.05, O.APPLY_MOMENTUM)
        losses.append(0.5 * (ls[0] + ls[1]))
    ref = O.run(model, sd.widen(w0), X.astype(np.float64), Y, 0.05, 0.9)
    np.testing.assert_allclose(W, np.concatenate(ref.W), rtol=0, atol=1e-13)
    np.testing.assert_allclose(losses, ref.losses, rtol=1e-13)


def test_hybrid_replica_rows_sum_to_the_stage_gradient():
    """Reading D25 (hybrid DP × PP): a replicated stage k < N−1
    splits each mini-batch by rows. Its upstream gradient already carries the 1/B of the
    GLOBAL batch-mean loss (computed once, by the unreplicated last stage), so the
    replicas' gradients must be SUMMED — unlike D23's data parallelism, where each shard
    computes its own batch mean and the shards are averaged. With the oracle's building
    blocks on a dense + conv stage: the row slices' outputs and input gradients
    concatenate to the whole batch's, and their gradients sum to the whole batch's
    gradient (so every other stage sees identical messages and the update is identical:
    the hybrid pipeline computes the unreplicated one). Averaging is off by 1/R."""
    rng = np.random.default_rng(31)
    for model, width_in in ((sd.mlp([24, 16, 12, 5], cuts=[2]), 24),
                            (sd.vgg(cfg=(4, "M"), fc=(6,), classes=3, hw=4, in_ch=2, cuts=[2]), 4 * 4 * 2)):
        layers = model.stage_layers(0)
        w = np.concatenate(sd.widen(sd.parity_inputs(model, 1, 8, seed=4)[0][:1]))
        B, R = 8, 4
        A = rng.standard_normal((B, width_in))
        out, stash = O.stage_forward(layers, w, A)
        dOut = rng.standard_normal(out.shape) / B  # the last stage's 1/B (global batch mean)
        g, dA = O.stage_backward(layers, w, stash, dOut)
        gs, outs, dAs = [], [], []
        for r in range(R):
            rows = slice(r * B // R, (r + 1) * B // R)
            o_r, st_r = O.stage_forward(layers, w, A[rows])
            g_r, dA_r = O.stage_backward(layers, w, st_r, dOut[rows])
            gs.append(g_r)
            outs.append(o_r)
            dAs.append(dA_r)
        np.testing.assert_allclose(np.concatenate(outs), out, rtol=1e-13, atol=1e-15)
        np.testing.assert_allclose(np.concatenate(dAs), dA, rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(np.sum(gs, axis=0), g, rtol=1e-12, atol=1e-15)
        assert np.linalg.norm(np.mean(gs, axis=0) - g) > 0.5 * np.linalg.norm(g)  # averaging would be wrong
