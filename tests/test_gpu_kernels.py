"""Kernel-level parity on the GPU (-m gpu): K-B fused update/prediction, the
stage GEMMs and softmax-CE against NumPy (fp64 / exact-product emulation)."""
import math
import numpy as np
import pytest
import torch

from oracle import spectrain_oracle as O

pytestmark = pytest.mark.gpu

GEMM_MODES = ["simt", "fp32x3", "tf32"]
TOL = {"simt": 1e-5, "fp32x3": 1e-5, "tf32": 3e-3}


@pytest.fixture(scope="module")
def st():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1809_02839_b200 as st
    return st


def _f32(x):
    return np.asarray(x, dtype=np.float64).astype(np.float32)


def _emulate_kb(W, V, G, lr, gamma, sF, sB, heavy):
    """fp32 kernel contract (SURVEY §8(c) 'Kernel-level contract for K-B'):
    v' = fma(γ, v, f32((1−γ)·g)), w' = fma(−η, v', w), wf = fma(−s_F·η, v', w')."""
    d = np.float64
    cg = d(np.float32(gamma))
    c1 = d(np.float32(1.0)) if heavy else d(np.float32(1.0 - d(np.float32(gamma))))
    ce = d(np.float32(lr))
    cf = d(np.float32(sF * d(np.float32(lr))))
    cb = d(np.float32(sB * d(np.float32(lr))))
    t = _f32(c1 * G.astype(d))
    vn = _f32(cg * V.astype(d) + t.astype(d))
    wn = _f32(-ce * vn.astype(d) + W.astype(d))
    wf = _f32(-cf * vn.astype(d) + wn.astype(d))
    wb = _f32(-cb * vn.astype(d) + wn.astype(d))
    return wn, vn, wf, wb


def _ulp_diff(a, b):
    ai = a.view(np.int32).astype(np.int64)
    bi = b.view(np.int32).astype(np.int64)
    ai = np.where(ai < 0, np.int64(-2**31) - ai, ai)
    bi = np.where(bi < 0, np.int64(-2**31) - bi, bi)
    return np.abs(ai - bi)


@pytest.mark.parametrize("n", [1, 3, 4, 1000, 1_000_003])
@pytest.mark.parametrize("sF,sB,heavy", [(0, 0, False), (3, 0, False), (6, 1, False), (5, 2, True), (4, 4, False)])
def test_update_predict_kernel(st, n, sF, sB, heavy):
    rng = np.random.default_rng(n + 7 * sF + sB)
    W = rng.standard_normal(n).astype(np.float32)
    V = (0.1 * rng.standard_normal(n)).astype(np.float32)
    G = rng.standard_normal(n).astype(np.float32)
    lr, gamma = 0.05, 0.9
    dev = torch.device("cuda", 0)
    tW, tV, tG = (torch.from_numpy(a.copy()).to(dev) for a in (W, V, G))
    tF = torch.full((n,), 123.0, device=dev) if sF > 0 else None
    tB = torch.full((n,), 321.0, device=dev) if (sB > 0 and sB != sF) else None
    st.update_predict_raw(tW, tV, tG, tF, tB, lr, gamma, sF, sB,
                          st.ST_MOMENTUM_HEAVY_BALL if heavy else st.ST_MOMENTUM_EMA)
    torch.cuda.synchronize()
    wn, vn, wf, wb = _emulate_kb(W, V, G, lr, gamma, sF, sB, heavy)
    assert _ulp_diff(tV.cpu().numpy(), vn).max() <= 1
    assert _ulp_diff(tW.cpu().numpy(), wn).max() <= 1
    if tF is not None:
        assert _ulp_diff(tF.cpu().numpy(), wf).max() <= 2
    if tB is not None:
        assert _ulp_diff(tB.cpu().numpy(), wb).max() <= 2
    # and against the fp64 oracle formulas (Eq. 1, D1, Eq. 4)
    v64 = O.update_smoothed(V.astype(np.float64), G.astype(np.float64), gamma,
                            O.MOMENTUM_HEAVY_BALL if heavy else O.MOMENTUM_EMA)
    w64 = W.astype(np.float64) - lr * v64
    np.testing.assert_allclose(tW.cpu().numpy(), w64, rtol=1e-5, atol=1e-6)
    if tF is not None:
        np.testing.assert_allclose(tF.cpu().numpy(), O.predict(w64, v64, sF, lr), rtol=1e-5, atol=1e-6)


def test_update_predict_s0_untouched_outputs(st):
    """s = 0: no prediction buffer is written (WF/WB alias W in the engine)."""
    n = 4096
    dev = torch.device("cuda", 0)
    W = torch.randn(n, device=dev)
    V = torch.zeros(n, device=dev)
    G = torch.randn(n, device=dev)
    w0 = W.clone()
    st.update_predict_raw(W, V, G, None, None, 0.1, 0.9, 0, 0)
    torch.cuda.synchronize()
    torch.testing.assert_close(V, 0.1 * G, rtol=1e-6, atol=1e-7)
    torch.testing.assert_close(W, w0 - 0.1 * V, rtol=1e-6, atol=1e-7)


MODES = {"simt": 2, "fp32x3": 0, "tf32": 1}


@pytest.mark.parametrize("mode", GEMM_MODES)
@pytest.mark.parametrize("B,n_in,n_out", [(32, 784, 256), (128, 300, 70), (5, 33, 17), (128, 1024, 1024),
                                          (96, 160, 200), (128, 4096, 512), (7, 264, 136), (128, 784, 384),
                                          (16, 128, 4096), (1100, 96, 200), (4480, 64, 136)])
def test_stage_gemms_vs_fp64(st, mode, B, n_in, n_out):
    """fwd (bias + ReLU), dX (ReLU mask), dW (+ bias grad) against fp64. B ≥ 1024 rows: the
    forward runs on the persistent TMEM-A kernel (tall forward; ragged last row tile)."""
    rng = np.random.default_rng(B * 7 + n_in)
    dev = torch.device("cuda", 0)
    X = rng.standard_normal((B, n_in)).astype(np.float32)
    W = (rng.standard_normal((n_in, n_out)) / np.sqrt(n_in)).astype(np.float32)
    b = rng.standard_normal(n_out).astype(np.float32)
    dZ = rng.standard_normal((B, n_out)).astype(np.float32)
    mask = np.maximum(rng.standard_normal((B, n_in)), 0).astype(np.float32)
    t = lambda a: torch.from_numpy(a).to(dev)
    m = MODES[mode]
    tol = TOL[mode]
    X64, W64, dZ64 = X.astype(np.float64), W.astype(np.float64), dZ.astype(np.float64)
    # fwd + bias + ReLU
    Z = torch.empty(B, n_out, device=dev)
    st.gemm_raw(0, m, B, n_in, n_out, t(X), t(W), t(b), None, Z, relu=True)
    ref = np.maximum(X64 @ W64 + b, 0)
    scale = np.abs(X64) @ np.abs(W64) + np.abs(b)
    torch.cuda.synchronize()
    assert np.all(np.abs(Z.cpu().numpy() - ref) <= tol * scale + 1e-30)
    # dX with ReLU mask
    D = torch.empty(B, n_in, device=dev)
    st.gemm_raw(1, m, B, n_in, n_out, t(dZ), t(W), t(mask), None, D)
    ref = (dZ64 @ W64.T) * (mask > 0)
    scale = np.abs(dZ64) @ np.abs(W64.T)
    torch.cuda.synchronize()
    assert np.all(np.abs(D.cpu().numpy() - ref) <= tol * scale + 1e-30)
    # dW + bias grad
    G = torch.empty(n_in, n_out, device=dev)
    gb = torch.empty(n_out, device=dev)
    st.gemm_raw(2, m, B, n_in, n_out, t(X), t(dZ), None, gb, G)
    ref = X64.T @ dZ64
    scale = np.abs(X64.T) @ np.abs(dZ64)
    torch.cuda.synchronize()
    assert np.all(np.abs(G.cpu().numpy() - ref) <= tol * scale + 1e-30)
    np.testing.assert_allclose(gb.cpu().numpy(), dZ64.sum(0), rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("B,C", [(32, 10), (128, 10), (7, 1000), (64, 10000), (3, 13), (5, 4096)])
def test_softmax_ce_vs_oracle(st, B, C):
    rng = np.random.default_rng(C + B)
    Z = (3 * rng.standard_normal((B, C))).astype(np.float32)
    y = rng.integers(0, C, B).astype(np.int32)
    dev = torch.device("cuda", 0)
    loss = torch.empty(1, device=dev)
    d = torch.empty(B, C, device=dev)
    st.softmax_ce_raw(torch.from_numpy(Z).to(dev), torch.from_numpy(y).to(dev), loss, d)
    torch.cuda.synchronize()
    l64, d64 = O.loss_and_grad("softmax_ce", Z.astype(np.float64), y)
    assert loss.item() == pytest.approx(l64, rel=2e-6)
    np.testing.assert_allclose(d.cpu().numpy(), d64, rtol=1e-5, atol=1e-7 / B)


@pytest.mark.parametrize("mode", ["fp32x3", "simt"])
@pytest.mark.parametrize("B,n_in,n_out,sF,sB", [(128, 1024, 512, 0, 0), (32, 784, 256, 3, 1), (7, 264, 136, 2, 2),
                                                (64, 256, 10, 1, 0), (128, 384, 640, 5, 2)])
def test_dw_update_fused_vs_fp64(st, mode, B, n_in, n_out, sF, sB):
    """dW fused with the K-B update (the st_run path): compare W, V, WF, WB with the
    fp64 formulas applied to g = [Xᵀ·dZ ; Σ_b dZ] (Eq. 1, D1 apply, Eq. 4)."""
    rng = np.random.default_rng(n_in + n_out + B)
    dev = torch.device("cuda", 0)
    P = n_in * n_out + n_out
    X = rng.standard_normal((B, n_in)).astype(np.float32)
    dZ = (rng.standard_normal((B, n_out)) / B).astype(np.float32)
    W = rng.standard_normal(P).astype(np.float32)
    V = (0.1 * rng.standard_normal(P)).astype(np.float32)
    lr, gamma = 0.05, 0.9
    t = lambda a: torch.from_numpy(a.copy()).to(dev)
    tW, tV = t(W), t(V)
    tF = torch.full((P,), 7.0, device=dev) if sF > 0 else None
    tB = torch.full((P,), 9.0, device=dev) if (sB > 0 and sB != sF) else None
    st.dw_update_raw(MODES[mode], t(X), t(dZ), tW, tV, tF, tB, lr, gamma, sF, sB)
    torch.cuda.synchronize()
    g = np.concatenate([(X.astype(np.float64).T @ dZ.astype(np.float64)).ravel(), dZ.astype(np.float64).sum(0)])
    v64 = 0.9 * V.astype(np.float64) + 0.1 * g
    w64 = W.astype(np.float64) - lr * v64
    scale_g = np.concatenate([(np.abs(X.astype(np.float64)).T @ np.abs(dZ.astype(np.float64))).ravel(),
                              np.abs(dZ.astype(np.float64)).sum(0)])
    tol_v = 0.1 * 1e-5 * scale_g + 2e-7 * np.abs(v64) + 1e-30
    assert np.all(np.abs(tV.cpu().numpy() - v64) <= tol_v)
    assert np.all(np.abs(tW.cpu().numpy() - w64) <= lr * tol_v + 2e-7 * np.abs(w64))
    if tF is not None:
        ref = O.predict(w64, v64, sF, lr)
        assert np.all(np.abs(tF.cpu().numpy() - ref) <= (sF + 1) * lr * tol_v + 4e-7 * np.abs(ref))
    if tB is not None:
        ref = O.predict(w64, v64, sB, lr)
        assert np.all(np.abs(tB.cpu().numpy() - ref) <= (sB + 1) * lr * tol_v + 4e-7 * np.abs(ref))


@pytest.mark.parametrize("n", [0, 5, 1_000_003])
def test_prediction_error_kernel_vs_oracle(st, n):
    """Fig. 7 prediction-accuracy sums against the oracle's RMSE on the same
    fp32 arrays (fp64 accumulation on both sides; only the summation order differs)."""
    rng = np.random.default_rng(n)
    Wo = rng.standard_normal(n).astype(np.float32)
    Vo = (0.1 * rng.standard_normal(n)).astype(np.float32)
    Wn = (Wo - 0.02 * rng.standard_normal(n)).astype(np.float32)
    lr = 0.05
    dev = torch.device("cuda", 0)
    t = [torch.from_numpy(a).to(dev) for a in (Wo, Vo, Wn)]
    for s_ in (0, 1, 2, 3):
        sp, ss = st.prediction_error_raw(t[0], t[1], t[2], s_, lr)
        if n == 0:
            assert sp == ss == 0.0
            continue
        rp, rs = O.prediction_rmse(Wo.astype(np.float64), Vo.astype(np.float64), Wn.astype(np.float64), s_,
                                   float(np.float32(lr)))
        assert math.sqrt(sp / n) == pytest.approx(rp, rel=1e-12)
        assert math.sqrt(ss / n) == pytest.approx(rs, rel=1e-12)
