"""Reading D24 pinned without the GPU: the oracle's own arithmetic run in NumPy float32
against the same arithmetic in float64, at BASELINE.json's full width (configs[1]: the
wide FCN 784 → 8 × 8192 → 10, batch 128, N = 1 so SpecTrain reduces to momentum SGD,
P:215-221), M mini-batches.

If the GPU/oracle spread of V and ΔW at full width comes from ReLU decisions taken on
pre-activations within fp32 rounding of 0 (D24) and not from a kernel error, a plain
fp32 CPU run of the same algorithm shows the same spread. The per-row statistics tell
the two apart: a flip moves whole rows of a gradient, so it raises the rel-L2 while
the median row error stays at the fp32 level; a systematic gradient error moves every
row. Output: profiles/r2_d24_fp32_vs_fp64.json (used to set the full-size gates in
tests/test_gpu_fullsize.py).

    python tools/d24_fp32_vs_fp64.py [--M 20] [--width 8192] [--layers 8]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synthdata as sd  # noqa: E402
from oracle import spectrain_oracle as O  # noqa: E402


def train(model, w0, X, Y, eta, gamma, dtype):
    """N = 1 SpecTrain = sequential momentum SGD (Eq. 1 + D1 apply) with the oracle's
    stage_forward / loss_and_grad / stage_backward / update_smoothed, every array in
    `dtype` (NumPy keeps float32 operands in float32: sgemm, float32 elementwise)."""
    W = np.array(w0, dtype=dtype)
    V = np.zeros_like(W)
    eta_, gamma_ = dtype(eta), dtype(gamma)
    losses = []
    for i in range(X.shape[0]):
        out, stash = O.stage_forward(model.layers, W, X[i].astype(dtype))
        loss, dZ = O.loss_and_grad(model.loss, out, Y[i])
        g, _ = O.stage_backward(model.layers, W, stash, dZ.astype(dtype), need_dA_in=False)
        V = O.update_smoothed(V, g.astype(dtype), gamma_).astype(dtype)
        W = (W - eta_ * V).astype(dtype)
        losses.append(loss)
    return W, V, np.array(losses)


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def row_stats(A, B, layers):
    """Per dense layer: rel-L2 and the median over weight rows of the row rel-error."""
    out = []
    off = 0
    for L in layers:
        n = L.n_in * L.n_out
        a = np.asarray(A[off:off + n], np.float64).reshape(L.n_in, L.n_out)
        b = np.asarray(B[off:off + n], np.float64).reshape(L.n_in, L.n_out)
        nb = np.linalg.norm(b, axis=1)
        ok = nb > 0
        re = np.linalg.norm(a - b, axis=1)[ok] / nb[ok]
        out.append({"rel_l2": rel(a, b), "row_median": float(np.median(re)) if re.size else 0.0,
                    "row_p99": float(np.quantile(re, 0.99)) if re.size else 0.0})
        off += L.n_params
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=20)
    ap.add_argument("--width", type=int, default=8192)
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_d24_fp32_vs_fp64.json"))
    a = ap.parse_args()
    model = sd.config_wide_fcn(1, width=a.width, hidden_layers=a.layers)
    w0, X, Y = sd.parity_inputs(model, a.M, 128, seed=a.seed)
    lr, gamma = float(np.float32(a.lr)), float(np.float32(0.9))
    t0 = time.time()
    W64, V64, l64 = train(model, np.asarray(w0[0], np.float64), X, Y, lr, gamma, np.float64)
    t1 = time.time()
    W32, V32, l32 = train(model, w0[0], X, Y, lr, gamma, np.float32)
    t2 = time.time()
    W0 = np.asarray(w0[0], np.float64)
    res = {
        "what": "oracle arithmetic in NumPy float32 vs float64 (reading D24 pin, no GPU involved)",
        "model": f"784-{a.layers}x{a.width}-10, B=128, N=1, lr={a.lr}, gamma=0.9, M={a.M}, seed={a.seed}",
        "w_rel_l2": rel(W32, W64), "dw_rel_l2": rel(W32 - W0, W64 - W0), "v_rel_l2": rel(V32, V64),
        "loss_rel_l2": rel(l32, l64),
        "v_per_layer": row_stats(V32, V64, model.layers),
        "dw_per_layer": row_stats(W32 - W0, W64 - W0, model.layers),
        "seconds": {"fp64": t1 - t0, "fp32": t2 - t1},
    }
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v for k, v in res.items() if not k.endswith("per_layer")}, indent=1))


if __name__ == "__main__":
    main()
