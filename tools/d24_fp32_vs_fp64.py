"""Reading D24 pinned without the GPU: the oracle's arithmetic in NumPy float32 against
the same arithmetic in float64, at BASELINE.json's full width (configs[1]: the wide FCN
784 → 8 × 8192 → 10, batch 128, N = 1 so SpecTrain is momentum SGD).

Three trainers run in lockstep on the same mini-batches:
  fp64  — the oracle's stage_forward / loss_and_grad / stage_backward / update_smoothed
          (spectrain_oracle.py) in float64;
  fp32  — the same oracle functions on float32 arrays (NumPy keeps float32: sgemm,
          float32 elementwise);
  fp32m — float32 arithmetic written out here (the same formulas: Z = A·W + b, ReLU,
          softmax CE, dZ = dA ⊙ mask, g = Aᵀ·dZ, dA = dZ·Wᵀ, Eq. 1, D1 apply) with every
          ReLU decision taken from the fp64 run (mask = 1[Z64 > 0]).
If the spread of V / ΔW between fp32 and fp64 comes from ReLU decisions on
pre-activations within rounding of 0 (D24), fp32m collapses to the fp32 rounding level
while fp32 does not. Output: profiles/r2_d24_fp32_vs_fp64.json (metrics after each
mini-batch count in --report); tests/test_gpu_fullsize.py sets its gates from it.

    python tools/d24_fp32_vs_fp64.py [--M 20] [--report 1,2,5,20] [--width 8192] [--layers 8]
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


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def masked_step(layers, W, V, X, Y, masks, eta, gamma):
    """One float32 momentum-SGD step with the ReLU decisions `masks` (one per hidden
    layer, from the fp64 run) instead of its own."""
    parts = O.unpack_stage(layers, W)
    A = X
    acts = []
    for li, (L, (Wl, bl)) in enumerate(zip(layers, parts)):
        Z = A @ Wl + bl
        acts.append(A)
        A = Z * masks[li] if L.act == "relu" else Z
    _, dZ = O.loss_and_grad("softmax_ce", A, Y)
    dZ = dZ.astype(np.float32)
    grads = [None] * len(layers)
    for li in range(len(layers) - 1, -1, -1):
        L = layers[li]
        Wl, _ = parts[li]
        if L.act == "relu":
            dZ = dZ * masks[li]
        grads[li] = (acts[li].T @ dZ, dZ.sum(axis=0))
        if li > 0:
            dZ = dZ @ Wl.T
    g = O.pack_stage(layers, grads).astype(np.float32)
    V = (np.float32(gamma) * V + np.float32(1.0 - gamma) * g).astype(np.float32)
    W = (W - np.float32(eta) * V).astype(np.float32)
    return W, V


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=20)
    ap.add_argument("--report", default="1,2,5,20")
    ap.add_argument("--width", type=int, default=8192)
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_d24_fp32_vs_fp64.json"))
    a = ap.parse_args()
    report = {int(x) for x in a.report.split(",")}
    model = sd.config_wide_fcn(1, width=a.width, hidden_layers=a.layers)
    layers = model.layers
    w0, X, Y = sd.parity_inputs(model, a.M, 128, seed=a.seed)
    eta, gamma = float(np.float32(a.lr)), float(np.float32(0.9))
    W0 = np.asarray(w0[0], np.float64)
    W64, V64 = W0.copy(), np.zeros_like(W0)
    W32, V32 = np.array(w0[0], np.float32), np.zeros(W0.size, np.float32)
    Wm, Vm = W32.copy(), V32.copy()
    out = {"what": "oracle arithmetic in NumPy float32 vs float64, plus float32 with the fp64 ReLU decisions "
                   "(reading D24 pin; no GPU involved)",
           "model": f"784-{a.layers}x{a.width}-10, B=128, N=1, lr={a.lr}, gamma=0.9, seed={a.seed}",
           "after": {}}
    t0 = time.time()
    for i in range(a.M):
        # fp64 oracle step (its ReLU decisions are recorded for fp32m)
        out64, st64 = O.stage_forward(layers, W64, X[i].astype(np.float64))
        masks = [(Z > 0.0).astype(np.float32) for (_, Z) in st64]
        _, dZ64 = O.loss_and_grad(model.loss, out64, Y[i])
        g64, _ = O.stage_backward(layers, W64, st64, dZ64, need_dA_in=False)
        del st64
        V64 = O.update_smoothed(V64, g64, gamma)
        W64 = W64 - eta * V64
        del g64
        # fp32: the oracle's functions on float32 arrays
        out32, st32 = O.stage_forward(layers, W32, X[i])
        _, dZ32 = O.loss_and_grad(model.loss, out32, Y[i])
        g32, _ = O.stage_backward(layers, W32, st32, dZ32.astype(np.float32), need_dA_in=False)
        flips = sum(int(np.count_nonzero((Z > 0) != (m > 0))) for (_, Z), m, L in zip(st32, masks, layers)
                    if L.act == "relu")
        del st32
        V32 = O.update_smoothed(V32, g32.astype(np.float32), np.float32(gamma)).astype(np.float32)
        W32 = (W32 - np.float32(eta) * V32).astype(np.float32)
        del g32
        # fp32 with the fp64 decisions
        Wm, Vm = masked_step(layers, Wm, Vm, X[i], Y[i], masks, eta, gamma)
        n = i + 1
        if n in report:
            out["after"][str(n)] = {
                "fp32": {"w": rel(W32, W64), "dw": rel(W32 - W0, W64 - W0), "v": rel(V32, V64)},
                "fp32_fp64_masks": {"w": rel(Wm, W64), "dw": rel(Wm - W0, W64 - W0), "v": rel(Vm, V64)},
                "relu_decisions_differing_this_step": flips,
                "relu_decisions_this_step": int(sum(m.size for m, L in zip(masks, layers) if L.act == "relu")),
            }
            print(n, json.dumps(out["after"][str(n)]), flush=True)
    out["seconds"] = time.time() - t0
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
