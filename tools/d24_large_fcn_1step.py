"""Reading D24 at the size of BASELINE.json configs[4] (784 → 16 × 16384 → 10, batch 128),
one mini-batch, without the GPU: the oracle's arithmetic (stage_forward / loss_and_grad /
stage_backward, one layer at a time — the model is 4.04G parameters, so each layer's
block is redrawn from its own seed as tests/test_gpu_fullsize.py does) in NumPy float32
against float64, plus float32 with every ReLU decision taken from the float64 run, plus an emulation of
the GPU's 3xTF32 products (operands truncated to tf32 — the tensor core truncates fp32
inputs, DESIGN §5 — hi·hi + lo·hi + hi·lo summed exactly in float64, the result rounded
to float32: the dropped lo·lo term is the dominant error, ≈ 2^-20 of each product).

After one update from V = 0, V = (1 − γ)·g, so the per-layer relative L2 spread of g
between the precisions is the spread of V that test_large_fcn_full_size_one_step_sampled
can expect between the GPU (3xTF32, fp32-faithful) and the fp64 oracle. Output:
profiles/r2_d24_large_fcn_1step.json (per layer: fp32 vs fp64, fp32-with-fp64-decisions
vs fp64, and how many decisions differ).

    python tools/d24_large_fcn_1step.py [--seed 11] [--width 16384] [--layers 16]
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


def trunc_tf32(x):
    x = np.ascontiguousarray(x, np.float32)
    return (x.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def mm_x3(a, b):
    """3xTF32 product as the GPU forms it (lo·lo dropped), exact sums, rounded to fp32."""
    ah, bh = trunc_tf32(a), trunc_tf32(b)
    al, bl = (a.astype(np.float32) - ah), (b.astype(np.float32) - bh)
    ah, bh, al, bl = (t.astype(np.float64) for t in (ah, bh, al, bl))
    return (ah @ bh + al @ bh + ah @ bl).astype(np.float32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seed", type=int, default=11)
    ap.add_argument("--width", type=int, default=16384)
    ap.add_argument("--layers", type=int, default=16)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_d24_large_fcn_1step.json"))
    ap.add_argument("--x3", action="store_true", help="add the 3xTF32 emulation (3 fp64 GEMMs per product)")
    a = ap.parse_args()
    model = sd.mlp([784] + [a.width] * a.layers + [10], cuts=[])
    L = model.layers
    B = 128
    X, Y = sd.images_and_labels(784, 10, 1, B, a.seed + 1, "teacher")
    t0 = time.time()
    A64, A32, A32m = X[0].astype(np.float64), X[0].astype(np.float32), X[0].astype(np.float32)
    st64, st32, st32m, masks, flips = [], [], [], [], []
    A3, st3, masks3, flips3 = X[0].astype(np.float32), [], [], []
    for i, layer in enumerate(L):
        w32 = sd.glorot_dense_layer_f32(layer, a.seed, i)
        w64 = w32.astype(np.float64)
        A64, s64 = O.stage_forward([layer], w64, A64)
        A32, s32 = O.stage_forward([layer], w32, A32)
        Wl, bl = O.unpack_stage([layer], w32)[0]
        Z = A32m @ Wl + bl
        st32m.append(A32m)
        if layer.act == "relu":
            m64 = (A64 > 0)
            masks.append(m64.astype(np.float32))
            flips.append(int(np.count_nonzero(m64 != (A32 > 0))))
            A32m = Z * masks[-1]
        else:
            masks.append(None)
            flips.append(0)
            A32m = Z
        st64.append(s64)
        st32.append(s32)
        if a.x3:
            st3.append(A3)
            Z3 = (mm_x3(A3, Wl) + bl).astype(np.float32)
            if layer.act == "relu":
                masks3.append((Z3 > 0).astype(np.float32))
                flips3.append(int(np.count_nonzero((A64 > 0) != (Z3 > 0))))
                A3 = Z3 * masks3[-1]
            else:
                masks3.append(None)
                flips3.append(0)
                A3 = Z3
        print(f"fwd layer {i}: {time.time() - t0:.0f} s, decisions differing {flips[-1]}"
              + (f" (3xTF32: {flips3[-1]})" if a.x3 else ""), flush=True)
    _, d64 = O.loss_and_grad(model.loss, A64, Y[0])
    _, d32 = O.loss_and_grad(model.loss, A32, Y[0])
    _, d32m = O.loss_and_grad(model.loss, A32m, Y[0])
    d32 = d32.astype(np.float32)
    d32m = d32m.astype(np.float32)
    if a.x3:
        _, d3 = O.loss_and_grad(model.loss, A3, Y[0])
        d3 = d3.astype(np.float32)
    per_layer = []
    for i in range(len(L) - 1, -1, -1):
        layer = L[i]
        w32 = sd.glorot_dense_layer_f32(layer, a.seed, i)
        w64 = w32.astype(np.float64)
        g64, d64 = O.stage_backward([layer], w64, st64[i], d64, need_dA_in=i > 0)
        g32, d32 = O.stage_backward([layer], w32, st32[i], d32, need_dA_in=i > 0)
        Wl, _ = O.unpack_stage([layer], w32)[0]
        dZ = d32m * masks[i] if masks[i] is not None else d32m
        gW = st32m[i].T @ dZ
        gb = dZ.sum(axis=0)
        g32m = np.concatenate([gW.ravel(), gb])
        if i > 0:
            d32m = (dZ @ Wl.T).astype(np.float32)
        rec = {"layer": i, "v_rel_fp32": rel(g32, g64), "v_rel_fp32_fp64_decisions": rel(g32m, g64),
               "decisions_differing_fwd": flips[i]}
        if a.x3:
            dZ3 = d3 * masks3[i] if masks3[i] is not None else d3
            g3 = np.concatenate([mm_x3(st3[i].T, dZ3).ravel(), dZ3.sum(axis=0)])
            if i > 0:
                d3 = mm_x3(dZ3, np.ascontiguousarray(Wl.T))
            st3[i] = None
            rec.update({"v_rel_3xtf32": rel(g3, g64), "decisions_differing_fwd_3xtf32": flips3[i]})
        per_layer.append(rec)
        st64[i] = st32[i] = st32m[i] = None
        print(f"bwd layer {i}: {time.time() - t0:.0f} s {per_layer[-1]}", flush=True)
    out = {"what": "reading D24 at BJ configs[4] full size, one mini-batch (V = (1-gamma) g after one update)",
           "model": f"784-{a.layers}x{a.width}-10, batch {B}, seed {a.seed} (tests/test_gpu_fullsize.py inputs)",
           "per_layer": per_layer, "seconds": round(time.time() - t0, 1)}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out["per_layer"], indent=0))


if __name__ == "__main__":
    main()
