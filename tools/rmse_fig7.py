"""Fig. 7 of the paper: accuracy of the weight prediction during pipelined
SpecTrain training — RMSE(Ŵ_t, W_t) of the Eq. 4 prediction made s updates earlier
against RMSE(W_{t−s}, W_t) of the stale weights, for s = 1, 2, 3.

Setting (synthetic stand-in): the SNN-shaped FCN — 32 fully-connected
layers of 2048 units on 3072-dim (CIFAR-shaped) inputs, 10 classes — but with ReLU
instead of SELU (the library has no SELU), batch 128, η = 1e-3, γ = 0.9, cut into 4
stages run on ONE GPU (LOCAL transport) task by task through the verbs API
(st_stage_forward / st_stage_backward / st_predict_and_update). After every update of
every stage the tool keeps (W, V) of the last 4 versions on the device and evaluates
both errors with the library's st_prediction_error_raw kernel; the per-version RMSE is
taken over all parameters of all stages.

    python tools/rmse_fig7.py [--steps 300] [--out profiles/r1_fig7_rmse.json]
"""
import argparse
import collections
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1809_02839_b200 as st  # noqa: E402
import synthdata as sd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--width", type=int, default=2048)
    ap.add_argument("--stages", type=int, default=4)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_fig7_rmse.json"))
    a = ap.parse_args()
    widths = [3072] + [a.width] * a.layers + [10]
    model = sd.mlp(widths, cuts=sd.even_cuts(len(widths) - 1, a.stages))
    B, M, N = 128, a.steps, a.stages
    dev = torch.device("cuda", 0)
    layers = [(l.n_in, l.n_out, st.ST_ACT_RELU if l.act == sd.RELU else st.ST_ACT_NONE, 1) for l in model.layers]
    stages = [st.Stage(layers, model.cuts, k, B, a.lr, 0.9, transport=st.ST_TRANSPORT_LOCAL, device=0,
                       max_minibatches=M) for k in range(N)]
    st.connect_local(stages)
    # He-uniform weights (±√(6/fan_in)), zero biases: a 32-layer ReLU stack keeps its
    # activation scale (Glorot would shrink it ~2× per layer and the gradients vanish);
    # SNN's own LeCun init assumes SELU
    rng = np.random.default_rng(0)
    w0 = []
    for k in range(N):
        parts = []
        for L in model.stage_layers(k):
            r = math.sqrt(6.0 / L.n_in)
            parts += [rng.uniform(-r, r, L.n_in * L.n_out), np.zeros(L.n_out)]
        w0.append(np.concatenate(parts).astype(np.float32))
    for s, w in zip(stages, w0):
        s.set_params(w)
    X, Y = sd.images_and_labels(3072, 10, M, B, 1, "teacher")
    xs = torch.from_numpy(X.astype(np.float32)).to(dev)
    ys = torch.from_numpy(Y).to(dev)
    n_k = [s.params for s in stages]
    hist = [collections.deque(maxlen=4) for _ in range(N)]  # (W, V) after each update of stage k
    for k, s in enumerate(stages):
        s.sync()
        with torch.cuda.stream(s.stream):
            hist[k].append((s.W[:4 * n_k[k]].view(torch.float32).clone(),
                            s.V[:4 * n_k[k]].view(torch.float32).clone()))
    # sums[t][s] = [Σ e_pred², Σ e_stale²] over stages (t = the stage-local update count)
    sums = collections.defaultdict(lambda: {1: [0.0, 0.0, 0], 2: [0.0, 0.0, 0], 3: [0.0, 0.0, 0]})
    progs = [st.program(N, k, M) for k in range(N)]
    pc = [0] * N
    done_f, done_b = set(), set()
    nupd = [0] * N
    losses = np.full(M, np.nan)
    t0 = time.time()
    while any(pc[k] < len(progs[k]) for k in range(N)):
        for k in range(N):
            while pc[k] < len(progs[k]):
                _, _, d, i = progs[k][pc[k]][:4]
                if d == st.ST_FWD and (k == 0 or (k - 1, i) in done_f):
                    l = stages[k].forward(i, xs[i] if k == 0 else None, ys[i] if k == N - 1 else None,
                                          want_loss=(k == N - 1))
                    if k == N - 1:
                        losses[i] = l
                    done_f.add((k, i))
                elif d == st.ST_BWD and (k == N - 1 or (k + 1, i) in done_b):
                    stages[k].backward(i)
                    stages[k].predict_and_update()
                    stages[k].sync()
                    Wn = stages[k].W[:4 * n_k[k]].view(torch.float32)
                    nupd[k] += 1
                    t = nupd[k]
                    for s_ in (1, 2, 3):
                        if len(hist[k]) >= s_:
                            Wo, Vo = hist[k][-s_]
                            ep, es = st.prediction_error_raw(Wo, Vo, Wn, s_, a.lr, stream=stages[k].stream)
                            e = sums[t][s_]
                            e[0] += ep
                            e[1] += es
                            e[2] += n_k[k]
                    with torch.cuda.stream(stages[k].stream):  # ordered before the stage's next update
                        hist[k].append((Wn.clone(), stages[k].V[:4 * n_k[k]].view(torch.float32).clone()))
                    done_b.add((k, i))
                else:
                    break
                pc[k] += 1
    wall = time.time() - t0
    curve = []
    for t in sorted(sums):
        row = {"t": t}
        for s_ in (1, 2, 3):
            p, q, n = sums[t][s_]
            if n == sum(n_k):  # every stage contributed
                row[f"rmse_pred_s{s_}"] = math.sqrt(p / n)
                row[f"rmse_stale_s{s_}"] = math.sqrt(q / n)
        curve.append(row)
    summary = {}
    for s_ in (1, 2, 3):
        rp = [r[f"rmse_pred_s{s_}"] for r in curve if f"rmse_pred_s{s_}" in r and r["t"] > M // 5]
        rs = [r[f"rmse_stale_s{s_}"] for r in curve if f"rmse_stale_s{s_}" in r and r["t"] > M // 5]
        summary[f"s{s_}"] = {"mean_rmse_pred": float(np.mean(rp)), "mean_rmse_stale": float(np.mean(rs)),
                             "pred_over_stale": float(np.mean(rp) / np.mean(rs))}
    res = {"what": "Fig. 7 (P:346-355): RMSE of Eq. 4-predicted vs stale weights during 4-stage SpecTrain training",
           "model": f"FCN {widths[0]}-{a.layers}x{a.width}-10 ReLU, He-uniform init (SNN-shaped, P:385; SELU -> ReLU)",
           "stages": N, "batch": B, "lr": a.lr, "gamma": 0.9, "minibatches": M,
           "data": "synthetic U[0,1) 3072-dim inputs, teacher labels (synthdata, seed 1)",
           "summary_t_gt": M // 5, "summary": summary, "loss_first_last": [float(losses[0]), float(losses[-1])],
           "wall_s": wall, "curve": curve}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "curve"}))
    for s in stages:
        s.close()


if __name__ == "__main__":
    main()
