"""Development: phase timeline of the persistent LSTM recurrence (k_lstm_rec.cu rec_mark).
Needs the dev build: ST_LIB_PATH=paper_1809_02839_b200/_var/dev/libspectrain.so ST_LSTM_DBG=1 (fwd) / 2 (bwd).
Runs the BJ configs[2] LM at one stage for 3 mini-batches and prints, per phase, the median
over CTAs and steps of: barrier→MMA done, MMA done→epilogue, epilogue→tile synced,
cells, and the step period."""
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import paper_1809_02839_b200 as st
    from paper_1809_02839_b200 import _lib
    import synthdata as sd
    model, B = bench.workload("lstm_lm", 1)[:2]
    kinds = {sd.DENSE: st.ST_LAYER_DENSE, sd.EMBED: st.ST_LAYER_EMBED, sd.LSTM: st.ST_LAYER_LSTM}
    layers = [(l.n_in, l.n_out, st.ST_ACT_RELU if l.act == sd.RELU else st.ST_ACT_NONE, 1 if l.bias else 0,
               kinds[l.kind], l.hw) for l in model.layers]
    T = model.seq_len
    M = 3
    dev = torch.device("cuda", 0)
    s = st.Stage(layers, [], 0, B, 1e-3, 0.9, gemm=st.ST_GEMM_FP32X3, transport=st.ST_TRANSPORT_NCCL, device=0,
                 max_minibatches=M, seq_len=T)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    import dataclasses
    bench.init_params(s, dataclasses.replace(model, cuts=()).layers, dev, g)
    xs = torch.randint(0, model.layers[0].n_in, (M, B * T), device=dev, dtype=torch.int32, generator=g)
    ys = torch.randint(0, model.layers[-1].n_out, (M, B * T), device=dev, dtype=torch.int32, generator=g)
    s.run(M, xs, ys)
    torch.cuda.synchronize()
    n = 40 * 160 * 8
    buf = (ctypes.c_uint64 * n)()
    lib = _lib.lib
    assert lib.st_dev_lstm_rec_timeline(buf, n) == 0
    a = np.frombuffer(buf, dtype=np.uint64).reshape(40, 160, 8).astype(np.int64)
    G = int((a[2, :, 0] > 0).sum())
    a = a[:, :G, :]
    out = {"ctas": G}
    ph = {"mma": (0, 1), "to_epilogue": (1, 2), "partial_write": (2, 6), "tile_sync": (6, 3), "cells": (3, 5), "first_batch": (3, 7),
          "cell_fences": (5, 4)}
    for k, (x, y) in ph.items():
        d = (a[1:T, :, y] - a[1:T, :, x]) / 1e3
        out[k + "_us_median"] = round(float(np.median(d)), 2)
        out[k + "_us_max"] = round(float(np.median(d.max(axis=1))), 2)
    # barrier: last cell arrival of step i−1 → this CTA's producer released
    lat = (a[2:T, :, 0] - a[1:T - 1, :, 4].max(axis=1, keepdims=True)) / 1e3
    out["barrier_release_us_median"] = round(float(np.median(lat)), 2)
    per = (a[2:T, :, 0].min(axis=1) - a[1:T - 1, :, 0].min(axis=1)) / 1e3
    if T <= 40:  # whole kernel: first CTA start to last CTA's final grid arrival
        out["kernel_us"] = round(float((a[T - 1, :, 4].max() - a[0, :, 6].min()) / 1e3), 1)
        out["first_mma_phase_us"] = round(float(np.median(a[1, :, 1] - a[1, :, 0]) / 1e3), 2)
        out["t0_cells_us"] = round(float((a[0, :, 4].max() - a[0, :, 6].min()) / 1e3), 2)
    out["step_period_us_median"] = round(float(np.median(per)), 2)
    print(json.dumps(out))
    s.close()


if __name__ == "__main__":
    main()
