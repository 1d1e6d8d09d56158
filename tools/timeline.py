"""Kernel timeline of a bench workload with real stream concurrency (CUPTI through
torch.profiler: every kernel the library launches, on the compute, side and comm
streams, with device start / end times — unlike ncu, which serialises launches).

    python tools/timeline.py [--workload large_fcn] [--stages 1] [--warm 3] [--M 2]
                             [--out gpurun_out/timeline_<workload>.json]

Prints, for the last mini-batch's backward, each dense layer's dX and dW + update
launches (stream, start, duration) and the per-phase totals: forward, backward, and how
much of the backward had both streams busy. The JSON has every kernel of the session.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="large_fcn")
    ap.add_argument("--stages", type=int, default=1)
    ap.add_argument("--warm", type=int, default=3)
    ap.add_argument("--M", type=int, default=2)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import bench
    import paper_1809_02839_b200 as st
    import synthdata as sd
    model, B, wname = bench.workload(a.workload, a.stages)
    kinds = {sd.DENSE: st.ST_LAYER_DENSE, sd.EMBED: st.ST_LAYER_EMBED, sd.LSTM: st.ST_LAYER_LSTM,
             sd.CONV: st.ST_LAYER_CONV, sd.POOL: st.ST_LAYER_POOL}
    layers = [(l.n_in, l.n_out, st.ST_ACT_RELU if l.act == sd.RELU else st.ST_ACT_NONE, 1 if l.bias else 0,
               kinds[l.kind], l.hw) for l in model.layers]
    dev = torch.device("cuda", 0)
    M = a.warm + a.M
    stages = [st.Stage(layers, model.cuts, k, B, 1e-3, 0.9, transport=(st.ST_TRANSPORT_NCCL if a.stages == 1 else
                                                                        st.ST_TRANSPORT_LOCAL),
                       device=0, max_minibatches=M, seq_len=model.seq_len) for k in range(a.stages)]
    if a.stages > 1:
        st.connect_local(stages)
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    for s in stages:
        bench.init_params(s, model.stage_layers(s.k), dev, g)
    R = B * model.seq_len
    if model.layers[0].kind == sd.EMBED:
        xs = torch.randint(0, model.layers[0].n_in, (M, R), device=dev, dtype=torch.int32, generator=g)
    else:
        xs = torch.rand(M, R, model.layers[0].width_in, device=dev, generator=g)
    ys = torch.randint(0, model.layers[-1].n_out, (M, R), device=dev, dtype=torch.int32, generator=g)

    def session(n, x, y):
        if len(stages) == 1:
            stages[0].run(n, x, y)
        else:
            st.run_group(stages, n, x, y, want_losses=False)

    session(a.warm, xs[:a.warm], ys[:a.warm])
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        session(a.M, xs[a.warm:], ys[a.warm:])
        torch.cuda.synchronize()
    ev = []
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        ev.append({"name": e.name, "start_us": e.time_range.start, "dur_us": e.time_range.end - e.time_range.start,
                   "stream": getattr(e, "device_resource_id", None) or getattr(e, "thread", None)})
    ev.sort(key=lambda d: d["start_us"])
    t0 = ev[0]["start_us"]
    for d in ev:
        d["start_us"] -= t0
    span = ev[-1]["start_us"] + ev[-1]["dur_us"]
    out = a.out or os.path.join(ROOT, "gpurun_out", f"timeline_{a.workload}_s{a.stages}.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    # busy intervals per stream -> concurrency
    streams = sorted({d["stream"] for d in ev}, key=str)
    busy = {}
    for s_ in streams:
        iv = sorted((d["start_us"], d["start_us"] + d["dur_us"]) for d in ev if d["stream"] == s_)
        merged = []
        for b, e_ in iv:
            if merged and b <= merged[-1][1]:
                merged[-1][1] = max(merged[-1][1], e_)
            else:
                merged.append([b, e_])
        busy[str(s_)] = merged
    grid = np.zeros(int(span) + 1, np.int8)
    for s_, iv in busy.items():
        for b, e_ in iv:
            grid[int(b):int(e_) + 1] += 1
    by_name = {}
    for d in ev:
        k = d["name"].split("(")[0][:90]
        t = by_name.setdefault(k, [0, 0.0])
        t[0] += 1
        t[1] += d["dur_us"]
    summary = {"workload": wname, "stages": a.stages, "minibatches": a.M, "span_us": span,
               "span_per_minibatch_us": span / a.M,
               "us_with_0_1_2plus_streams_busy": [int((grid == 0).sum()), int((grid == 1).sum()),
                                                  int((grid >= 2).sum())],
               "per_kernel": sorted([[k, v[0], round(v[1], 1)] for k, v in by_name.items()], key=lambda x: -x[2])}
    with open(out, "w") as f:
        json.dump({"summary": summary, "kernels": ev}, f)
    print(json.dumps(summary, indent=1))
    for s in stages:
        s.close()


if __name__ == "__main__":
    main()
