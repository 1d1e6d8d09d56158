"""Per-layer forward / backward time of a workload at one stage (ST_PROF_LAYERS brackets,
st_get_layer_profile) with each layer's fp32 FLOP rate against the 3xTF32 effective peak.

  python tools/layer_prof.py vgg16 [--reps 5]   -> JSON lines, one per layer
"""
import argparse
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import paper_1809_02839_b200 as st
    import synthdata as sd
    p = argparse.ArgumentParser()
    p.add_argument("workload")
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--warm", type=int, default=3)
    a = p.parse_args()
    model, B = bench.workload(a.workload, 1)[:2]
    dev = torch.device("cuda", 0)
    kinds = {sd.DENSE: st.ST_LAYER_DENSE, sd.EMBED: st.ST_LAYER_EMBED, sd.LSTM: st.ST_LAYER_LSTM,
             sd.CONV: st.ST_LAYER_CONV, sd.POOL: st.ST_LAYER_POOL}
    layers = [(l.n_in, l.n_out, st.ST_ACT_RELU if l.act == sd.RELU else st.ST_ACT_NONE, 1 if l.bias else 0,
               kinds[l.kind], l.hw) for l in model.layers]
    T = model.seq_len
    R = B * T
    M = a.warm + a.reps
    s = st.Stage(layers, [], 0, B, 1e-3, 0.9, pred=st.ST_PRED_NONE, gemm=st.ST_GEMM_FP32X3,
                 transport=st.ST_TRANSPORT_NCCL, device=0, max_minibatches=M, seq_len=T)
    g = torch.Generator(device=dev)
    g.manual_seed(4321)
    bench.init_params(s, dataclasses.replace(model, cuts=()).layers, dev, g)
    if model.layers[0].kind == sd.EMBED:
        xs = torch.randint(0, model.layers[0].n_in, (M, R), device=dev, dtype=torch.int32, generator=g)
    else:
        xs = torch.rand(M, R, model.layers[0].width_in, device=dev, generator=g)
    ys = torch.randint(0, model.layers[-1].n_out, (M, R), device=dev, dtype=torch.int32, generator=g)
    s.run(a.warm, xs[:a.warm], ys[:a.warm])
    s.set_layer_profiling(True)
    s.run(a.reps, xs[a.warm:], ys[a.warm:])
    ms, cnt = s.layer_profile()
    s.close()
    peak = bench.measured_tensor_peak()[2]  # 3xTF32 effective, TFLOP/s
    tot = [0.0, 0.0]
    for i, L in enumerate(model.layers):
        f = 0.0
        if L.kind == sd.CONV:
            f = 2.0 * B * L.hw * L.hw * L.n_in * L.n_out * 9
        elif L.kind == sd.DENSE:
            f = 2.0 * R * L.n_in * L.n_out
        elif L.kind == sd.LSTM:
            f = 2.0 * B * T * (L.n_in + L.n_out) * 4 * L.n_out
        fw = float(ms[i, 0] / max(1, cnt[i, 0]))
        bw = float(ms[i, 1] / max(1, cnt[i, 1]))
        tot[0] += fw
        tot[1] += bw
        nb = 2 if i > 0 else 1
        print(json.dumps({"layer": i, "kind": L.kind, "n_in": L.n_in, "n_out": L.n_out, "hw": L.hw,
                          "fwd_us": round(fw * 1e3, 1), "bwd_us": round(bw * 1e3, 1),
                          "fwd_frac": round(f / (fw * 1e-3) / (peak * 1e12), 3) if f and fw else None,
                          "bwd_frac": round(nb * f / (bw * 1e-3) / (peak * 1e12), 3) if f and bw else None}))
    print(json.dumps({"total_fwd_us": round(tot[0] * 1e3, 1), "total_bwd_us": round(tot[1] * 1e3, 1),
                      "tf32x3_peak_tflops": round(peak, 1)}))


if __name__ == "__main__":
    main()
