"""VGG-16 full size, M mini-batches: the V / ΔW spread against the fp64 oracle for the
8-stage pipeline and the 1-stage run, with the 3xTF32 tensor-core GEMMs and with the
CUDA-core fp32 GEMMs (ST_GEMM_SIMT) — if both arithmetic paths show the same spread, it
comes from the fp32-vs-fp64 ReLU / max-pool decisions (reading D24), not a kernel."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synthdata as sd
from oracle import spectrain_oracle as O
from tests.gpu_helpers import build_pipeline, rel_l2, run_pipeline
import paper_1809_02839_b200 as st

M, B, LR = int(sys.argv[1]) if len(sys.argv) > 1 else 10, 128, 0.01
out = {}
for S in (8, 1):
    model = sd.config_vgg16(S)
    w0, X, Y = sd.parity_inputs(model, M, B, seed=0)
    ref = O.run(model, sd.widen(w0), X.astype(np.float64), Y, float(np.float32(LR)), float(np.float32(0.9)))
    W0 = np.concatenate(sd.widen(w0))
    for gname, gemm in (("fp32x3", st.ST_GEMM_FP32X3), ("simt_fp32", st.ST_GEMM_SIMT)):
        stages = build_pipeline(model, B, LR, gemm=gemm, max_mb=M)
        try:
            W, V, losses, traces = run_pipeline(stages, w0, X, Y)
        finally:
            for s in stages:
                s.close()
        Wc, Wr = np.concatenate(W), np.concatenate(ref.W)
        out[f"S{S}_{gname}"] = {"loss": rel_l2(losses, ref.losses), "w": rel_l2(Wc, Wr),
                                "dw": rel_l2(Wc - W0, Wr - W0), "v": rel_l2(np.concatenate(V), np.concatenate(ref.V))}
        print(f"S{S}_{gname}", out[f"S{S}_{gname}"], flush=True)
json.dump(out, open(os.path.join("gpurun_out", f"vgg_spread_M{M}.json"), "w"), indent=1)
