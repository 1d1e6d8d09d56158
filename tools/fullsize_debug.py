"""Development: per-layer V / W errors of the full-size wide FCN (1 stage, bench path) vs the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthdata as sd
from oracle import spectrain_oracle as O
import paper_1809_02839_b200 as st
from tests.gpu_helpers import layers_of, rel_l2
LR = 0.01
GEMM = {"fp32x3": st.ST_GEMM_FP32X3, "simt": st.ST_GEMM_SIMT}[os.environ.get("GEMM", "fp32x3")]
M = int(os.environ.get("M", "2"))
model = sd.config_wide_fcn(1, width=int(os.environ.get("WIDTH", "8192")), hidden_layers=int(os.environ.get("LAYERS", "8")))
w0, X, Y = sd.parity_inputs(model, M, 128, seed=0)
dev = torch.device("cuda", 0)
s = st.Stage(layers_of(model), model.cuts, 0, 128, LR, 0.9, transport=st.ST_TRANSPORT_NCCL, device=0, max_minibatches=M, gemm=GEMM)
s.set_params(w0[0])
losses = s.run(M, torch.from_numpy(X).to(dev), torch.from_numpy(Y).to(dev), want_losses=True)
W, V, _ = s.get_params()
s.close()
ref = O.run(model, sd.widen(w0), X.astype(np.float64), Y, float(np.float32(LR)), float(np.float32(0.9)))
print("loss", losses, ref.losses)
off = 0
for i, L in enumerate(model.layers):
    n = L.n_in * L.n_out
    for name, a, b in (("W", V[off:off + n], ref.V[0][off:off + n]), ("b", V[off + n:off + n + L.n_out], ref.V[0][off + n:off + n + L.n_out])):
        d = np.abs(a - b)
        print(f"layer {i} {name}: relL2 {rel_l2(a, b):.3e} maxabs {d.max():.3e} |ref| {np.abs(b).max():.3e} n_bad(>1e-3 rel) {(d > 1e-3 * np.abs(b).max()).sum()}")
    off += L.n_params
