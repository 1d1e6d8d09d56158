"""Development: per-CTA timeline of the FP32X3 fwd TS kernel (ST_GEMM_DEV_FLAGS bit 7 must be
set): python tools/ts_timeline.py op B in out"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1809_02839_b200 as st
op, B, n_in, n_out = (int(a) for a in sys.argv[1:5])
dev = torch.device("cuda", 0)
X = torch.randn(B, n_in, device=dev); W = torch.randn(n_in, n_out, device=dev) * 0.01
dZ = torch.randn(B, n_out, device=dev); bias = torch.randn(n_out, device=dev)
work = torch.zeros(int(st._lib.lib.st_gemm_workspace_bytes(B, n_in, n_out)), dtype=torch.uint8, device=dev)
args = (X, W, bias, None, torch.empty(B, n_out, device=dev)) if op == 0 else (dZ, W, X, None, torch.empty(B, n_in, device=dev))
reps = int(os.environ.get("REPS", "100"))  # warm back-to-back launches; the last one is reported
for rep in range(reps):
    st.gemm_raw(op, 0, B, n_in, n_out, *args, relu=(op == 0), work=work)
torch.cuda.synchronize()
t = work[32768:32768 + 240 * 128].cpu().numpy().view(np.uint64).reshape(240, 16).astype(np.int64)
used = t[:, 0] > 0
t = t[used]
t0 = t[:, 0].min()
rel = np.where(t > 0, t - t0, -1)
names = ["start", "setup", "mma_done", "acc_full", "partial", "atomic", "fixup", "epi_end", "dealloc"]
print("CTAs:", used.sum(), " kernel span (ns):", rel.max())
for i, n in enumerate(names):
    col = rel[:, i]; col = col[col >= 0]
    if len(col): print(f"{n:9s} min {col.min():7d}  median {int(np.median(col)):7d}  max {col.max():7d}  (n={len(col)})")
acct = ["mma wait t_full", "mma wait b_full", "mma issue+commit", "conv wait a_full", "conv wait t_empty",
        "conv st+arrive", "prodA wait a_free"]
for i, n in enumerate(acct):
    col = t[:, 9 + i]; col = col[col > 0]
    if len(col): print(f"{n:18s} cycles: median {int(np.median(col)):9d}  max {col.max():9d}  (n={len(col)})")
mm = t[:, 9:12].sum(1)
ok = (mm > 0) & (t[:, 2] > 0)
if ok.any():
    print("SM clock during the main loop (MMA-thread cycles / ns): %.2f GHz" % np.median(mm[ok] / (t[ok, 2] - t[ok, 1])))
