"""Development: FP32X3 fwd / dX time vs K (in for fwd, out for dX) at fixed M = 8192, B = 128,
to separate per-k-block pipeline cost from fixed (epilogue / launch) cost."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.time_gemm import t_op
for K in (256, 1024, 4096, 8192):
    f = t_op(0, 0, 128, K, 8192)[0]
    d = t_op(1, 0, 128, 8192, K)[0]
    print(f"K={K:5d} fwd {f:7.1f} us  dX {d:7.1f} us", flush=True)
