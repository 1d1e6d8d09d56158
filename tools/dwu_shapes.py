"""Development: fused dW + update time for equal-parameter layer shapes (DRAM locality test)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.time_gemm import t_op
for (i, o) in [(8192, 8192), (65536, 1024), (16384, 4096), (4096, 16384), (1024, 65536)]:
    us, tf, gbs = t_op(3, 0, 128, i, o)
    print(f"dWU in={i} out={o}: {us:8.1f} us  {gbs:7.1f} GB/s (16 B/param)")
