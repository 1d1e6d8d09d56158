"""Run a single stage GEMM (for ncu): python tools/one_gemm.py op mode B in out"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.time_gemm import t_op
op, mode, B, i, o = (int(a) for a in sys.argv[1:6])
print(t_op(op, mode, B, i, o, reps=2))
