"""Time the stage GEMMs through st_gemm_raw (CUDA events, warm) — development tool."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1809_02839_b200 as st

def t_op(op, mode, B, n_in, n_out, reps=10):
    dev = torch.device("cuda", 0)
    X = torch.randn(B, n_in, device=dev)
    W = torch.randn(n_in, n_out, device=dev) * 0.01
    dZ = torch.randn(B, n_out, device=dev)
    bias = torch.randn(n_out, device=dev)
    work = torch.zeros(int(st._lib.lib.st_gemm_workspace_bytes(B, n_in, n_out)), dtype=torch.uint8, device=dev)
    if op == 3:
        Wb = torch.randn(n_in * n_out + n_out, device=dev) * 0.01
        Vb = torch.zeros_like(Wb)
        Gs = torch.empty_like(Wb)
        f = lambda: st.dw_update_raw(mode, X, dZ, Wb, Vb, None, None, 1e-3, 0.9, 0, 0, work=work, G_scratch=Gs)
        f(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(50_000_000)
        e0.record()
        for _ in range(reps): f()
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / reps
        return us, 2.0 * B * n_in * n_out / us / 1e6, 16.0 * n_in * n_out / us / 1e3
    if op == 0: args = (X, W, bias, None, torch.empty(B, n_out, device=dev))
    elif op == 1: args = (dZ, W, X, None, torch.empty(B, n_in, device=dev))
    else: args = (X, dZ, None, torch.empty(n_out, device=dev), torch.empty(n_in, n_out, device=dev))
    f = lambda: st.gemm_raw(op, mode, B, n_in, n_out, *args, relu=(op == 0), work=work)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(50_000_000)  # let the host enqueue every rep before the GPU starts: pure device time
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    flops = 2.0 * B * n_in * n_out
    byts = 4.0 * n_in * n_out
    return us, flops / us / 1e6, byts / us / 1e3

if __name__ == "__main__":
    shapes = [(128, 8192, 8192)] + ([(128, 784, 8192), (128, 8192, 10)] if "--all" in sys.argv else [])
    modes = ((0, "fp32x3"), (1, "tf32"))
    if "--shape" in sys.argv:  # --shape B,in,out: fp32x3 only
        shapes = [tuple(int(v) for v in sys.argv[sys.argv.index("--shape") + 1].split(","))]
        modes = ((0, "fp32x3"),)
    for (B, i, o) in shapes:
        for mode, mname in modes:
            for op, oname in ((0, "fwd"), (1, "dX"), (2, "dW"), (3, "dWU")):
                us, tf, gbs = t_op(op, mode, B, i, o)
                print(f"{oname:3s} {mname:6s} B={B} in={i} out={o}: {us:8.1f} us  {tf:7.1f} TFLOP/s  weight-bytes {gbs:7.1f} GB/s")
