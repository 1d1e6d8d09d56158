"""cuBLAS reference timings for the stage GEMM shapes (development context only)."""
import torch
dev = torch.device("cuda", 0)
def t(f, reps=20):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps
B, n = 128, 8192
X = torch.randn(B, n, device=dev); W = torch.randn(n, n, device=dev); dZ = torch.randn(B, n, device=dev)
for tf32 in (True, False):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    print(f"tf32={tf32}: fwd X@W {t(lambda: X @ W):7.1f} us | dX dZ@W.T {t(lambda: dZ @ W.T):7.1f} us | dW X.T@dZ {t(lambda: X.T @ dZ):7.1f} us")
Wb = W.bfloat16(); Xb = X.bfloat16()
print(f"bf16 fwd {t(lambda: Xb @ Wb):7.1f} us")
G = torch.empty(n, n, device=dev)
print(f"copy 268MB (W->G) {t(lambda: G.copy_(W)):7.1f} us")
