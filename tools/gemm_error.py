"""Pre-activation error of the forward GEMM at the large-FCN shape (128 × 16384 × 16384)
against fp64, and how many ReLU decisions it flips — library 3xTF32 vs a plain fp32
CUDA-core GEMM (torch, TF32 off) (reading D24 diagnostics)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1809_02839_b200 as st

torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev); g.manual_seed(7)
for (B, n_in, n_out) in [(128, 16384, 16384), (128, 8192, 8192), (128, 4096, 4096)]:
    A = torch.relu(torch.randn(B, n_in, device=dev, generator=g))
    r = (6.0 / (n_in + n_out)) ** 0.5
    W = (torch.rand(n_in, n_out, device=dev, generator=g) * 2 - 1) * r
    bias = torch.zeros(n_out, device=dev)
    work = torch.zeros(int(st._lib.lib.st_gemm_workspace_bytes(B, n_in, n_out)), dtype=torch.uint8, device=dev)
    Z = torch.empty(B, n_out, device=dev)
    st.gemm_raw(0, 0, B, n_in, n_out, A, W, bias, None, Z, relu=False, work=work)
    torch.cuda.synchronize()
    Z64 = A.double() @ W.double()
    Z32 = A @ W
    scale = Z64.pow(2).mean().sqrt()
    for name, Zx in (("3xTF32 (library)", Z), ("fp32 (torch, TF32 off)", Z32)):
        e = (Zx.double() - Z64) / scale
        flips = int(((Zx > 0) != (Z64 > 0)).sum())
        print(f"{B}x{n_in}x{n_out} {name:24s}: err rms {e.pow(2).mean().sqrt().item():.3e} max {e.abs().max().item():.3e}"
              f"  ReLU decisions differing {flips} of {Z.numel()}")
