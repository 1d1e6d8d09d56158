"""Development: max error / scale of the stage GEMMs and the fused dW + update at large shapes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1809_02839_b200 as st
dev = torch.device("cuda", 0)
def rep(name, got, ref, scale):
    e = (got.double() - ref).abs() / (scale + 1e-30)
    r = ((got.double() - ref).norm() / ref.norm()).item()
    print(f"{name}: max err/scale {e.max().item():.3e}  relL2 {r:.3e}")
SHAPES = [(128, 2048, 2048), (128, 8192, 8192), (128, 784, 8192), (128, 8192, 784), (128, 4096, 4096)]
if os.environ.get('TALL'): SHAPES = [(8192, 1024, 1024), (32768, 512, 512), (4480, 1500, 6000)]
for (B, i, o) in SHAPES:
    g = torch.Generator(device=dev); g.manual_seed(0)
    X = torch.randn(B, i, device=dev, generator=g).relu()
    W = torch.randn(i, o, device=dev, generator=g) / i ** 0.5
    b = torch.randn(o, device=dev, generator=g)
    dZ = torch.randn(B, o, device=dev, generator=g) / B
    work = torch.zeros(int(st._lib.lib.st_gemm_workspace_bytes(B, i, o)), dtype=torch.uint8, device=dev)
    Z = torch.empty(B, o, device=dev)
    st.gemm_raw(0, 0, B, i, o, X, W, b, None, Z, relu=False, work=work)
    ref = X.double() @ W.double() + b.double()
    rep(f"fwd {B}x{i}x{o}", Z, ref, X.double().abs() @ W.double().abs() + b.double().abs())
    D = torch.empty(B, i, device=dev)
    st.gemm_raw(1, 0, B, i, o, dZ, W, None, None, D, work=work)
    ref = dZ.double() @ W.double().T
    rep(f"dX  {B}x{i}x{o}", D, ref, dZ.double().abs() @ W.double().abs().T)
    G = torch.empty(i, o, device=dev); gb = torch.empty(o, device=dev)
    st.gemm_raw(2, 0, B, i, o, X, dZ, None, gb, G, work=work)
    ref = X.double().T @ dZ.double()
    rep(f"dW  {B}x{i}x{o}", G, ref, X.double().abs().T @ dZ.double().abs())
    if os.environ.get('TALL'): continue
    P = i * o + o
    Wb = torch.randn(P, device=dev, generator=g) * 0.01
    Vb = torch.zeros(P, device=dev)
    Gs = torch.empty(P, device=dev)
    st.dw_update_raw(0, X, dZ, Wb, Vb, None, None, 0.01, 0.9, 0, 0, work=work, G_scratch=Gs)
    gref = torch.cat([(X.double().T @ dZ.double()).reshape(-1), dZ.double().sum(0)])
    sc = torch.cat([(X.double().abs().T @ dZ.double().abs()).reshape(-1), dZ.double().abs().sum(0)])
    rep(f"dWU V {B}x{i}x{o}", Vb, 0.1 * gref, 0.1 * sc)
    torch.cuda.synchronize()
