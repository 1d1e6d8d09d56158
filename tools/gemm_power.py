"""Development: SM clock / power / throttle reasons (NVML) during ~3 s of back-to-back
FP32X3 GEMMs: python tools/gemm_power.py op B in out"""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, pynvml
import paper_1809_02839_b200 as st
op, B, n_in, n_out = (int(a) for a in sys.argv[1:5])
dev = torch.device("cuda", 0)
X = torch.randn(B, n_in, device=dev); W = torch.randn(n_in, n_out, device=dev) * 0.01
dZ = torch.randn(B, n_out, device=dev); bias = torch.randn(n_out, device=dev)
work = torch.zeros(int(st._lib.lib.st_gemm_workspace_bytes(B, n_in, n_out)), dtype=torch.uint8, device=dev)
if op == 3:  # fused dW + K-B update
    Wb = torch.randn(n_in * n_out + n_out, device=dev) * 0.01
    Vb = torch.zeros_like(Wb); Gs = torch.empty_like(Wb)
    f = lambda: st.dw_update_raw(0, X, dZ, Wb, Vb, None, None, 1e-3, 0.9, 0, 0, work=work, G_scratch=Gs)
else:
    args = (X, W, bias, None, torch.empty(B, n_out, device=dev)) if op == 0 else (dZ, W, X, None, torch.empty(B, n_in, device=dev))
    f = lambda: st.gemm_raw(op, 0, B, n_in, n_out, *args, relu=(op == 0), work=work)
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples, stop = [], False
def sampler():
    while not stop:
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
        time.sleep(0.02)
for _ in range(200): f()
torch.cuda.synchronize()
th = threading.Thread(target=sampler); th.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 0; t0 = time.time(); e0.record()
while time.time() - t0 < 3.0:
    for _ in range(100): f()
    n += 100
    torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize(); stop = True; th.join()
s = np.array([(a, b) for a, b, _ in samples]); reasons = set(r for _, _, r in samples)
print(f"op {op}: {e0.elapsed_time(e1) * 1e3 / n:.1f} us/GEMM; SM MHz median {np.median(s[:,0]):.0f} min {s[:,0].min():.0f};"
      f" power W median {np.median(s[:,1]):.0f} max {s[:,1].max():.0f}; throttle reasons {sorted(hex(r) for r in reasons)}")
