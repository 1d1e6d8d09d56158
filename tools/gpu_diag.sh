# Diagnostics call: kernel timelines (real concurrency), standalone per-op times, ncu metric names
mkdir -p gpurun_out/diag
timeout 300 python tools/timeline.py --workload large_fcn --M 2 > gpurun_out/diag/tl_large.txt 2>&1
timeout 300 python tools/timeline.py --workload wide_fcn --M 3 > gpurun_out/diag/tl_wide.txt 2>&1
timeout 300 python - > gpurun_out/diag/ops.txt 2>&1 <<'PY'
import sys; sys.path.insert(0, '.')
from tools.time_gemm import t_op
for (i, o) in [(8192, 8192), (16384, 16384)]:
    for op, name in ((0, "fwd"), (1, "dX"), (3, "dWU")):
        us, tf, gbs = t_op(op, 0, 128, i, o)
        print(f"{name} {i}x{o}: {us:9.1f} us {tf:7.1f} TF/s  {gbs:7.1f} GB/s(4B)  {gbs*4:7.1f} GB/s(16B)")
PY
ncu --query-metrics --chip gb100 > gpurun_out/diag/ncu_metrics_all.txt 2>&1 || ncu --query-metrics > gpurun_out/diag/ncu_metrics_all.txt 2>&1
grep -i -E "tensor|utc|tmem|tcgen|mma" gpurun_out/diag/ncu_metrics_all.txt > gpurun_out/diag/ncu_metrics_tensor.txt
nvidia-smi -q | grep -i -E "clocks|power" -A2 | head -60 > gpurun_out/diag/smi_q.txt
