# ncu --set full with source of one standalone 16384² fused dW + update launch: warp stalls per source line
mkdir -p gpurun_out/r2dwus
cat > /tmp/one_dwu.py <<'PY'
import sys; sys.path.insert(0, '.')
from tools.time_gemm import t_op
t_op(3, 0, 128, 16384, 16384, reps=1)
PY
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:tc_dw_kernel -s 1 -c 1 \
  -o gpurun_out/r2dwus/dwu python /tmp/one_dwu.py > gpurun_out/r2dwus/dwu.log 2>&1
python tools/ncu_lines.py gpurun_out/r2dwus/dwu.ncu-rep 45 > gpurun_out/r2dwus/dwu_lines.txt 2>&1
python tools/summarize_ncu.py full gpurun_out/r2dwus/dwu.ncu-rep > gpurun_out/r2dwus/dwu_full.txt 2>&1
ncu -i gpurun_out/r2dwus/dwu.ncu-rep --page details --csv > gpurun_out/r2dwus/dwu_details.csv 2>/dev/null
rm -f gpurun_out/r2dwus/dwu.ncu-rep
