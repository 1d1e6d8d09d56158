# ncu --set full with source of one 16384² CTA-pair dX launch (and one forward), warp stalls per source line
mkdir -p gpurun_out/r2dxs
cat > /tmp/one_op.py <<'PY'
import sys; sys.path.insert(0, '.')
from tools.time_gemm import t_op
t_op(int(sys.argv[1]), 0, 128, 16384, 16384, reps=1)
PY
for op in 1 0; do
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:ts2 -s 1 -c 1 \
    -o gpurun_out/r2dxs/op$op python /tmp/one_op.py $op > gpurun_out/r2dxs/op$op.log 2>&1
  python tools/ncu_lines.py gpurun_out/r2dxs/op$op.ncu-rep 40 > gpurun_out/r2dxs/op${op}_lines.txt 2>&1
  python tools/summarize_ncu.py full gpurun_out/r2dxs/op$op.ncu-rep > gpurun_out/r2dxs/op${op}_full.txt 2>&1
  rm -f gpurun_out/r2dxs/op$op.ncu-rep
done
