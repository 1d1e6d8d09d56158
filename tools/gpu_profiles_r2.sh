# Round-2 profiles (profiles/r2_*): large-FCN launch list, in-step ncu --set full of the fused
# dW + update, standalone dW + update DRAM bytes / duration at 8192² and 16384²
mkdir -p gpurun_out/p2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p2/launches_large_fcn.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/p2/launches_large_fcn.log 2>&1
python tools/summarize_ncu.py launches gpurun_out/p2/launches_large_fcn.csv > gpurun_out/p2/launches_large_fcn_summary.csv
# in-step: the dW + update launches of the first timed step (skip the warm-up's 3 x 16)
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'tc_dw_kernel' \
    -s 48 -c 4 -o gpurun_out/p2/dwu_instep python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/p2/dwu_instep.log 2>&1
ncu -i gpurun_out/p2/dwu_instep.ncu-rep --page raw --csv > gpurun_out/p2/dwu_instep_raw.csv 2>/dev/null
python tools/summarize_ncu.py full gpurun_out/p2/dwu_instep.ncu-rep > gpurun_out/p2/dwu_instep_full.txt 2>&1
rm -f gpurun_out/p2/dwu_instep.ncu-rep
cat > /tmp/dwu_sa.py <<'PY'
import sys; sys.path.insert(0, '.')
from tools.time_gemm import t_op
for (i, o) in [(8192, 8192), (16384, 16384)]:
    t_op(3, 0, 128, i, o, reps=1)
PY
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:tc_dw_kernel --csv python /tmp/dwu_sa.py > gpurun_out/p2/dwu_standalone.csv 2> gpurun_out/p2/dwu_standalone.err
