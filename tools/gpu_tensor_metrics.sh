# Tensor-pipe evidence for the tcgen05 GEMMs (which counters see UTCHMMA work on sm_100)
mkdir -p gpurun_out/tm
cat > /tmp/tm_ops.py <<'PY'
import sys; sys.path.insert(0, '.')
from tools.time_gemm import t_op
for op in (0, 1, 3):
    t_op(op, 0, 128, 8192, 8192, reps=1)
PY
M1=gpu__time_duration.sum,sm__ops_path_tensor_src_tf32_dst_fp32.sum,sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32.sum,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_src_tf32_dst_fp32.sum.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_src_tf32_dst_fp32.sum.peak_sustained,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M1 --clock-control none -k regex:tc_ --csv python /tmp/tm_ops.py > gpurun_out/tm/gemm_8192.csv 2> gpurun_out/tm/gemm_8192.err
timeout 600 ncu --metrics $M1 --clock-control none -k regex:tc_tsg -s 30 -c 12 --csv python bench.py --workload vgg16 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/tm/vgg.csv 2> gpurun_out/tm/vgg.err
timeout 600 ncu --metrics $M1 --clock-control none -k regex:tc_ -s 40 -c 12 --csv python bench.py --workload lstm_lm --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/tm/lstm.csv 2> gpurun_out/tm/lstm.err
