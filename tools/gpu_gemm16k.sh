# fwd / dX / dW+update of one 16384² and one 8192² layer standalone (CUDA events), and ncu
# DRAM / L2 / tensor-pipe metrics of the 16384² fwd and dX CTA-pair kernels
TAG=${TAG:-r2g16}; mkdir -p gpurun_out/$TAG
for s in ${SHAPES:-128,16384,16384 128,8192,8192}; do timeout 300 python tools/time_gemm.py --shape $s >> gpurun_out/$TAG/time.txt 2>&1; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,dram__sectors_read.sum
timeout 600 ncu --clock-control none --kernel-name-base demangled -k regex:ts2 -s 12 -c 2 --metrics $M \
  --csv python tools/time_gemm.py --shape 128,16384,16384 > gpurun_out/$TAG/ncu_dx.csv 2>&1
timeout 600 ncu --clock-control none --kernel-name-base demangled -k regex:ts2 -s 2 -c 2 --metrics $M \
  --csv python tools/time_gemm.py --shape 128,16384,16384 > gpurun_out/$TAG/ncu_fwd.csv 2>&1
