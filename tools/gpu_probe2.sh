mkdir -p gpurun_out/r2probe
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe2 tools/probe_mma_rate2.cu && timeout 120 /tmp/probe2 > gpurun_out/r2probe/probe2.txt 2>&1
nvidia-smi --query-gpu=clocks.sm --format=csv >> gpurun_out/r2probe/probe2.txt
