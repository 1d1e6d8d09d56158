# dX mask prefetch: standalone fwd / dX at 16384² and 8192² (x3), GEMM parity tests, large-FCN bench
mkdir -p gpurun_out/r2dxpf
for r in 1 2 3; do for s in 128,16384,16384 128,8192,8192; do timeout 300 python tools/time_gemm.py --shape $s 2>&1 | grep -E "^(fwd|dX)" >> gpurun_out/r2dxpf/time.txt; done; done
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py -q --timeout=600 > gpurun_out/r2dxpf/pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2dxpf/pytest.log
timeout 600 python bench.py --no-cpu --no-e2e --steps 30 > gpurun_out/r2dxpf/large_fcn.json 2>&1
