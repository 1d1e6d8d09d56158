mkdir -p gpurun_out/dp
timeout 600 python -m pytest tests/test_gpu_dp.py tests/test_gpu_kernels.py -x -q > gpurun_out/dp/pytest.log 2>&1; echo "exit $?" >> gpurun_out/dp/pytest.log
timeout 300 python bench.py --parallel dp --steps 30 --warmup 3 > gpurun_out/dp/dp1.json 2> gpurun_out/dp/dp1.err
timeout 300 python bench.py > gpurun_out/dp/pp1.json 2> gpurun_out/dp/pp1.err
