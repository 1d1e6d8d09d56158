mkdir -p gpurun_out/tssa
timeout 300 python tools/dbg_kernels.py > gpurun_out/tssa/k0.txt 2>&1
ST_TS_SPLIT_ACC=1 timeout 300 python tools/dbg_kernels.py > gpurun_out/tssa/k1.txt 2>&1
ST_TS_SPLIT_ACC=1 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py tests/test_gpu_fullsize.py -q -x > gpurun_out/tssa/pytest.log 2>&1; echo "exit $?" >> gpurun_out/tssa/pytest.log
ST_TS_SPLIT_ACC=1 M=2 timeout 600 python tools/fullsize_debug.py > gpurun_out/tssa/fs1.txt 2>&1
for i in 1 2; do
timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/tssa/b0_$i.json 2>/dev/null
ST_TS_SPLIT_ACC=1 timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/tssa/b1_$i.json 2>/dev/null
done
