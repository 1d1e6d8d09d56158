mkdir -p gpurun_out/rmse
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k prediction_error > gpurun_out/rmse/pytest.log 2>&1; echo "exit $?" >> gpurun_out/rmse/pytest.log
timeout 900 python tools/rmse_fig7.py --out gpurun_out/rmse/r1_fig7_rmse.json > gpurun_out/rmse/run.log 2>&1
