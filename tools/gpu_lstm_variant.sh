mkdir -p gpurun_out/r2lstmB
timeout 1200 python -m pytest tests/test_gpu_lstm.py tests/test_gpu_variants.py -k "lstm" -q --timeout=900 > gpurun_out/r2lstmB/pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2lstmB/pytest.log
