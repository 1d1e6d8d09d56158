mkdir -p gpurun_out/pdl
timeout 600 python -m pytest tests/test_gpu_lstm.py tests/test_gpu_fullsize.py -k "lstm" -q -x > gpurun_out/pdl/pytest.log 2>&1; echo "exit $?" >> gpurun_out/pdl/pytest.log
for p in 1 0; do for i in 1 2; do ST_PDL=$p timeout 300 python bench.py --workload lstm_lm --no-cpu --no-e2e > gpurun_out/pdl/lstm_${p}_$i.json 2>/dev/null; done; done
