mkdir -p gpurun_out/r2ce
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_lstm.py tests/test_gpu_pipeline.py -q --timeout=600 > gpurun_out/r2ce/pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2ce/pytest.log
for r in 1 2; do timeout 300 python bench.py --workload lstm_lm --no-cpu --steps 30 > gpurun_out/r2ce/lstm_lm_r$r.json 2>&1; done
timeout 300 python tools/layer_prof.py lstm_lm > gpurun_out/r2ce/lstm_prof.jsonl 2>&1
