# persistent LSTM recurrence: parity tests (LSTM, full size, P2P / NCCL / graph sessions), sanitizer,
# LM bench and per-layer profile
TAG=${TAG:-r2lstm}; mkdir -p gpurun_out/$TAG
timeout 1200 python -m pytest tests/test_gpu_lstm.py tests/test_gpu_variants.py -k "lstm" -q --timeout=300 > gpurun_out/$TAG/pytest_lstm.log 2>&1; echo "exit $?" >> gpurun_out/$TAG/pytest_lstm.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -k lstm --timeout=300 > gpurun_out/$TAG/pytest_full_lstm.log 2>&1; echo "exit $?" >> gpurun_out/$TAG/pytest_full_lstm.log
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 3 python -m pytest tests/test_gpu_lstm.py -q -k "persistent and 100" > gpurun_out/$TAG/memcheck.log 2>&1; echo "exit $?" >> gpurun_out/$TAG/memcheck.log
timeout 600 compute-sanitizer --tool racecheck --error-exitcode 3 python -m pytest tests/test_gpu_lstm.py -q -k "persistent and 100" > gpurun_out/$TAG/racecheck.log 2>&1; echo "exit $?" >> gpurun_out/$TAG/racecheck.log
timeout 300 python bench.py --workload lstm_lm --no-cpu --steps 20 > gpurun_out/$TAG/lstm_lm.json 2>&1
timeout 300 python bench.py --workload lstm_lm --no-cpu --steps 20 --stages 4 > gpurun_out/$TAG/lstm_lm_s4.json 2>&1
timeout 300 python tools/layer_prof.py lstm_lm > gpurun_out/$TAG/lstm_prof.jsonl 2>&1
