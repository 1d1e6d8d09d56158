# LSTM: parity tests + LM bench + launch list
mkdir -p gpurun_out/lstm
timeout 600 python -m pytest tests/test_gpu_lstm.py -x -q > gpurun_out/lstm/pytest.log 2>&1; echo "exit $?" >> gpurun_out/lstm/pytest.log
timeout 300 python bench.py --workload lstm_lm --no-cpu --no-e2e > gpurun_out/lstm/lm.json 2> gpurun_out/lstm/lm.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lstm/launches.csv python bench.py --workload lstm_lm --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
python tools/summarize_ncu.py launches gpurun_out/lstm/launches.csv > gpurun_out/lstm/summary.csv
