# Persistent LSTM recurrence (development variant, k_lstm_rec.cu): LSTM parity in the product
# build and with ST_LSTM_PERSIST=1 (tests/test_gpu_variants.py), the per-step phase timeline
# (dev build, ST_LSTM_DBG=1 fwd / 2 bwd), the LM bench and the per-layer profile of both paths.
TAG=${TAG:-r2lstm}; mkdir -p gpurun_out/$TAG
DEV=paper_1809_02839_b200/_var/dev/libspectrain.so
timeout 1200 python -m pytest tests/test_gpu_lstm.py tests/test_gpu_variants.py -k lstm -q --timeout=900 > gpurun_out/$TAG/pytest_lstm.log 2>&1; echo "exit $?" >> gpurun_out/$TAG/pytest_lstm.log
for d in 1 2; do ST_LIB_PATH=$DEV ST_LSTM_DBG=$d ST_LSTM_PERSIST=1 timeout 300 python tools/lstm_rec_timeline.py > gpurun_out/$TAG/timeline_$d.json 2>&1; done
timeout 300 python bench.py --workload lstm_lm --no-cpu --steps 20 > gpurun_out/$TAG/lstm_lm.json 2>&1
ST_LIB_PATH=$DEV ST_LSTM_PERSIST=1 timeout 300 python bench.py --workload lstm_lm --no-cpu --steps 20 > gpurun_out/$TAG/lstm_lm_persistent.json 2>&1
timeout 300 python tools/layer_prof.py lstm_lm > gpurun_out/$TAG/lstm_prof.jsonl 2>&1
ST_LIB_PATH=$DEV ST_LSTM_PERSIST=1 timeout 300 python tools/layer_prof.py lstm_lm > gpurun_out/$TAG/lstm_prof_persistent.jsonl 2>&1
timeout 300 python tools/layer_prof.py vgg16 > gpurun_out/$TAG/vgg16_prof.jsonl 2>&1
