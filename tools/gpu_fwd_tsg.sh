# tall dense forward on the persistent TMEM-A kernel (dev ST_FWD_TSG=1) vs the CTA-pair kernel: parity + LM timing
TAG=${TAG:-r2ft}; mkdir -p gpurun_out/$TAG
DEV=paper_1809_02839_b200/_var/dev/libspectrain.so
ST_LIB_PATH=$DEV ST_FWD_TSG=1 timeout 900 python -m pytest tests/test_gpu_lstm.py tests/test_gpu_kernels.py -q -x --timeout=600 > gpurun_out/$TAG/pytest.log 2>&1; echo "exit $?" >> gpurun_out/$TAG/pytest.log
ST_LIB_PATH=$DEV ST_FWD_TSG=1 timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -k "lstm_lm_full_size_single" --timeout=600 >> gpurun_out/$TAG/pytest.log 2>&1; echo "exit $?" >> gpurun_out/$TAG/pytest.log
for r in 1 2; do for v in 0 1; do
  ST_LIB_PATH=$DEV ST_FWD_TSG=$v timeout 300 python bench.py --workload lstm_lm --no-cpu --no-e2e --steps 30 > gpurun_out/$TAG/lstm_t${v}_r$r.json 2>&1
done; done
ST_LIB_PATH=$DEV ST_FWD_TSG=1 timeout 300 python tools/layer_prof.py lstm_lm > gpurun_out/$TAG/lstm_prof_t1.jsonl 2>&1
