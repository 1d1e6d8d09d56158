# persistent LSTM recurrence per direction (dev build): ST_LSTM_PERSIST 0 (per-step path) / 1 (both) / 2 (bwd) / 3 (fwd)
TAG=${TAG:-r2lpm}; mkdir -p gpurun_out/$TAG
DEV=paper_1809_02839_b200/_var/dev/libspectrain.so
for d in 1 2; do ST_LIB_PATH=$DEV ST_LSTM_DBG=$d ST_LSTM_PERSIST=1 timeout 300 python tools/lstm_rec_timeline.py > gpurun_out/$TAG/timeline_$d.json 2>&1; done
for r in 1 2; do for v in 0 1 2 3; do
  ST_LIB_PATH=$DEV ST_LSTM_PERSIST=$v timeout 300 python bench.py --workload lstm_lm --no-cpu --no-e2e --steps 30 > gpurun_out/$TAG/bench_p${v}_r$r.json 2>&1
done; done
