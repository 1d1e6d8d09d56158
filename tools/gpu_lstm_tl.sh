TAG=${TAG:-r2lstm3}; mkdir -p gpurun_out/$TAG
DEV=paper_1809_02839_b200/_var/dev/libspectrain.so
for d in ${DIRS:-1 2}; do ST_LIB_PATH=$DEV ST_LSTM_DBG=$d timeout 300 python tools/lstm_rec_timeline.py > gpurun_out/$TAG/timeline_$d.json 2>&1; done
