# Large FCN: overlapped dX(l-1) || dW+update(l) for the 16384² layers at several SM splits (dev build)
TAG=${TAG:-r2split}; mkdir -p gpurun_out/$TAG
DEV=paper_1809_02839_b200/_var/dev/libspectrain.so
timeout 300 python bench.py --no-cpu --no-e2e --steps 20 --warmup 3 > gpurun_out/$TAG/serial.json 2>&1
for s in 48 64 74 88 104; do
  ST_LIB_PATH=$DEV ST_BWD_SERIAL=0 ST_DWU_SMS=$s timeout 300 python bench.py --no-cpu --no-e2e --steps 20 --warmup 3 > gpurun_out/$TAG/ov_$s.json 2>&1
done
ST_LIB_PATH=$DEV timeout 300 python bench.py --no-cpu --no-e2e --steps 20 --warmup 3 > gpurun_out/$TAG/serial_dev.json 2>&1
