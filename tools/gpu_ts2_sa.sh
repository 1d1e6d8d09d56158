# CTA-pair fwd / dX with one accumulator (dev ST_TS_SPLIT_ACC=0: 6 TMEM A slots of look-ahead instead of 4)
mkdir -p gpurun_out/r2sa
DEV=paper_1809_02839_b200/_var/dev/libspectrain.so
for r in 1 2; do for v in 1 0; do
  echo "SPLIT_ACC=$v" >> gpurun_out/r2sa/time.txt
  for s in 128,16384,16384 128,8192,8192; do
    ST_LIB_PATH=$DEV ST_TS_SPLIT_ACC=$v timeout 300 python tools/time_gemm.py --shape $s 2>&1 | grep -E "^(fwd|dX)" >> gpurun_out/r2sa/time.txt
  done
done; done
for v in 1 0; do ST_LIB_PATH=$DEV ST_TS_SPLIT_ACC=$v timeout 600 python bench.py --no-cpu --no-e2e --steps 30 > gpurun_out/r2sa/large_fcn_sa$v.json 2>&1; done
