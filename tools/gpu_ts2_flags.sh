# CTA-pair fwd / dX GEMM (8192² and 16384²) with parts switched off (dev ST_GEMM_DEV_FLAGS, timing only):
# 1 no MMAs, 2 no converter math, 16 no TMEM stores, 32 no wait::st, 8 no A loads, 256 drop one of the 3 MMAs
mkdir -p gpurun_out/r2flags
DEV=paper_1809_02839_b200/_var/dev/libspectrain.so
for f in 0 1 2 16 32 48 8 256; do
  echo "FLAGS=$f" >> gpurun_out/r2flags/time.txt
  for s in 128,16384,16384 128,8192,8192; do
    ST_LIB_PATH=$DEV ST_GEMM_DEV_FLAGS=$f timeout 300 python tools/time_gemm.py --shape $s 2>&1 | grep -E "^(fwd|dX)" >> gpurun_out/r2flags/time.txt
  done
done
