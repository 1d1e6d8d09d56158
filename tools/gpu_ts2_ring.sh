# CTA-pair fwd / dX GEMM with deeper weight rings (build variants ST_TS_RA = 6 / 8 / 10)
mkdir -p gpurun_out/r2ring
for v in dev ra8 ra10 dev ra8 ra10; do
  echo "VARIANT=$v" >> gpurun_out/r2ring/time.txt
  for s in 128,16384,16384 128,8192,8192; do
    ST_LIB_PATH=paper_1809_02839_b200/_var/$v/libspectrain.so timeout 300 python tools/time_gemm.py --shape $s 2>&1 | grep -E "^(fwd|dX)" >> gpurun_out/r2ring/time.txt
  done
done
