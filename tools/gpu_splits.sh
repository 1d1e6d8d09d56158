mkdir -p gpurun_out/sp
export ST_LIB_PATH=paper_1809_02839_b200/_var/dev/libspectrain.so
for f in 1 2 4 8 16; do
  ST_FORCE_SPLITS=$f timeout 300 python tools/gemm_error.py > gpurun_out/sp/err_splits$f.txt 2>&1
done
