# Development: time fwd / dX of each ring-depth variant under paper_1809_02839_b200/_var
mkdir -p gpurun_out/exp
for v in "" paper_1809_02839_b200/_var/*.so; do
  for F in ${FLAGS:-0 31}; do
    echo "$(basename ${v:-default}) FLAGS=$F $(ST_LIB_PATH=$v ST_GEMM_DEV_FLAGS=$F timeout 60 python tools/time_gemm.py 2>&1 | grep fp32x3 | grep -E '^(fwd|dX |dWU)' | awk '{print $1, $6}' | tr '\n' ' ')"
  done
done
