# A/B of the fused dW + update variants and the backward schedule (development library)
mkdir -p gpurun_out/dwv
timeout 300 python tools/gemm_error.py > gpurun_out/dwv/gemm_error.txt 2>&1

export ST_LIB_PATH=paper_1809_02839_b200/_var/dev/libspectrain.so
for d in 0 1; do
  ST_DW_DIRECT=$d timeout 300 python - > gpurun_out/dwv/ops_direct$d.txt 2>&1 <<'PY'
import sys; sys.path.insert(0, '.')
from tools.time_gemm import t_op
for (i, o) in [(8192, 8192), (16384, 16384), (16384, 4096)]:
    us, tf, gbs = t_op(3, 0, 128, i, o, reps=10)
    print(f"dWU {i}x{o}: {us:9.1f} us  {gbs:7.1f} GB/s (16 B/param)")
PY
done
for w in large_fcn wide_fcn; do
  for ser in 0 1; do
    for d in 0 1; do
      ST_BWD_SERIAL=$ser ST_DW_DIRECT=$d timeout 400 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/dwv/${w}_ser${ser}_dir${d}.json 2> gpurun_out/dwv/${w}_ser${ser}_dir${d}.err
    done
  done
done
