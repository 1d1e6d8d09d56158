# How much of the fwd / dX / dW(+update) time is tensor work? (development experiment)
# flags 256 = drop one of the three 3xTF32 MMAs (timing only, numerics wrong)
mkdir -p gpurun_out/exp
for f in 0 256; do
  ST_GEMM_DEV_FLAGS=$f python tools/time_gemm.py --all > gpurun_out/exp/time_gemm_f$f.txt 2>&1
  ST_GEMM_PAIR=1 ST_GEMM_DEV_FLAGS=$f python tools/time_gemm.py > gpurun_out/exp/time_gemm_pair_f$f.txt 2>&1
  ST_GEMM_DEV_FLAGS=$f timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/exp/bench_f$f.json 2>&1
done
timeout 300 python bench.py --no-cpu --no-e2e --gemm tf32 > gpurun_out/exp/bench_tf32.json 2>&1
timeout 300 python bench.py --no-cpu > gpurun_out/exp/bench_default.json 2>&1
