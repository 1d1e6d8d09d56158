# Every workload on one GPU (N=1 and co-located stage counts), JSON lines into gpurun_out/r1bench/
mkdir -p gpurun_out/r1bench
for w in wide_fcn lstm_lm vgg16 mlp deep_mlp; do
  timeout 300 python bench.py --workload $w --no-cpu > gpurun_out/r1bench/$w.json 2> gpurun_out/r1bench/$w.err
done
for s in 2 4 8; do
  timeout 300 python bench.py --workload wide_fcn --stages $s --no-cpu > gpurun_out/r1bench/wide_fcn_s$s.json 2>&1
done
timeout 300 python bench.py --workload lstm_lm --stages 4 --no-cpu > gpurun_out/r1bench/lstm_lm_s4.json 2>&1
timeout 300 python bench.py --workload vgg16 --stages 8 --no-cpu > gpurun_out/r1bench/vgg16_s8.json 2>&1
timeout 600 python bench.py --workload large_fcn --no-cpu --steps 10 --warmup 3 > gpurun_out/r1bench/large_fcn.json 2>&1
for s in 2 4 8; do
  timeout 600 python bench.py --workload large_fcn --stages $s --no-cpu --steps 10 --warmup 3 > gpurun_out/r1bench/large_fcn_s$s.json 2>&1
done
