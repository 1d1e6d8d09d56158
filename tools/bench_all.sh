mkdir -p gpurun_out/r1bench
for w in wide_fcn lstm_lm vgg16 mlp deep_mlp; do
  timeout 300 python bench.py --workload $w --no-cpu > gpurun_out/r1bench/$w.json 2> gpurun_out/r1bench/$w.err
done
timeout 300 python bench.py --workload wide_fcn --stages 8 --no-cpu > gpurun_out/r1bench/wide_fcn_s8.json 2>&1
timeout 300 python bench.py --workload wide_fcn --stages 4 --no-cpu > gpurun_out/r1bench/wide_fcn_s4.json 2>&1
timeout 300 python bench.py --workload lstm_lm --stages 4 --no-cpu > gpurun_out/r1bench/lstm_lm_s4.json 2>&1
timeout 300 python bench.py --workload vgg16 --stages 8 --no-cpu > gpurun_out/r1bench/vgg16_s8.json 2>&1
timeout 600 python bench.py --workload large_fcn --no-cpu --steps 5 --warmup 3 > gpurun_out/r1bench/large_fcn.json 2>&1
