mkdir -p gpurun_out/pdl6
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pdl6/pytest.log 2>&1; echo "exit $?" >> gpurun_out/pdl6/pytest.log
timeout 600 python bench.py --workload large_fcn --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/pdl6/large.json 2>/dev/null
timeout 300 python bench.py --stages 2 --no-cpu --no-e2e > gpurun_out/pdl6/wide2.json 2>/dev/null
for i in 1 2; do timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/pdl6/wide1_$i.json 2>/dev/null; done
for w in vgg16 lstm_lm mlp deep_mlp; do timeout 300 python bench.py --workload $w --no-cpu --no-e2e > gpurun_out/pdl6/$w.json 2>/dev/null; done
