mkdir -p gpurun_out/pdl4
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pdl4/pytest.log 2>&1; echo "exit $?" >> gpurun_out/pdl4/pytest.log
for w in mlp deep_mlp wide_fcn lstm_lm vgg16; do timeout 300 python bench.py --workload $w --no-cpu --no-e2e > gpurun_out/pdl4/$w.json 2>/dev/null; done
