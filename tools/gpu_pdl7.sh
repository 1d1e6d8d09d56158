mkdir -p gpurun_out/pdl7
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pdl7/pytest.log 2>&1; echo "exit $?" >> gpurun_out/pdl7/pytest.log
for w in mlp deep_mlp wide_fcn; do timeout 300 python bench.py --workload $w --no-cpu --no-e2e > gpurun_out/pdl7/$w.json 2>/dev/null; done
timeout 600 python bench.py --workload large_fcn --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/pdl7/large.json 2>/dev/null
