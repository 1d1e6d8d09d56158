mkdir -p gpurun_out/q2
timeout 600 python -m pytest tests/test_gpu_pipeline.py -q -x > gpurun_out/q2/pytest.log 2>&1; echo "exit $?" >> gpurun_out/q2/pytest.log
for i in 1 2; do timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/q2/b$i.json 2>/dev/null; done
timeout 600 python bench.py --workload large_fcn --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/q2/large.json 2>/dev/null
