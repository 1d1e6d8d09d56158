mkdir -p gpurun_out/pdl2
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_kernels.py tests/test_gpu_fullsize.py -q -x > gpurun_out/pdl2/pytest.log 2>&1; echo "exit $?" >> gpurun_out/pdl2/pytest.log
for i in 1 2; do for p in 1 0; do ST_PDL_DENSE=$p timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/pdl2/wide_${p}_$i.json 2>/dev/null; done; done
for p in 1 0; do ST_PDL_DENSE=$p timeout 300 python bench.py --workload deep_mlp --no-cpu --no-e2e > gpurun_out/pdl2/deep_${p}.json 2>/dev/null; done
