mkdir -p gpurun_out/stash
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_variants.py -x -q > gpurun_out/stash/pytest.log 2>&1; echo "exit $?" >> gpurun_out/stash/pytest.log
for p in spectrain stash none; do
timeout 300 python bench.py --workload wide_fcn --stages 4 --pred $p --no-cpu --no-e2e > gpurun_out/stash/wide4_$p.json 2> gpurun_out/stash/wide4_$p.err
done
