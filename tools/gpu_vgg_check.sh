mkdir -p gpurun_out/r2vgg
timeout 1500 python -m pytest tests/test_gpu_conv.py tests/test_gpu_variants.py tests/test_gpu_fullsize.py -k "conv or vgg" -q --timeout=900 > gpurun_out/r2vgg/pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2vgg/pytest.log
for r in 1 2; do timeout 300 python bench.py --workload vgg16 --no-cpu > gpurun_out/r2vgg/vgg16_r$r.json 2>&1; done
timeout 300 python bench.py --workload vgg16 --stages 8 --no-cpu > gpurun_out/r2vgg/vgg16_s8.json 2>&1
