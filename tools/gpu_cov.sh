mkdir -p gpurun_out/cov
timeout 600 python -m pytest tests/test_gpu_conv.py -q -x > gpurun_out/cov/pytest.log 2>&1; echo "exit $?" >> gpurun_out/cov/pytest.log
for o in 1 0; do ST_CONV_OVERLAP=$o timeout 300 python bench.py --workload vgg16 --no-cpu --no-e2e > gpurun_out/cov/vgg_$o.json 2>/dev/null; done
for n in 64 96; do ST_DWU_SMS=$n timeout 300 python bench.py --workload vgg16 --no-cpu --no-e2e > gpurun_out/cov/vgg_d$n.json 2>/dev/null; done
