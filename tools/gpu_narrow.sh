mkdir -p gpurun_out/nar
timeout 600 python -m pytest tests/test_gpu_conv.py tests/test_gpu_lstm.py -q -x > gpurun_out/nar/pytest.log 2>&1; echo "exit $?" >> gpurun_out/nar/pytest.log
for n in 1 0; do ST_TSG_NARROW=$n timeout 300 python bench.py --workload vgg16 --no-cpu --no-e2e > gpurun_out/nar/vgg_$n.json 2>/dev/null; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/nar/launches_vgg16.csv python bench.py --workload vgg16 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
