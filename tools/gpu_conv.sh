# implicit-GEMM conv: parity tests + VGG bench (TMEM-A / persistent smem-A kernels)
mkdir -p gpurun_out/conv
timeout 600 python -m pytest tests/test_gpu_conv.py -x -q > gpurun_out/conv/pytest.log 2>&1; echo "exit $?" >> gpurun_out/conv/pytest.log
timeout 300 python bench.py --workload vgg16 --no-cpu --no-e2e > gpurun_out/conv/vgg.json 2> gpurun_out/conv/vgg.err
ST_CONV_TS=0 timeout 300 python bench.py --workload vgg16 --no-cpu --no-e2e > gpurun_out/conv/vgg_np.json 2> gpurun_out/conv/vgg_np.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/conv/launches_vgg16.csv python bench.py --workload vgg16 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
