# implicit-GEMM conv: parity tests + VGG bench (implicit vs ST_CONV_IM2COL=1)
mkdir -p gpurun_out/conv
timeout 600 python -m pytest tests/test_gpu_conv.py -x -q > gpurun_out/conv/pytest.log 2>&1; echo "exit $?" >> gpurun_out/conv/pytest.log
timeout 300 python bench.py --workload vgg16 --no-cpu --no-e2e > gpurun_out/conv/vgg.json 2> gpurun_out/conv/vgg.err
ST_CONV_IM2COL=1 timeout 300 python bench.py --workload vgg16 --no-cpu --no-e2e > gpurun_out/conv/vgg_im2col.json 2> gpurun_out/conv/vgg_im2col.err
