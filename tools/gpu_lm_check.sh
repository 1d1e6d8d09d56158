# LM / conv parity after a bias-gradient heuristic change, LM + VGG benches, LM launch list
TAG=${TAG:-r2bg}; mkdir -p gpurun_out/$TAG
timeout 1200 python -m pytest tests/test_gpu_lstm.py tests/test_gpu_conv.py tests/test_gpu_kernels.py -q --timeout=600 > gpurun_out/$TAG/pytest.log 2>&1; echo "exit $?" >> gpurun_out/$TAG/pytest.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -k "lstm or vgg16_full_size_single" --timeout=600 >> gpurun_out/$TAG/pytest.log 2>&1; echo "exit $?" >> gpurun_out/$TAG/pytest.log
for r in 1 2; do timeout 300 python bench.py --workload lstm_lm --no-cpu --no-e2e --steps 30 > gpurun_out/$TAG/lstm_r$r.json 2>&1; done
timeout 300 python bench.py --workload vgg16 --no-cpu --no-e2e > gpurun_out/$TAG/vgg16.json 2>&1
WORKLOADS=lstm_lm TAG=$TAG bash tools/gpu_launch_lists.sh
