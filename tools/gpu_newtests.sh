# GPU call: the tests of the round-2 additions (P2P transport, hybrid DP x PP, per-layer profile) + pipeline regressions
mkdir -p gpurun_out/nt
timeout 1500 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_hybrid.py tests/test_gpu_partition.py tests/test_gpu_pipeline.py tests/test_gpu_nccl.py tests/test_gpu_lstm.py tests/test_gpu_conv.py -m gpu -q --durations=15 > gpurun_out/nt/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/nt/pytest.log
