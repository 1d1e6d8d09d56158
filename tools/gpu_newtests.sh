# GPU call: P2P (IPC processes) tests, per-test timeout
mkdir -p gpurun_out/nt
timeout 1200 python -u -m pytest tests/test_gpu_p2p.py -m gpu -v --timeout=300 > gpurun_out/nt/test_gpu_p2p.log 2>&1; echo "exit $?" >> gpurun_out/nt/test_gpu_p2p.log
