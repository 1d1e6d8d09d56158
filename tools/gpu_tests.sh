# GPU test suite (no -x: every failure reported), slowest tests listed, smoke
TAG=${TAG:-r2t}
mkdir -p gpurun_out/$TAG
timeout 2400 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/$TAG/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$TAG/smoke.log 2>&1
