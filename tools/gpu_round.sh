# One GPU call: GPU tests (per-test timeout), smoke, default bench, every workload (JSON lines under gpurun_out/$TAG/)
TAG=${TAG:-r2}
mkdir -p gpurun_out/$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/$TAG/smi.txt 2>&1
timeout 2400 python -u -m pytest tests -m gpu -q --timeout=900 --durations=20 > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/$TAG/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$TAG/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/$TAG/bench_default.json 2> gpurun_out/$TAG/bench_default.err
OUT=gpurun_out/$TAG bash tools/bench_all.sh
