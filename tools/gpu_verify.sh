TAG=r2v
mkdir -p gpurun_out/$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/$TAG/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/$TAG/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/$TAG/bench_default.json 2> gpurun_out/$TAG/bench_default.err
timeout 2400 python -u -m pytest tests -m gpu -q --timeout=900 --durations=30 > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/$TAG/pytest_gpu.log
