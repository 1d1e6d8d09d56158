mkdir -p gpurun_out/s2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/s2/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s2/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/s2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/s2/bench_default.json 2> gpurun_out/s2/bench_default.err
mkdir -p gpurun_out/r1bench
bash tools/bench_all.sh
cp -r gpurun_out/r1bench gpurun_out/s2/
