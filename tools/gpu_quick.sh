# quick GPU check: parity tests, GEMM timings, default bench
mkdir -p gpurun_out/q
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/q/pytest.log 2>&1; echo "exit $?" >> gpurun_out/q/pytest.log
timeout 120 python tools/time_gemm.py > gpurun_out/q/time_gemm.txt 2>&1
timeout 300 python bench.py --no-cpu ${BENCH_ARGS} > gpurun_out/q/bench.json 2> gpurun_out/q/bench.err
