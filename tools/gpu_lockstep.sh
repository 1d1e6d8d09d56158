mkdir -p gpurun_out/ls
python tools/dwu_shapes.py > gpurun_out/ls/dwu_default.txt 2>&1
ST_DW_LOCKSTEP=1 python tools/dwu_shapes.py > gpurun_out/ls/dwu_lockstep.txt 2>&1
timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/ls/b_default.json 2>/dev/null
ST_DW_LOCKSTEP=1 timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/ls/b_lock.json 2>/dev/null
for n in 64 72 96; do ST_DW_LOCKSTEP=1 ST_DWU_SMS=$n timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/ls/b_lock_$n.json 2>/dev/null; done
ST_DW_LOCKSTEP=1 timeout 600 python bench.py --workload large_fcn --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ls/large_lock.json 2>/dev/null
timeout 600 python bench.py --workload large_fcn --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ls/large_def.json 2>/dev/null
ST_DW_LOCKSTEP=1 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_pipeline.py -q -x > gpurun_out/ls/pytest.log 2>&1; echo "exit $?" >> gpurun_out/ls/pytest.log
