# co-located 8-stage runs repeated (a wide-FCN 8-stage bench hit bench.py's 4-minute watchdog once)
mkdir -p gpurun_out/r2s8
for r in 1 2 3 4; do
  timeout 300 python bench.py --workload wide_fcn --stages 8 --no-cpu > gpurun_out/r2s8/w8_r$r.json 2>&1; echo "w8 r$r exit $?" >> gpurun_out/r2s8/status.txt
done
for r in 1 2; do
  timeout 300 python bench.py --workload large_fcn --stages 8 --no-cpu --steps 10 --warmup 3 > gpurun_out/r2s8/l8_r$r.json 2>&1; echo "l8 r$r exit $?" >> gpurun_out/r2s8/status.txt
done
