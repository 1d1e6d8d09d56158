mkdir -p gpurun_out/pdl5
for p in 0 1; do
ST_PDL_DENSE=$p timeout 600 python bench.py --workload large_fcn --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/pdl5/large_$p.json 2>/dev/null
ST_PDL_DENSE=$p timeout 300 python bench.py --stages 2 --no-cpu --no-e2e > gpurun_out/pdl5/wide2_$p.json 2>/dev/null
ST_PDL_DENSE=$p timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/pdl5/wide1_$p.json 2>/dev/null
done
