mkdir -p gpurun_out/pdl3
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pdl3/pytest.log 2>&1; echo "exit $?" >> gpurun_out/pdl3/pytest.log
for p in 1 0; do
  ST_PDL_DENSE=$p timeout 300 python bench.py --workload vgg16 --no-cpu --no-e2e > gpurun_out/pdl3/vgg_$p.json 2>/dev/null
  ST_PDL_DENSE=$p timeout 300 python bench.py --workload lstm_lm --no-cpu --no-e2e > gpurun_out/pdl3/lstm_$p.json 2>/dev/null
  ST_PDL_DENSE=$p timeout 300 python bench.py --workload mlp --no-cpu --no-e2e > gpurun_out/pdl3/mlp_$p.json 2>/dev/null
  ST_PDL_DENSE=$p timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/pdl3/wide_$p.json 2>/dev/null
done
