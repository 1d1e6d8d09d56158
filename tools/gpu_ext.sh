mkdir -p gpurun_out/ext
for e in 2 3; do
  for i in 1 2; do ST_EXT_REDUCE=$e timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/ext/wide_e${e}_$i.json 2>/dev/null; done
  ST_EXT_REDUCE=$e timeout 300 python bench.py --workload vgg16 --no-cpu --no-e2e > gpurun_out/ext/vgg_e$e.json 2>/dev/null
  ST_EXT_REDUCE=$e timeout 300 python bench.py --workload lstm_lm --no-cpu --no-e2e > gpurun_out/ext/lstm_e$e.json 2>/dev/null
done
