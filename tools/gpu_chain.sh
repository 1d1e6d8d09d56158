mkdir -p gpurun_out/chain
for c in 0 32 16; do
  ST_MAX_CHAIN_KB=$c M=1 WIDTH=8192 LAYERS=2 timeout 600 python tools/fullsize_debug.py > gpurun_out/chain/dbg_$c.txt 2>&1
  ST_MAX_CHAIN_KB=$c timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/chain/wide_$c.json 2>/dev/null
  ST_MAX_CHAIN_KB=$c timeout 300 python bench.py --workload vgg16 --no-cpu --no-e2e > gpurun_out/chain/vgg_$c.json 2>/dev/null
  ST_MAX_CHAIN_KB=$c timeout 300 python bench.py --workload lstm_lm --no-cpu --no-e2e > gpurun_out/chain/lstm_$c.json 2>/dev/null
done
