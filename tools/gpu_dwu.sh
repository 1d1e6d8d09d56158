mkdir -p gpurun_out/exp
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/exp/pytest.log 2>&1; echo "exit $?" >> gpurun_out/exp/pytest.log
bash tools/sweep_variants.sh > gpurun_out/exp/variants_dwu.txt 2>&1
for v in "" paper_1809_02839_b200/_var/*.so; do
  echo "$(basename ${v:-default}) $(ST_LIB_PATH=$v timeout 300 python bench.py --no-cpu --no-e2e 2>&1 | tail -1)" >> gpurun_out/exp/bench_dwu.txt
done
