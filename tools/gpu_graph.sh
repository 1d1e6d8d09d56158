# GPU call: graph-mode tests and eager-vs-graph benches, P2P hung-peer test
mkdir -p gpurun_out/gr
timeout 600 python -u -m pytest tests/test_gpu_p2p.py tests/test_gpu_graph.py -m gpu -v --timeout=300 > gpurun_out/gr/pytest.log 2>&1; echo "exit $?" >> gpurun_out/gr/pytest.log
for w in mlp deep_mlp lstm_lm vgg16 wide_fcn; do
  for g in off on; do
    timeout 300 python bench.py --workload $w --graph $g --no-cpu --no-e2e > gpurun_out/gr/${w}_$g.json 2> gpurun_out/gr/${w}_$g.err
  done
done
