mkdir -p gpurun_out/tsg2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tsg2/pytest.log 2>&1; echo "exit $?" >> gpurun_out/tsg2/pytest.log
for w in vgg16 lstm_lm; do timeout 300 python bench.py --workload $w --no-cpu --no-e2e > gpurun_out/tsg2/$w.json 2> gpurun_out/tsg2/$w.err; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tsg2/launches_vgg16.csv python bench.py --workload vgg16 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
