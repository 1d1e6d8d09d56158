mkdir -p gpurun_out/tsg
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tsg/pytest.log 2>&1; echo "exit $?" >> gpurun_out/tsg/pytest.log
for w in vgg16 lstm_lm wide_fcn; do
timeout 300 python bench.py --workload $w --no-cpu --no-e2e > gpurun_out/tsg/$w.json 2> gpurun_out/tsg/$w.err
done
ST_CONV_TS=0 timeout 300 python bench.py --workload lstm_lm --no-cpu --no-e2e > gpurun_out/tsg/lstm_lm_nots.json 2> /dev/null
