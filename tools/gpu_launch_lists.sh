# ncu launch lists (durations only, serialised and cold) of the LSTM LM and VGG-16 steps + summaries
TAG=${TAG:-r2ll}; mkdir -p gpurun_out/$TAG
for w in ${WORKLOADS:-lstm_lm vgg16}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$TAG/launches_$w.csv \
      python bench.py --workload $w --steps 2 --warmup 3 --no-e2e --no-cpu --graph off > gpurun_out/$TAG/launches_$w.log 2>&1
  python tools/summarize_ncu.py launches gpurun_out/$TAG/launches_$w.csv > gpurun_out/$TAG/launches_${w}_summary.csv
done
