# round-1 profiles of the VGG and LSTM steps: ncu launch lists (+summaries) and a full
# capture of the TMEM-A GEMM kernels (tensor-pipe / DRAM metrics)
mkdir -p gpurun_out/prof2
for w in vgg16 lstm_lm; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof2/launches_$w.csv \
      python bench.py --workload $w --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
  python tools/summarize_ncu.py launches gpurun_out/prof2/launches_$w.csv > gpurun_out/prof2/launches_${w}_summary.csv
done
ncu --set full --clock-control none --kernel-name-base demangled -k regex:'tc_tsg_kernel' -s 30 -c 6 \
    -o gpurun_out/prof2/tsg_vgg16 python bench.py --workload vgg16 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/prof2/tsg.log 2>&1
python tools/summarize_ncu.py full gpurun_out/prof2/tsg_vgg16.ncu-rep > gpurun_out/prof2/tsg_vgg16_full.txt
rm -f gpurun_out/prof2/tsg_vgg16.ncu-rep
