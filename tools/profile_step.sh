# Profiles for profiles/ (run on the GPU box through gpurun):
#  1) launch list of a short bench run (ncu, durations only, serialised / cold)
#  2) one --set full capture of every library kernel of ONE timed bench step
#     (our kernels only: demangled names in namespace st::; the warm-up session's
#     kernels are skipped by count).
# usage: bash tools/profile_step.sh <workload> <kernels_per_step> <warmup_steps>
set -u
W=${1:-wide_fcn}; K=${2:-62}; WU=${3:-3}
mkdir -p gpurun_out/prof
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_$W.csv \
    python bench.py --workload $W --steps 2 --warmup $WU --no-e2e --no-cpu > gpurun_out/prof/launches_$W.log 2>&1
ncu --set full --clock-control none --kernel-name-base demangled -k regex:'st::' \
    -s $((K * WU)) -c $K -o gpurun_out/prof/step_$W \
    python bench.py --workload $W --steps 1 --warmup $WU --no-e2e --no-cpu > gpurun_out/prof/step_$W.log 2>&1
tail -3 gpurun_out/prof/step_$W.log
# summaries on the box (the full report is too large to bring back)
ncu -i gpurun_out/prof/step_$W.ncu-rep --page raw --csv > gpurun_out/prof/step_${W}_raw.csv 2>/dev/null
python tools/summarize_ncu.py full gpurun_out/prof/step_$W.ncu-rep > gpurun_out/prof/step_${W}_full.txt
python tools/summarize_ncu.py traffic gpurun_out/prof/step_$W.ncu-rep 'tc_dw_kernel|bias_grad_update|update_predict' \
    > gpurun_out/prof/step_${W}_dw_traffic.txt
python tools/summarize_ncu.py launches gpurun_out/prof/launches_$W.csv > gpurun_out/prof/launches_${W}_summary.csv
rm -f gpurun_out/prof/step_$W.ncu-rep
cat gpurun_out/prof/step_${W}_dw_traffic.txt
