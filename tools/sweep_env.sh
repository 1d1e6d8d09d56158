# Development: bench step time of each workload under environment variants
for W in ${WORKLOADS:-wide_fcn lstm_lm vgg16}; do for E in "${@}"; do
  echo "$W [$E] $(env $E timeout 300 python bench.py --workload $W --no-cpu --no-e2e --steps 40 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])')"
done; done
