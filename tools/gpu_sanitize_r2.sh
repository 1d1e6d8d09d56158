mkdir -p gpurun_out/san
D=$(mktemp -d); PORT=29533
for r in 0 1; do
  timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_r2.py p2p_rank $r $PORT $D > gpurun_out/san/r2_memcheck_p2p_rank$r.log 2>&1 &
done
wait
ls $D >> gpurun_out/san/r2_memcheck_p2p_rank0.log
