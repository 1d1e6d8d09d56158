mkdir -p gpurun_out/san
for w in hybrid graph layers; do
  timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_r2.py $w > gpurun_out/san/r2_memcheck_$w.log 2>&1
done
timeout 900 compute-sanitizer --tool memcheck --target-processes all --print-limit 20 python tools/sanitize_r2.py p2p > gpurun_out/san/r2_memcheck_p2p.log 2>&1
timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_r2.py hybrid > gpurun_out/san/r2_synccheck_hybrid.log 2>&1
