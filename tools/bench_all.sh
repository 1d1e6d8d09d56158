# Every workload on one GPU (N=1 and co-located stage counts), JSON lines into $OUT/
OUT=${OUT:-gpurun_out/r1bench}; mkdir -p $OUT
for w in wide_fcn lstm_lm vgg16 mlp deep_mlp; do
  timeout 300 python bench.py --workload $w --no-cpu > $OUT/$w.json 2> $OUT/$w.err
done
for s in 2 4 8; do
  timeout 300 python bench.py --workload wide_fcn --stages $s --no-cpu > $OUT/wide_fcn_s$s.json 2>&1
done
timeout 300 python bench.py --workload lstm_lm --stages 4 --no-cpu > $OUT/lstm_lm_s4.json 2>&1
timeout 300 python bench.py --workload vgg16 --stages 8 --no-cpu > $OUT/vgg16_s8.json 2>&1
timeout 600 python bench.py --workload large_fcn --no-cpu --steps 10 --warmup 3 > $OUT/large_fcn.json 2>&1
for s in 2 4 8; do
  timeout 600 python bench.py --workload large_fcn --stages $s --no-cpu --steps 10 --warmup 3 > $OUT/large_fcn_s$s.json 2>&1
done
# NEXT-4 on VGG-16's imbalanced 8-stage pipeline (co-located): profiled cuts, a replicated conv front
timeout 600 python bench.py --workload vgg16 --stages 8 --partition profiled --no-cpu > $OUT/vgg16_s8_profiled.json 2>&1
timeout 600 python bench.py --workload vgg16 --replicas 2,1,1,1,1,1,1,1 --no-cpu > $OUT/vgg16_s8_rep2.json 2>&1
# 1xTF32 "fast" mode of the tensor-bound workloads (parity is checked in 3xTF32 only)
for w in vgg16 lstm_lm wide_fcn; do
  timeout 300 python bench.py --workload $w --gemm tf32 --no-cpu > $OUT/${w}_tf32.json 2> $OUT/${w}_tf32.err
done
