# The driver's N > 1 launch (torchrun, one rank per GPU, NCCL) exercised on a one-GPU box:
# ST_BENCH_SHARED_GPU=1 puts every rank on cuda:0 (distinct NCCL hosts). Checks the whole
# path — NCCL parity leg, comm plans, barrier + max-over-ranks timing, the JSON line — not speed.
TAG=${TAG:-r2tr}; mkdir -p gpurun_out/$TAG
for n in 2 4; do
  ST_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + n)) bench.py --gpus $n --steps 4 --warmup 3 > gpurun_out/$TAG/large_fcn_n$n.json 2> gpurun_out/$TAG/large_fcn_n$n.err
  echo "exit $?" >> gpurun_out/$TAG/large_fcn_n$n.err
done
ST_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29510 bench.py --gpus 2 --steps 4 --warmup 3 --impl reference > gpurun_out/$TAG/ref_n2.json 2> gpurun_out/$TAG/ref_n2.err
echo "exit $?" >> gpurun_out/$TAG/ref_n2.err
