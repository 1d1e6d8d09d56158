# wide FCN: SM budget of the overlapped dW + update (dev ST_DWU_SMS; dX gets the rest), two passes
mkdir -p gpurun_out/r2ws
DEV=paper_1809_02839_b200/_var/dev/libspectrain.so
for r in 1 2; do for s in 80 72 88 96 104 112; do
  ST_LIB_PATH=$DEV ST_DWU_SMS=$s timeout 300 python bench.py --workload wide_fcn --no-cpu --no-e2e --steps 50 > gpurun_out/r2ws/w_${s}_r$r.json 2>&1
done; done
