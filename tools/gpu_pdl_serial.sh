# programmatic launches in the serialised large-layer backward: A/B on one box (dev ST_PDL_SERIAL)
mkdir -p gpurun_out/r2pdls
DEV=paper_1809_02839_b200/_var/dev/libspectrain.so
for r in 1 2; do for v in 0 1; do
  ST_LIB_PATH=$DEV ST_PDL_SERIAL=$v timeout 600 python bench.py --no-cpu --no-e2e --steps 30 > gpurun_out/r2pdls/large_fcn_p${v}_r$r.json 2>&1
done; done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -k "16384" --timeout=900 > gpurun_out/r2pdls/pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2pdls/pytest.log
