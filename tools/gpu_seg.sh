mkdir -p gpurun_out/seg3
export ST_LIB_PATH=paper_1809_02839_b200/_var/dev/libspectrain.so
for sg in 0 32 64; do
  ST_TSG_SEG=$sg timeout 900 python tools/vgg_spread.py 10 > gpurun_out/seg3/vgg_spread_seg$sg.txt 2>&1
  for w in vgg16 lstm_lm; do
    ST_TSG_SEG=$sg timeout 300 python bench.py --workload $w --no-cpu --no-e2e > gpurun_out/seg3/${w}_seg$sg.json 2> gpurun_out/seg3/${w}_seg$sg.err
  done
done
