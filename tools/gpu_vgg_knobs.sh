# VGG-16 at one stage: the opt-in conv variants (dev build) re-measured against the default
TAG=${TAG:-r2vk}; mkdir -p gpurun_out/$TAG
DEV=paper_1809_02839_b200/_var/dev/libspectrain.so
for r in 1 2; do
  for cfg in "X=0" "ST_CONV_OVERLAP=1" "ST_CONV_PAIR=1" "ST_CONV_OVERLAP=1 ST_CONV_PAIR=1" "ST_TSG_NARROW=0"; do
    tag=$(echo $cfg | tr ' =' '__')
    env $cfg ST_LIB_PATH=$DEV timeout 300 python bench.py --workload vgg16 --no-cpu --no-e2e --steps 50 > gpurun_out/$TAG/vgg_${tag}_r$r.json 2>&1
  done
done
