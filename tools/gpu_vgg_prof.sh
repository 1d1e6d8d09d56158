# ncu --set full with source of a few VGG-16 implicit-conv GEMM launches (stall reasons per line)
mkdir -p gpurun_out/vp
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'tc_tsg_kernel' \
    -s 40 -c 6 -o gpurun_out/vp/tsg python bench.py --workload vgg16 --steps 1 --warmup 2 --no-e2e --no-cpu --graph off > gpurun_out/vp/tsg.log 2>&1
ncu -i gpurun_out/vp/tsg.ncu-rep --page raw --csv > gpurun_out/vp/tsg_raw.csv 2>/dev/null
ncu -i gpurun_out/vp/tsg.ncu-rep --page source --csv --print-source sass > gpurun_out/vp/tsg_source.csv 2>/dev/null
ncu -i gpurun_out/vp/tsg.ncu-rep --page details --csv > gpurun_out/vp/tsg_details.csv 2>/dev/null
python tools/summarize_ncu.py full gpurun_out/vp/tsg.ncu-rep > gpurun_out/vp/tsg_full.txt 2>&1
rm -f gpurun_out/vp/tsg.ncu-rep
