# Development: time the FP32X3 fwd / dX GEMM (8192², B=128) with pipeline stages disabled
# (ST_GEMM_DEV_FLAGS bits, see TcParams::dev_flags) for the single-CTA and CTA-pair kernels.
FLAGS=${FLAGS:-"0 1 2 4 8 3 12 13"}
for P in 0 1; do for F in $FLAGS; do
echo "PAIR=$P FLAGS=$F $(ST_GEMM_PAIR=$P ST_GEMM_DEV_FLAGS=$F timeout 60 python tools/time_gemm.py 2>&1 | grep fp32x3 | grep -E '^(fwd|dX )' | awk '{print $1, $6}' | tr '\n' ' ')"
done; done
