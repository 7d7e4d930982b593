OUT=gpurun_out/tsncu
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32_kernel -c 3 \
    -o $OUT/ts_c4 python tools/profile_config.py c4 > $OUT/log 2>&1
ls -la $OUT
