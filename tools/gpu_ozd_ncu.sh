OUT=gpurun_out/ozdncu
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ozd_kernel -c 2 \
    -o $OUT/ozd python tools/probe/oz_time.py 202599 4096 80 74 16 --stored > $OUT/log 2>&1
ls -la $OUT
