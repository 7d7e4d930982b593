# ncu of the INT8-emulated GEMM with and without FP64-tile multicast (C2 ax shape)
OUT=gpurun_out/mcncu
mkdir -p $OUT
for mc in 0 1; do
  RSVD_B200_OZ_MC=$mc timeout 600 ncu --set full --clock-control none -k regex:gemm_oz_kernel -c 1 \
      -o $OUT/mc$mc python tools/probe/oz_time.py 202599 4096 80 74 3 > $OUT/mc$mc.log 2>&1
done
ls -la $OUT
