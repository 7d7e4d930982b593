# INT8-emulated GEMM (C2 shapes, ax + atx launches): independent FP64-tile loads vs multicast
OUT=gpurun_out/mc3
mkdir -p $OUT
for mc in 0 1; do
  RSVD_B200_OZ_MC=$mc timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_oz_kernel --csv --log-file $OUT/t$mc.csv python tools/probe/oz_time.py 202599 4096 80 74 3 > /dev/null 2>&1
  echo "mc $mc: $(grep gemm_oz $OUT/t$mc.csv | awk -F'","' '{print $5 " " $NF}' | tr -d '"' | sed 's/rsvdb200::oz::gemm_oz_kernel//' | tr '\n' ' ')"
done
RSVD_B200_OZ_MC=1 timeout 300 python -m pytest tests/test_gpu_oz.py -q -x 2>&1 | tail -2
