OUT=gpurun_out/${1:-ozdiag}
mkdir -p $OUT
for cfg in "202599 4096 80 74 23" "202599 4096 48 42 23" "202599 4096 32 30 23" "202599 4096 96 90 23"; do
  for d in 0 4; do
    RSVD_B200_OZ_DIAG=$d timeout 300 ncu --metrics gpu__time_duration.sum,lts__t_bytes.sum,dram__bytes_read.sum --clock-control none -k regex:gemm_oz_kernel --csv --log-file $OUT/d.csv python tools/probe/oz_time.py $cfg > /dev/null 2>&1
    echo "cfg $cfg diag $d: $(grep gemm_oz $OUT/d.csv | head -3 | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"' | tr '\n' ' ')"
  done
done
