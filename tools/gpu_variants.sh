# time the emulated GEMM (C2 shapes) under each prebuilt variant library in _variants/
OUT=gpurun_out/variants
mkdir -p $OUT
cp paper_2110_03423_b200/_lib/librsvd_b200.so /tmp/lib_orig.so
for v in ${VARIANTS:-$(ls _variants)}; do
  cp _variants/$v/librsvd_b200.so paper_2110_03423_b200/_lib/librsvd_b200.so
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_oz_kernel --csv --log-file $OUT/$v.csv python tools/probe/oz_time.py 202599 4096 80 74 3 > /dev/null 2>&1
  echo "$v: $(grep gemm_oz $OUT/$v.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"
done
cp /tmp/lib_orig.so paper_2110_03423_b200/_lib/librsvd_b200.so
