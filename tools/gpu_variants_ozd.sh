# stored-digit GEMM variants (C2 shapes)
OUT=gpurun_out/variants_ozd
mkdir -p $OUT
cp paper_2110_03423_b200/_lib/librsvd_b200.so /tmp/lib_orig.so
for v in $(ls _variants); do
  cp _variants/$v/librsvd_b200.so paper_2110_03423_b200/_lib/librsvd_b200.so
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_ozd --csv --log-file $OUT/$v.csv python tools/probe/oz_time.py 202599 4096 80 74 16 --stored > $OUT/$v.log 2>&1
  echo "$v: $(grep gemm_ozd $OUT/$v.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ') $(grep 'max rel' $OUT/$v.log | tr '\n' ' ')"
done
cp /tmp/lib_orig.so paper_2110_03423_b200/_lib/librsvd_b200.so
