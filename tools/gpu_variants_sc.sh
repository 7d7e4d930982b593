# oz_scan_convert variants in the C2 pipeline (ncu launch times)
OUT=gpurun_out/variants_sc
mkdir -p $OUT
cp paper_2110_03423_b200/_lib/librsvd_b200.so /tmp/lib_orig.so
for v in $(ls _variants); do
  cp _variants/$v/librsvd_b200.so paper_2110_03423_b200/_lib/librsvd_b200.so
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:oz_scan_convert --csv --log-file $OUT/$v.csv python tools/profile_config.py c2 > /dev/null 2>&1
  echo "$v: $(grep scan_convert $OUT/$v.csv | awk -F'","' '{print $(NF-2) "=" $NF}' | tr -d '"' | tr '\n' ' ')"
done
cp /tmp/lib_orig.so paper_2110_03423_b200/_lib/librsvd_b200.so
