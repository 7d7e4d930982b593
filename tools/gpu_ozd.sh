OUT=gpurun_out/${1:-ozd}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_oz.py -q -x > $OUT/t.log 2>&1; tail -3 $OUT/t.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/l.csv python tools/probe/oz_time.py --stored > $OUT/time.log 2>&1
cat $OUT/time.log
grep -E "ozd|convert|digits" $OUT/l.csv | awk -F'","' '{print $5, $NF}' | cut -c1-60,150-
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_ozd -c 2 -o $OUT/ozd python tools/probe/oz_time.py --stored > /dev/null 2>&1
