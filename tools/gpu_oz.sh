set -x
OUT=gpurun_out/${1:-oz}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_oz.py -q -x > $OUT/pytest_oz.log 2>&1; echo "exit $?" >> $OUT/pytest_oz.log
timeout 300 python tools/probe/oz_time.py > $OUT/oz_time.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/oz_launches.csv python tools/probe/oz_time.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_oz_kernel -c 1 -o $OUT/oz_ax python tools/probe/oz_time.py > /dev/null 2>&1
ls -la $OUT
