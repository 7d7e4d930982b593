# full GPU check: all -m gpu tests, bench lines for every config (C2 with the CPU leg), launch
# lists, ncu of the dominant kernels (stored-digit emulated passes + the fused conversion)
set -x
OUT=gpurun_out/${1:-full}
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py --config c2 --steps 10 > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 900 python bench.py --config c1 --steps 50 --warmup 5 --e2e-steps 5 --no-cpu > $OUT/bench_c1.json 2> $OUT/bench_c1.err
for c in c3 c4 c5 c5ill; do
  timeout 900 python bench.py --config $c --steps 5 --e2e-steps 1 --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
for c in c1 c2 c3 c4 c5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$c.csv python tools/profile_config.py $c > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_ozd_kernel|oz_scan_convert" -c 3 -o $OUT/ozd_c2 python tools/profile_config.py c2 > /dev/null 2>&1
ls -la $OUT
