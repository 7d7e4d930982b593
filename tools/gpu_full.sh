# full GPU check: all -m gpu tests, C2/C1/C4 bench lines, C2 launch list
set -x
OUT=gpurun_out/${1:-full}
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 10 --no-cpu > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 600 python bench.py --config c1 --steps 20 --no-cpu > $OUT/bench_c1.json 2> $OUT/bench_c1.err
timeout 900 python bench.py --config c5 --steps 3 --e2e-steps 1 --no-cpu > $OUT/bench_c5.json 2> $OUT/bench_c5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c2.csv python tools/profile_config.py c2 > /dev/null 2>&1
ls -la $OUT
