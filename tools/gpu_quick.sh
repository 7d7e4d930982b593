# quick check: parity tests + C2/C1 bench + C2 launch list
set -x
OUT=gpurun_out/${1:-quick}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_parity.py tests/test_gpu_graph.py -q -x > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 600 python bench.py --steps 10 --no-cpu > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 600 python bench.py --config c1 --steps 20 --no-cpu > $OUT/bench_c1.json 2> $OUT/bench_c1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c2.csv python tools/profile_config.py c2 > /dev/null 2>&1
ls -la $OUT
