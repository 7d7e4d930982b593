#!/bin/bash
set -x
OUT=gpurun_out/${1:-check}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 5 --no-cpu > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 600 python bench.py --config c1 --steps 20 --no-cpu > $OUT/bench_c1.json 2> $OUT/bench_c1.err
timeout 900 python bench.py --config c4 --steps 5 --e2e-steps 1 --no-cpu > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c1.csv python tools/profile_config.py c1 > $OUT/launches_c1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c4.csv python tools/profile_config.py c4 > $OUT/launches_c4.log 2>&1
ls -la $OUT
