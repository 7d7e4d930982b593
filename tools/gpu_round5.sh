#!/bin/bash
set -x
OUT=gpurun_out/${1:-r1e}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_tf32.py tests/test_gpu_f32.py -q > $OUT/pytest_f32.log 2>&1; echo "exit $?" >> $OUT/pytest_f32.log
timeout 900 python bench.py --config c4 --steps 5 --e2e-steps 1 --no-cpu > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c4.csv python tools/profile_config.py c4 > $OUT/launches_c4.log 2>&1
ls -la $OUT
