#!/bin/bash
# Full GPU check: tests, then the bench for every config (no CPU leg), launch lists C2.
set -x
OUT=gpurun_out/${1:-all}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
for c in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --e2e-steps 1 --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c2.csv python tools/profile_config.py c2 > /dev/null 2>&1
ls -la $OUT
