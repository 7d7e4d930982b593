#!/bin/bash
# Full GPU check: tests, the bench for every config (C2 with the CPU leg), the reference arm,
# launch lists of every config.
set -x
OUT=gpurun_out/${1:-all}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py --config c2 --steps 5 > $OUT/bench_c2.json 2> $OUT/bench_c2.err
for c in c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
for c in c1 c2 c3 c4 c5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$c.csv python tools/profile_config.py $c > /dev/null 2>&1
done
ls -la $OUT
