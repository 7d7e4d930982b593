#!/bin/bash
set -x
OUT=gpurun_out/${1:-r1d}
mkdir -p $OUT
timeout 900 python bench.py --config c4 --steps 5 --e2e-steps 1 > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c4.csv python tools/profile_config.py c4 > $OUT/launches_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32_kernel -c 2 -o $OUT/prof_tf32 python tools/profile_config.py c4 > $OUT/prof_tf32.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
ls -la $OUT
