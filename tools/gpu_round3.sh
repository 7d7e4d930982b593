#!/bin/bash
set -x
OUT=gpurun_out/${1:-r1c}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "sizes or wide_sketch or fallback" > $OUT/pytest_wide.log 2>&1; echo "exit $?" >> $OUT/pytest_wide.log
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 5 > $OUT/bench_c2.json 2> $OUT/bench_c2.err
ls -la $OUT
