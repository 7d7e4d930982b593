#!/bin/bash
# gpurun: sharded GPU tests, the whole GPU suite, bench on C2 (default) and C1/C3/C5.
set -x
OUT=gpurun_out/${1:-r1b}
mkdir -p $OUT
free -g > $OUT/host.txt; nproc >> $OUT/host.txt
timeout 600 python -m pytest tests/test_gpu_sharded.py -x -q > $OUT/pytest_sharded.log 2>&1; echo "exit $?" >> $OUT/pytest_sharded.log
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "exit $?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 300 python bench.py --config c1 --steps 20 > $OUT/bench_c1.json 2> $OUT/bench_c1.err
timeout 900 python bench.py --config c3 --steps 5 --e2e-steps 1 > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 900 python bench.py --config c5 --steps 3 --e2e-steps 1 > $OUT/bench_c5.json 2> $OUT/bench_c5.err
timeout 300 python bench.py --impl reference --steps 1 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
ls -la $OUT
