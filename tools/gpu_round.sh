#!/bin/bash
# One gpurun call: GPU tests, bench, DMMA peak probe, ncu launch list and full captures.
# Usage (on the box): bash tools/gpu_round.sh [tag]
set -x
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/probe/fp64_peak.cu && /tmp/fp64_peak > $OUT/fp64_peak.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/profile_solve.py > $OUT/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_ax_kernel -c 1 -o $OUT/prof_ax python tools/profile_solve.py > $OUT/prof_ax.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_atx_kernel -c 1 -o $OUT/prof_atx python tools/profile_solve.py > $OUT/prof_atx.log 2>&1
ls -la $OUT
