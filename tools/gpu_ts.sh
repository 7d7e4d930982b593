# 3xTF32 GEMM with A in TMEM (TS) vs shared memory (SS): tests, C4 launch lists, bench
OUT=gpurun_out/ts
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tf32.py tests/test_gpu_f32.py -q -x 2>&1 | tail -3
for v in ts ss; do
  if [ $v = ss ]; then export RSVD_B200_TF32_SS=1; else unset RSVD_B200_TF32_SS; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_$v.csv python tools/profile_config.py c4 > /dev/null 2>&1
  echo "== $v"; python tools/launch_summary.py $OUT/launches_$v.csv 2>&1 | head -8
done
unset RSVD_B200_TF32_SS
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | cut -c1-400
