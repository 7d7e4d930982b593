# 3xTF32 GEMM (TS): tests, C4 launch list, bench
OUT=gpurun_out/ts2
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_tf32.py tests/test_gpu_f32.py -q -x 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python tools/profile_config.py c4 > /dev/null 2>&1
python tools/launch_summary.py $OUT/launches.csv 2>&1 | head -6
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | cut -c1-300
