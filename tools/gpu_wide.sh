# wide-row conversion (scan + tiles) at C3 / C5: tests + bench + launch lists
OUT=gpurun_out/wide
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_oz_solves.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
for c in c3 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --e2e-steps 1 --no-cpu 2>&1 | tail -1 > $OUT/bench_$c.json
  python -c "import json; d=json.load(open('$OUT/bench_$c.json')); print('$c', d['ms_per_step'], d['value'], d.get('clocks'))"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$c.csv python tools/profile_config.py $c > /dev/null 2>&1
  python tools/launch_summary.py $OUT/launches_$c.csv 2>/dev/null | head -6
done
