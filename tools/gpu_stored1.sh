# single stored layout (ax tiles read transposed by the atx passes): tests + timing
OUT=gpurun_out/stored1
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_oz.py -q -x 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_oz_solves.py tests/test_gpu_fullsize_parity.py -q -x 2>&1 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/l.csv python tools/profile_config.py c2 > /dev/null 2>&1
python tools/launch_summary.py $OUT/l.csv 2>/dev/null | head -4; python tools/launch_summary.py $OUT/l.csv 2>/dev/null | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 > $OUT/bench_c2.json
python -c "import json; d=json.load(open('$OUT/bench_c2.json')); print('C2', d['ms_per_step'], d['value'], d.get('clocks'))"
