# faster column digits of the small operand: tests + launch times + C2 bench
timeout 1200 python -m pytest tests/test_gpu_oz.py tests/test_gpu_oz_solves.py tests/test_gpu_fullsize_parity.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dcols2.csv python tools/profile_config.py c2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/dcols2.csv 2>/dev/null | grep -i "digits\|colmax\|total"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
