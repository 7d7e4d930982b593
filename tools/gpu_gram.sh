# upper-triangle DMMA Grams + padding-row skip in gemm_atx: tests + C2 / C1 launch lists + bench
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in c2 c1; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gram_$c.csv python tools/profile_config.py $c > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/gram_$c.csv 2>/dev/null | grep -i "gemm_atx\|total"
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
timeout 600 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C1', d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
