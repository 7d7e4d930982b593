# conversion / sketch overlap on the side stream: tests + C2 timing for chunk counts 0 (off), 4, 8
timeout 1200 python -m pytest tests/test_gpu_oz_solves.py tests/test_gpu_graph.py tests/test_gpu_fullsize_parity.py tests/test_gpu_sharded.py -q -x 2>&1 | tail -2
for ov in 0 4 8; do
  RSVD_B200_OZ_OVERLAP=$ov timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('overlap $ov', d['ms_per_step'], d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
