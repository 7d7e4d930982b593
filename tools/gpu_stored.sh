# stored-digit atx passes: emulated-path tests, full-size parity, general parity, C2 bench
OUT=gpurun_out/stored
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_oz_solves.py tests/test_gpu_oz.py tests/test_gpu_fullsize_parity.py tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_graph.py tests/test_gpu_fullsize.py -q 2>&1 | tail -4
timeout 300 python tools/probe/stored_accuracy.py 2>&1 | tail -4
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 > $OUT/bench_c2.json
python -c "import json; d=json.load(open('$OUT/bench_c2.json')); print('C2', d['ms_per_step'], d['value'], d.get('clocks'), d['e2e']['ms_per_step'] if 'ms_per_step' in d['e2e'] else d['e2e'])"
