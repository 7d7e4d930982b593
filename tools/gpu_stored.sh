# stored-digit atx passes: emulated-path tests, full-size parity, general parity, C2 bench
OUT=gpurun_out/stored
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_oz_solves.py tests/test_gpu_oz.py tests/test_gpu_fullsize_parity.py tests/test_gpu_parity.py tests/test_gpu_sharded.py tests/test_gpu_graph.py tests/test_gpu_fullsize.py -q 2>&1 | tail -4
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 > $OUT/bench_c2.json
python -c "import json; d=json.load(open('$OUT/bench_c2.json')); print('C2', d['ms_per_step'], d['value'], d.get('clocks'), d['e2e'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"oz_scan_convert|gemm_oz" --csv --log-file $OUT/sc.csv python tools/profile_config.py c2 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/stored/sc.csv")))
h=None
for r in rows:
    if "Kernel Name" in r: h=r; continue
    if h and len(r)==len(h) and 'scan_convert' in r[h.index("Kernel Name")]:
        print(r[h.index("Metric Name")], r[h.index("Metric Value")])
PY
