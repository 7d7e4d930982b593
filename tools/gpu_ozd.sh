# stored-digit emulated GEMM (C2 shapes): scan + tiled conversion, both passes; tests
OUT=gpurun_out/ozd2
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_oz.py -q -x -k "stored" 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/ozd.csv python tools/probe/oz_time.py 202599 4096 80 74 16 --stored > $OUT/ozd.log 2>&1
tail -2 $OUT/ozd.log
python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/ozd2/ozd.csv")))
h=None
seen={}
for r in rows:
    if "Kernel Name" in r: h=r; continue
    if h and len(r)==len(h) and 'oz' in r[h.index("Kernel Name")]:
        k=r[h.index("Kernel Name")].split('(')[0][-40:]
        seen.setdefault(k,{})[r[h.index("Metric Name")]]=r[h.index("Metric Value")]
for k,v in seen.items(): print(k, v)
PY
