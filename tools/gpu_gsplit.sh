# stored-digit GEMM with the accumulator groups split over the CTA pair (gsplit) vs 48+32 columns
timeout 600 python -m pytest tests/test_gpu_oz.py -q -x -k stored 2>&1 | tail -2
for gs in 1 0; do
  RSVD_B200_OZD_GSPLIT=$gs timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_ozd --csv --log-file gpurun_out/gs$gs.csv python tools/probe/oz_time.py 202599 4096 80 74 16 --stored > gpurun_out/gs$gs.log 2>&1
  echo "gsplit=$gs: $(grep gemm_ozd gpurun_out/gs$gs.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ') $(grep 'max rel' gpurun_out/gs$gs.log | tr '\n' ' ')"
done
timeout 900 python -m pytest tests/test_gpu_oz_solves.py tests/test_gpu_fullsize_parity.py -q -x 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
