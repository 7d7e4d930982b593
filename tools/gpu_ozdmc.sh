# stored-digit GEMM: chunk CTAs clustered with multicast (1) vs independent (0)
for mc in 1 0; do
  RSVD_B200_OZD_MC=$mc timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_ozd --csv --log-file gpurun_out/ozdmc$mc.csv python tools/probe/oz_time.py 202599 4096 80 74 16 --stored > gpurun_out/ozdmc$mc.log 2>&1
  echo "mc=$mc: $(grep gemm_ozd gpurun_out/ozdmc$mc.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ') $(grep 'max rel' gpurun_out/ozdmc$mc.log | tr '\n' ' ')"
  RSVD_B200_OZD_MC=$mc timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  C2', d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
RSVD_B200_OZD_MC=0 timeout 600 python -m pytest tests/test_gpu_oz.py -q -x -k stored 2>&1 | tail -2
