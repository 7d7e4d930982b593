# blocked Cholesky writing its factors in place: tests + C4 bench + launch list
timeout 1500 python -m pytest tests/test_gpu_small.py tests/test_gpu_parity.py tests/test_gpu_f32.py tests/test_gpu_fullsize.py tests/test_gpu_householder.py -q -x 2>&1 | tail -2
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4', d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/chol_c4.csv python tools/profile_config.py c4 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/chol_c4.csv 2>/dev/null | grep -i "chol\|small_gemm\|copy2d\|fill\|total"
