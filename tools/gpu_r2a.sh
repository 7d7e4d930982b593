set -x
OUT=gpurun_out/${1:-r2b}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_parity.py tests/test_gpu_graph.py tests/test_gpu_sharded.py tests/test_gpu_f32.py tests/test_gpu_tf32.py -q -x > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 600 python bench.py --steps 10 --no-cpu > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 600 python bench.py --config c1 --steps 20 --no-cpu > $OUT/bench_c1.json 2> $OUT/bench_c1.err
timeout 600 python bench.py --config c4 --steps 5 --e2e-steps 1 --no-cpu > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c2.csv python tools/profile_config.py c2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_atx_kernel -c 1 -o $OUT/atx_c2 python tools/profile_config.py c2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ax_kernel -c 1 -o $OUT/ax_c2 python tools/profile_config.py c2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:jacobi_kernel -c 1 -o $OUT/jacobi_c2 python tools/profile_config.py c2 > /dev/null 2>&1
ls -la $OUT
