# ncu source-level captures of the s-side kernels (Jacobi, Cholesky, block Jacobi)
OUT=gpurun_out/${1:-small}
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"jacobi_kernel|cholesky_kernel" -c 3 \
    -o $OUT/small_c1 python tools/profile_config.py c1 > $OUT/c1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"block_jacobi|cholesky_kernel" -c 3 \
    -o $OUT/small_c4 python tools/profile_config.py c4 > $OUT/c4.log 2>&1
ls -la $OUT
