# each config with the emulated passes and with DMMA
OUT=gpurun_out/${1:-cmp}
mkdir -p $OUT
for c in c3 c5 c2; do
  for g in oz dmma; do
    RSVD_B200_GEMM=$g timeout 900 python bench.py --config $c --steps 3 --e2e-steps 1 --no-cpu > $OUT/b_${c}_$g.json 2> $OUT/b_${c}_$g.err
    python -c "import json;d=json.load(open('$OUT/b_${c}_$g.json'));print('$c $g', d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['ms_per_launch'])"
  done
done
