#!/bin/bash
# Small-SVD kernel A/B: in-smem Jacobi vs the multi-CTA block Jacobi for all widths.
for c in c1 c2 c4; do
  echo "== $c default"; timeout 600 python bench.py --config $c --steps 5 --e2e-steps 1 --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])"
  echo "== $c block"; RSVD_B200_JACOBI_SMEM_MAX=0 timeout 600 python bench.py --config $c --steps 5 --e2e-steps 1 --no-cpu | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])"
done
RSVD_B200_JACOBI_SMEM_MAX=0 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f32.py -q -x 2>&1 | tail -2
