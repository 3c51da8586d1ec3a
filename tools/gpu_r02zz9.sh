#!/bin/bash
# append placement on unsplit one-wave grids with long suffixes (M7 r=0 / 0.25 per-rank slices at P=8, r=0 at P=4)
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
A="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
for rep in 1 2; do for O in 0 1; do
  for r in 0.0 0.25; do PCR_APPEND_OWNER=$O timeout 400 python bench.py --workload M7 --ratio $r --rank-slice 8 $A 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('owner=$O M7 r=$r P=8 ttft', round(j['ttft_ms'],3), 'T*', round(j['ttft_over_t_star'],3), 'own', round(j['roofline_attn']['isolated']['achieved']))"; done
  PCR_APPEND_OWNER=$O timeout 400 python bench.py --workload M7 --ratio 0.0 --rank-slice 4 $A 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('owner=$O M7 r=0 P=4 ttft', round(j['ttft_ms'],3), 'T*', round(j['ttft_over_t_star'],3), 'own', round(j['roofline_attn']['isolated']['achieved']))"
done; done
