#!/bin/bash
# append placement A/B on the one-wave long-suffix slices (same box): M7 r=0.5 at P = 4 and 8
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
A="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
for rep in 1 2; do for O in 0 1; do for P in 4 8; do
  PCR_APPEND_OWNER=$O timeout 400 python bench.py --workload M7 --ratio 0.5 --rank-slice $P $A 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('owner=$O P=$P ttft', round(j['ttft_ms'],3), 'T*', round(j['ttft_over_t_star'],3), 'own', round(j['roofline_attn']['isolated']['achieved']))"
done; done; done
