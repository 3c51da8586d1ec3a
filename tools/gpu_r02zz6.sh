#!/bin/bash
# split-KV vs none on small long-suffix grids (M7 per-rank slices at P=8, r = 0.5 / 0.75 / 0.875; L70 r=0.875)
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
A="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
for r in 0.5 0.75 0.875; do for N in 136 1; do
  PCR_ATTN_SMS=$N timeout 400 python bench.py --workload M7 --ratio $r --rank-slice 8 $A 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('M7 r=$r P=8 sms=$N ttft', round(j['ttft_ms'],3), 'T*', round(j['ttft_over_t_star'],3), 'own', round(j['roofline_attn']['isolated']['achieved']), 'ld', round(j['gather_ms_per_layer']*1e3,1))"
done; done
for N in 136 1; do PCR_ATTN_SMS=$N timeout 600 python bench.py --workload L70 --ratio 0.875 --rank-slice 8 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('L70 r=.875 P=8 sms=$N ttft', round(j['ttft_ms'],3), 'T*', round(j['ttft_over_t_star'],3), 'own', round(j['roofline_attn']['isolated']['achieved']))"; done
for N in 136 1; do PCR_ATTN_SMS=$N timeout 400 python bench.py --rank-slice 8 $A 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('L8 P=8 sms=$N ttft', round(j['ttft_ms'],3), 'T*', round(j['ttft_over_t_star'],3))"; done
