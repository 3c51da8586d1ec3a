#!/bin/bash
# split only grids under 48 CTAs: full suite, per-rank slices, L8 line
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
A="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
for r in 0.0 0.25 0.5 0.75 0.875 1.0; do timeout 400 python bench.py --workload M7 --ratio $r --rank-slice 8 $A 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('M7 r=$r P=8 ttft', round(j['ttft_ms'],3), 'T*', round(j['ttft_over_t_star'],3), 'own', round(j['roofline_attn']['isolated']['achieved']))"; done
for P in 2 4; do timeout 400 python bench.py --workload M7 --ratio 0.75 --rank-slice $P $A 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('M7 r=.75 P=$P ttft', round(j['ttft_ms'],3), 'T*', round(j['ttft_over_t_star'],3))"; done
for r in 0.5 0.75 0.875; do timeout 600 python bench.py --workload L70 --ratio $r --rank-slice 8 --steps 5 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('L70 r=$r P=8 ttft', round(j['ttft_ms'],3), 'T*', round(j['ttft_over_t_star'],3))"; done
for P in 1 2 4 8; do timeout 400 python bench.py --rank-slice $P $A 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('L8 P=$P ttft', round(j['ttft_ms'],3), 'T*', round(j['ttft_over_t_star'],3), 'own us', round(j['roofline_attn']['isolated']['avg_launch_ms']*1e3,1))"; done
