#!/bin/bash
# fused-append placement chosen per launch (owner placement for one-wave grids with long suffixes)
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for SH in 4096,4224,32,8 4096,4224,4,1 4096,4224,8,2 4096,4224,16,4 0,8320,32,8 4096,128,32,8 8192,8320,8,1; do timeout 300 python tools/attn_bench.py --shape $SH --iters 10 2>&1 | tail -1 | cut -c1-160; done
A="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
for P in 2 4 8; do timeout 400 python bench.py --workload M7 --ratio 0.5 --rank-slice $P $A 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('M7 r=.5 P=$P ttft', round(j['ttft_ms'],3), 'T*', round(j['ttft_over_t_star'],3), 'own', round(j['roofline_attn']['isolated']['achieved']))"; done
