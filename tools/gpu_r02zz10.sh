#!/bin/bash
# placement heuristic v3: full suite + per-rank slices
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
A="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
for P in 8 4; do for r in 0.0 0.25 0.5; do timeout 400 python bench.py --workload M7 --ratio $r --rank-slice $P $A 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('M7 r=$r P=$P ttft', round(j['ttft_ms'],3), 'T*', round(j['ttft_over_t_star'],3), 'own', round(j['roofline_attn']['isolated']['achieved']))"; done; done
