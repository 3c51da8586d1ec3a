#!/bin/bash
# split-KV sizing on 136 SMs by default: full GPU suite, short-suffix microbench, the bench's L8 line
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python tools/attn_bench.py --small 2>&1 | tail -5
timeout 600 python bench.py --no-cpu-baseline | python -c "import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline_attn']; print('L8 ttft', j['ttft_ms'], 'own', r['isolated'], 'M7', j['north_star_point']['ttft_ms'])"
