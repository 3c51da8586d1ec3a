#!/bin/bash
# why the bench's back-to-back attention is slower than attn_bench's: layers 4 vs 32, bench own figure
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for Ly in 4 32 4 32; do timeout 300 python tools/attn_bench.py --shape 4096,4224,32,8 --layers $Ly --iters 10 2>&1 | tail -1; done
for Ly in 4 32; do timeout 300 python tools/attn_bench.py --shape 0,8320,32,8 --layers $Ly --iters 10 2>&1 | tail -1; done
timeout 300 python bench.py --workload M7 --ratio 0.5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | python -c "import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline_attn']; print('bench M7 r=.5 ttft', j['ttft_ms'], 'own', r['isolated'], 'clk', j['clocks']['sm_mhz'])"
