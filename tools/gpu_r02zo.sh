#!/bin/bash
# fused append by the owning CTA (PCR_APPEND_OWNER=1, default) vs by the last M-block: full GPU suite,
# attention microbench (32 layers) for both, the M7 r=0 / 0.5 bench points
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
ATTN_BENCH_ARGS="--iters 20" PYTEST_K="fused_append" bash tools/gpu_variant.sh "" "-DPCR_APPEND_OWNER=0" "" "-DPCR_APPEND_OWNER=0" 2>&1
for r in 0.0 0.5; do timeout 300 python bench.py --workload M7 --ratio $r --steps 10 --warmup 3 --no-e2e --no-cpu-baseline | python -c "import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline_attn']; print('M7', j['config']['N1'], 'ttft', round(j['ttft_ms'],3), 'own', round(r['isolated']['achieved']), 'clk', j['clocks']['sm_mhz'])"; done
