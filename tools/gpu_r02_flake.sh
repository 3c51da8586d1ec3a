#!/bin/bash
# repeatability of the driver's round-end checks on a fresh box: GPU suite twice, smoke, default bench
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for i in 1 2; do timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -1; done
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r02_flake_bench.jsonl 2> gpurun_out/r02_flake_bench.err; echo "bench rc=$?"
python -c "
import json; j=json.loads(open('gpurun_out/r02_flake_bench.jsonl').read().strip().splitlines()[-1]); ns=j['north_star_point']
print('L8 ttft', round(j['ttft_ms'],3), 'value', round(j['value']), 'frac', round(j['roofline']['frac'],3), 'e2e', round(j['e2e']['value']), 'cpu', j['cpu_baseline']['value'], j['cpu_baseline']['cores'], 'launches', j['gpu_launches'], '| M7', round(ns['ttft_ms'],2), round(ns['attn_frac_of_bf16_peak'],3))"
