#!/bin/bash
# every bench mode still runs on the final build (short runs): modes, offload, layer body, context
# split, copy-engine baselines, T preset, Z trace (DRAM and SSD tiers, Poisson passes)
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
run() { local tag="$1"; shift; timeout 900 python bench.py "$@" > gpurun_out/r02zu_$tag.jsonl 2> gpurun_out/r02zu_$tag.err; local rc=$?;
  python -c "
import json,sys
try:
    j=json.loads(open('gpurun_out/r02zu_$tag.jsonl').read().strip().splitlines()[-1])
    print('$tag rc=$rc', j.get('metric','')[:40], 'value', round(j.get('value') or 0, 1), 'ttft', j.get('ttft_ms') and round(j['ttft_ms'],3), 'dev', j.get('ttft_device_ms') and round(j['ttft_device_ms'],3))
except Exception as e: print('$tag rc=$rc PARSE FAIL', e)"; grep -iE "traceback|error" gpurun_out/r02zu_$tag.err | head -3; }
A="--steps 5 --warmup 3 --no-cpu-baseline --no-target-point --no-e2e"
run sync --mode sync $A
run onlyup --mode only-up --offload --workload M7 --ratio 0.5 $A
run onlydown --mode only-down --offload --workload M7 --ratio 0.5 $A
run body --layer-body $A
run ctx --rank-slice 8 --shard context $A
run ceruns --load-mode ce_runs $A
run tpreset --workload T --steps 5 --warmup 3 --no-target-point
run z --workload Z --requests 200 --no-target-point --no-cpu-baseline
run zssd --workload Z --requests 200 --ssd-frac 0.25 --rho 0.5 --no-target-point --no-cpu-baseline
run l70 --workload L70 --rank-slice 8 --ratio 0.75 $A
