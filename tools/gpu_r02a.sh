#!/bin/bash
# round-2 first check: smoke, GPU parity suite, one default bench line
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02a_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02a_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=15 > gpurun_out/r02a_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02a_gpu_tests.log
timeout 600 python bench.py > gpurun_out/r02a_bench.jsonl 2> gpurun_out/r02a_bench.err; echo "bench rc=$?" >> gpurun_out/r02a_bench.err
tail -3 gpurun_out/r02a_smoke.log; grep -E "passed|failed|error" gpurun_out/r02a_gpu_tests.log | tail -5; tail -c 1500 gpurun_out/r02a_bench.jsonl; tail -3 gpurun_out/r02a_bench.err
