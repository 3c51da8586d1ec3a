#!/bin/bash
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 1200 python -m pytest tests/test_bench_gpu.py -q -x 2>&1 | tail -30
