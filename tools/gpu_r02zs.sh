#!/bin/bash
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tma_store_epilogue or default_priority" 2>&1 | tail -15
