#!/bin/bash
# GPU check: smoke + gpu tests, each under its own timeout so a hung kernel cannot wedge the box.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 240 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q ${PYTEST_ARGS:--x} > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -5 gpurun_out/smoke.log; tail -30 gpurun_out/gpu_tests.log
