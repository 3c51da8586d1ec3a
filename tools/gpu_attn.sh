#!/bin/bash
# attention variants: parity first, then the microbenchmark for each -D variant.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; rc=$?; echo "pytest rc=$rc" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
if [ $rc -ne 0 ]; then grep -E "Error|assert|FAILED" gpurun_out/gpu_tests.log | head -20; exit 1; fi
echo "== default"; timeout 300 python tools/attn_bench.py 2>&1 | tail -6
for V in "${@}"; do
  echo "== $V"
  PCR_NVCC_EXTRA="$V" python -m paper_2603_23049_b200.build --force > /dev/null 2>&1 && timeout 300 python tools/attn_bench.py 2>&1 | tail -6
done
