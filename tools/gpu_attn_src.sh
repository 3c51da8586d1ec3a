#!/bin/bash
# Compare attention kernel sources: for each source, parity tests (attention subset) + microbenchmark.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for SRC in "$@"; do
  echo "== $SRC"
  PCR_ATTN_SRC=$SRC python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; continue; }
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/t.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/t.log
  grep -E "assert|Error" gpurun_out/t.log | head -5
  timeout 300 python tools/attn_bench.py 2>&1 | tail -5
done
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
