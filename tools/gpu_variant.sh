#!/bin/bash
# Kernel variant under compile-time flags: gpu_variant.sh "-DA=1" ... ("" = default build):
# attention parity subset, then the attention microbenchmark.  Restores the default build.
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for F in "$@"; do
  echo "== flags: $F"
  PCR_NVCC_EXTRA="$F" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; continue; }
  timeout 600 python -m pytest tests -m gpu -q -x -k "${PYTEST_K:-attention_and_pool or split_kv or self_consistency or page_size or l8_full or m7_half}" 2>&1 | tail -3
  timeout 300 python tools/attn_bench.py $ATTN_BENCH_ARGS 2>&1 | tail -6
done
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
