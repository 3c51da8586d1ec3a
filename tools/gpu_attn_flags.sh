#!/bin/bash
# Attention microbenchmark under compile-time experiment flags: gpu_attn_flags.sh "-DA=1" "-DB=2" ...
# ("" = default build).  Timing only; parity is the default build's job.
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
for F in "$@"; do
  echo "== flags: $F"
  PCR_NVCC_EXTRA="$F" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; continue; }
  timeout 300 python tools/attn_bench.py $ATTN_BENCH_ARGS 2>&1 | tail -5
done
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
