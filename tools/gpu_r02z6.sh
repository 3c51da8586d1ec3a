#!/bin/bash
# deferred fused-append stores + shift page math + one-thread K/V check: full GPU suite, attention
# microbench, per-phase clocks
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || tail -5 gpurun_out/build.log
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python tools/attn_bench.py 2>&1 | tail -5
timeout 300 python tools/attn_bench.py --small 2>&1 | tail -5
for F in "-DPCR_ATTN_TIMING=1"; do
  echo "== timing flags: $F"
  PCR_NVCC_EXTRA="$F" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; continue; }
  timeout 120 python tools/attn_bench.py --shape 4096,4224,32,8 --iters 1 2>&1 | grep -E "TIMING" | tail -33
done
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
