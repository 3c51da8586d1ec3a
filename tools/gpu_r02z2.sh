#!/bin/bash
# per-phase clocks (PCR_ATTN_TIMING) with the kv wait split into V / K and the producers' empty waits
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for F in "-DPCR_ATTN_TIMING=1" "-DPCR_ATTN_TIMING=1 -DPCR_EXP_PINGPONG=0"; do
  echo "== timing flags: $F"
  PCR_NVCC_EXTRA="$F" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; continue; }
  for SH in 4096,4224,32,8; do echo "shape $SH"; timeout 120 python tools/attn_bench.py --shape $SH --iters 1 2>&1 | grep -E "TIMING" | tail -22; done
done 2>&1 | tee gpurun_out/r02z2_timing.txt
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
