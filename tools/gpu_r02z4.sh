#!/bin/bash
# (1) the q4 / S128 / N0+333 failure of the rotated and 128-key builds, verbose;
# (2) per-phase clocks with the K/V TMA loads skipped (PCR_ATTN_PROFILE=4): is the producer the bound?
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
for F in "-DPCR_KV_ROTATE=7" "-DPCR_BLOCK_N=128"; do
  echo "== flags: $F"
  PCR_NVCC_EXTRA="$F" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; continue; }
  timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "attention_and_pool and S128N0" 2>&1 | grep -E "assert|Error|passed|failed" | head -20
done
for F in "-DPCR_ATTN_TIMING=1 -DPCR_ATTN_PROFILE=4" "-DPCR_ATTN_PROFILE=4"; do
  echo "== flags: $F"
  PCR_NVCC_EXTRA="$F" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; continue; }
  timeout 120 python tools/attn_bench.py --shape 4096,4224,32,8 --iters 3 2>&1 | grep -E "TIMING|tflops" | tail -23
done
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
