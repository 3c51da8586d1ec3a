#!/bin/bash
# rotated key-tile order (PCR_KV_ROTATE) vs in-order; then per-phase clocks of the rotated build
mkdir -p gpurun_out; export PYTHONUNBUFFERED=1
PYTEST_K="attention_and_pool or split_kv or self_consistency or page_size or l8_full or m7_half or fused_append or sharding or bitwise" \
  bash tools/gpu_variant.sh "" "-DPCR_KV_ROTATE=0" "-DPCR_KV_ROTATE=3" "-DPCR_KV_ROTATE=7 -DPCR_BLOCK_N=128" 2>&1 | tee gpurun_out/r02z3_variant.txt
for F in "-DPCR_ATTN_TIMING=1"; do
  echo "== timing flags: $F"
  PCR_NVCC_EXTRA="$F" python -m paper_2603_23049_b200.build --force > gpurun_out/build.log 2>&1 || { tail -5 gpurun_out/build.log; continue; }
  for SH in 4096,4224,32,8; do echo "shape $SH"; timeout 120 python tools/attn_bench.py --shape $SH --iters 1 2>&1 | grep -E "TIMING" | tail -22; done
done 2>&1 | tee gpurun_out/r02z3_timing.txt
python -m paper_2603_23049_b200.build --force > /dev/null 2>&1
